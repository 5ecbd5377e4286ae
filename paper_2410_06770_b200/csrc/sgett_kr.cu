// SGETT "k-run" kernel: 3xTF32 on tcgen05 for contractions whose TMEM-side
// operand X has a short contiguous inner k run (c5: orig-A rows hold 40
// contiguous k).  Replaces the fp32 hot loop (kernel.py:48-78 for sgett) for
// such calls.
//
// One k-block = one whole k run of KR floats (KR % 8 == 0, <= 64), so the
// loads follow the data's own contiguity:
//   * X (the accumulator's 128 rows): one TMA box [KR][rows] per k-block, no
//     swizzle, landing dense as [row][KR] — for c5 the box reads 8 runs of
//     2.5 KB (orig-A's k run and its next free mode are adjacent), where the
//     SW32 K-major boxes of sgett_tc.cu issued one 32 B line per row per 8 k.
//     The split warps read each row and write hi (the raw value: the tensor
//     core truncates to tf32) and lo = x - trunc(x) into TMEM with
//     tcgen05.st: X never has to be in a UMMA shared-memory layout.
//   * Y (N = NT <= 128 columns, a multiple of 16; c5: 96, no padding): rows-
//     major boxes [KR k][NT rows], transposed by the split warps into K-major
//     no-swizzle core matrices (hi in place, lo in a small ring).
//   * MMA warp: per 8-k step either the three tf32 MMAs of the 3xTF32 split
//     (hi*hi, hi*lo, lo*hi) or — MIX, the default — one tf32 MMA hi*hi plus one
//     bf16 MMA (K = 16) carrying both cross terms; A from TMEM, B from shared
//     memory, M = 128 (256 for a CTA pair, cta_group::2), N = NT.
//   * Launched as a programmatic dependent (PDL) when g_launch_pdl: the
//     prologue overlaps the predecessor's tail, griddepcontrol.wait precedes
//     the first global access.
//   * Split-K (few output tiles, long K): partials [splits][NY][MX] (x
//     fastest), then the CTAs of a tile reduce them themselves: each
//     publishes its partial and counts in with one atomicInc on the tile's
//     counter (it wraps back to 0 after the last of the `splits` arrivals, so
//     nothing needs resetting between launches or graph replays); the last
//     arriver bumps the tile's generation; a CTA that sees the bump (bounded
//     wait) claims its own slice of the tile for that generation, and the
//     last arriver then claims whatever slice is still unclaimed (no
//     co-residency assumption: a CTA that timed out leaves its slice to it).
//     Each element is summed from -0.0 over the splits in order and added to
//     C once — bitwise what the separate reduce kernel
//     (kernels.cu gett_splitk_reduce_t_kernel) computes.
#include <cuda_bf16.h>

#include <cstdint>
#include <cstdio>

#include "device.cuh"
#include "kernels.hpp"
#include "tmem_io.cuh"

// tuning builds only: skip the TMA loads (1), the X split (2), the Y split (4)
#ifndef GETT_KR_ABLATE
#define GETT_KR_ABLATE 0
#endif

namespace gett {
namespace kr {

constexpr int WG = 128;
constexpr int SPLIT = 2 * WG;
constexpr int MMA_WARP = (WG + SPLIT) / 32;  // warp 12
constexpr int THREADS = WG + SPLIT + 32;
constexpr int NT_MAX = 128;
constexpr uint32_t TMEM_COLS = 512;

constexpr int cmin(int a, int b) { return a < b ? a : b; }

constexpr int MAX_SLOTS = 8;
constexpr int BAR_BYTES = 512;
constexpr int SMEM_MAX = 227 * 1024;

// KRN runs per k-block (1, or 2 for runs <= 40: the k-block is then two
// consecutive runs, the next outer k digit boxed 2 wide): twice the MMAs per
// ready wait + fence + commit, which cost ~350 clk of MMA issue per k-block
// (tools/mma_rate.cu: 15 MMAs 1159 clk, 30 MMAs 1836 clk)
template <int KR, int KRN = 1>
struct Cfg {
  // X staging [run][row][XP]: the box is KR + 4 wide (4 out-of-bounds,
  // zero-filled columns) so the row pitch is an odd multiple of 16 B modulo
  // 128 B and a quarter warp's 16-byte row reads hit 8 distinct bank groups
  static constexpr int XP = KR + 4;
  static constexpr int XB = 128 * XP * 4;      // one run's X box (a multiple of 1 KB: KR + 4 is even)
  static constexpr int XB_AL = (XB + 1023) / 1024 * 1024;  // Y starts 1 KB aligned
  static constexpr int KE = KRN * KR;          // k per k-block
  static constexpr int CHK = KE / 4;           // 16-byte k chunks of an operand row
  static constexpr int CHR = KR / 4;           // ... of one run
  static constexpr uint32_t SBO = CHK * 128;   // bytes between 8-row groups (K-major no swizzle)
  static_assert(KR % 8 == 0 && KR >= 8 && KR <= 64 && (KRN == 1 || (KRN == 2 && KR <= 40)), "k run");
  static_assert(5 * MAX_SLOTS + 1 + 1 + 8 <= BAR_BYTES / 8, "barrier area");
};

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n));
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t"
      "}" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t"
      "}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// K-major no-swizzle shared-memory descriptor (sm_100 version bit 46)
// CTA-pair helpers (cta_group::2): the leader (rank 0) issues the pair MMAs;
// both CTAs' split warps arrive on the leader's ready barrier, its commits
// are multicast to the same barrier offsets in both CTAs
__device__ __forceinline__ void arrive_leader(uint32_t local_bar) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(local_bar));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t"
      "}" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_pair(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t"
      "}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void cluster_sync2() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
         (1ull << 46);
}
__device__ __forceinline__ float tf32_lo(float x) {
  return x - __uint_as_float(__float_as_uint(x) & 0xffffe000u);
}
// mixed split: hi = x rounded to tf32 (half up in magnitude; the tensor core's
// truncation of it is then a no-op), lo = x - hi exactly
__device__ __forceinline__ float tf32_rn(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}
// two floats -> bf16x2 (a in the low half: the even k of a TMEM column / the
// first k of a shared-memory pair)
__device__ __forceinline__ uint32_t bf16x2(float a, float b) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&v);
}
__device__ __forceinline__ void mma_bf16(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tma_load5(uint32_t dst, const CUtensorMap* map, const int32_t* c, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(bar)
      : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// row coordinates of a tile's first row over up to 3 row dims (inner first)
__device__ __forceinline__ void row_coords(int32_t* c, int row0, int nr, const int32_t* ext, const int32_t* pos) {
  int q = row0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    if (i < nr) {
      const int v = q % ext[i];
      q /= ext[i];
#pragma unroll
      for (int j = 0; j < 5; ++j)
        if (pos[i] == j) c[j] = v;
    }
  }
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// claim a slice for generation g: true for exactly one caller per generation
__device__ __forceinline__ bool claim_gen(uint32_t* p, uint32_t g) {
  uint32_t cur = *reinterpret_cast<volatile uint32_t*>(p);
  while (cur != g) {
    const uint32_t prev = atomicCAS(p, cur, g);
    if (prev == cur) return true;
    cur = prev;
  }
  return false;
}

// sum of slice `sl` of tile (x0, y0) over the splits, added to C (threads t
// of nthr).  Every partial of a thread's two elements is loaded before the
// in-order sums (one L2 round trip per 32 splits instead of one per 8).
__device__ __forceinline__ void reduce_slice(const KrParams& p, int x0, int y0, int sl, int t, int nthr) {
  const int64_t E = (int64_t)128 * p.NT;  // tile grid: x = e & 127 (< x_rows), y = e >> 7 (< y_rows)
  const int64_t e0 = E * sl / p.splits, e1 = E * (sl + 1) / p.splits;
  const int64_t mn = (int64_t)p.MX * p.NY;
  for (int64_t eb = e0 + t; eb < e1; eb += 2 * nthr) {
    const float* w[2];
    bool ok[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t e = eb + u * nthr;
      const int x = x0 + (int)(e & 127), y = y0 + (int)(e >> 7);
      ok[u] = e < e1 && (int)(e & 127) < p.x_rows && (int)(e >> 7) < p.y_rows && x < p.MX && y < p.NY;
      w[u] = ok[u] ? p.ws + (int64_t)y * p.MX + x : p.ws;
    }
    float s[2] = {-0.0f, -0.0f};
    for (int sp0 = 0; sp0 < p.splits; sp0 += 32) {
      float v[2][32];
#pragma unroll
      for (int j = 0; j < 32; ++j)
#pragma unroll
        for (int u = 0; u < 2; ++u) v[u][j] = (ok[u] && sp0 + j < p.splits) ? __ldcg(w[u] + (sp0 + j) * mn) : 0.f;
#pragma unroll
      for (int j = 0; j < 32; ++j)
#pragma unroll
        for (int u = 0; u < 2; ++u)
          if (sp0 + j < p.splits) s[u] = s[u] + v[u][j];
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (!ok[u]) continue;
      const int64_t e = eb + u * nthr;
      const int x = x0 + (int)(e & 127), y = y0 + (int)(e >> 7);
      float* c = p.C + p.gx.off(1, x) + p.gy.off(1, y);
      *c = epi(*c, s[u], p.neg);
    }
  }
}

// PAIR: clusters of 2 CTAs (cta_group::2, M = 256): each CTA holds its own
// 128 X rows in TMEM and half of Y's NT rows (Y rows rank * NT/2 ...) as the
// K-major operand in its shared memory; the leader issues one pair MMA per
// (k-step, product) for both — per SM half the Y bytes (loads, split,
// B-operand reads) and half the MMA instructions of the one-CTA form.
// MIX: the mixed split (tools/umma_mixed_test.cu) — per 8 k one tf32 MMA
// hi * hi (hi rounded to tf32) and ONE bf16 MMA (K = 16) whose 16 k are
// [bf16(x) | bf16(x_lo)] against [bf16(y_lo) ; bf16(y)]: both cross terms at
// the bf16 rate, 2 MMAs per 8 k instead of 3.  The lo TMEM columns and the lo
// shared-memory tile hold the bf16 operands in the same geometry (8 columns /
// two 16-byte chunks per 8 k).
template <int KR, int KRN, bool PAIR, bool MIX>
__global__ void __launch_bounds__(THREADS, 1) sgett_kr_kernel(const __grid_constant__ KrParams p) {
  using G = Cfg<KR, KRN>;
  constexpr int KE = G::KE;
  // three rings: load slots [X raw | Y raw] of ONE k run each (TMA -> split;
  // freed by the split warps as soon as they have read them, so the loads run
  // ahead by SL runs whatever the k-block size), operand slots [Y hi | Y lo]
  // K-major of one k-block = KRN runs (split -> MMA; freed by the MMA's commit)
  // and TMEM A slots (hi, lo columns; freed by the commit).  SO == 2 and
  // SL >= 2 KRN (host): a split warpgroup first waits for the commit of its
  // previous k-block (kb - 2), which implies every run up to k-block kb - 2 has
  // landed and been read, and the run that last used any of its load slots is
  // at least 2 KRN runs back — so no full-barrier wait is two phases ahead.
  const int SL = p.lslots, SO = p.oslots, TA = p.aslots;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.bar_off);  // [SL] TMA landed
  uint64_t* lfree = full + MAX_SLOTS;                              // [SL] split read it
  uint64_t* ready = lfree + MAX_SLOTS;                             // [SO] operands + TMEM A written
  uint64_t* ofree = ready + MAX_SLOTS;                             // [SO] MMAs done with the operands
  uint64_t* afree = ofree + MAX_SLOTS;                             // [TA] MMAs done with the TMEM A slot
  uint64_t* done = afree + MAX_SLOTS;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  int* sh = reinterpret_cast<int*>(tmem_slot + 2);  // epilogue broadcast words
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#ifdef GETT_KR_TRACE
  const long long tr_c0 = clock64();
  const unsigned long long tr_start = globaltimer();
  unsigned long long tr_done = 0, tr_arr = 0, tr_own = 0;
  int tr_n = 0;
#endif

  const int ntiles = p.tiles_x * p.tiles_y;
  uint32_t rank = 0;
  if (PAIR) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  int tile, split, tx, ty;
  if (PAIR) {
    // cluster c covers X tiles (2 tp, 2 tp + 1) of column tile ty, K slice split
    const int tx2 = p.tiles_x >> 1, cl = blockIdx.x >> 1;
    const int tpair = cl % (tx2 * p.tiles_y);
    split = cl / (tx2 * p.tiles_y);
    tx = 2 * (tpair % tx2) + (int)rank;
    ty = tpair / tx2;
    tile = ty * p.tiles_x + tx;
  } else {
    tile = blockIdx.x % ntiles;
    split = blockIdx.x / ntiles;
    tx = tile % p.tiles_x;
    ty = tile / p.tiles_x;
  }
  // rows of Y this CTA loads and splits (its half of the pair's N = NT)
  const int yrows_me = PAIR ? p.NT / 2 : p.y_rows;
  const int x0 = tx * p.x_rows, y0 = ty * p.y_rows;
  const int kb0 = split * p.kpc;
  const int nkb = max(0, min(p.nkb, kb0 + p.kpc) - kb0);
  const uint32_t tile_bytes = (uint32_t)(KR * yrows_me * 4);  // one run's Y box (raw [KR][rows])

  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&p.mx) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&p.my) : "memory");
    for (int s = 0; s < SL; ++s) {
      mbar_init(smem_u32(full + s), 1);
      mbar_init(smem_u32(lfree + s), 4);  // the 4 warps of the split warpgroup
    }
    for (int s = 0; s < SO; ++s) {
      mbar_init(smem_u32(ready + s), PAIR ? 8 : 4);  // (pair: the leader's, 4 warps of each CTA)
      mbar_init(smem_u32(ofree + s), 1);  // tcgen05.commit
    }
    for (int s = 0; s < TA; ++s) mbar_init(smem_u32(afree + s), 1);
    mbar_init(smem_u32(done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) {
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (PAIR) cluster_sync2();  // both CTAs' barriers initialised before any remote arrival
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer (one thread) ----------------
    if (lane == 0 && nkb > 0) {
      // launched as a programmatic dependent (g_launch_pdl): the prologue above
      // overlapped the previous kernel's tail; its results (and its reads of the
      // split-K workspace) are complete from here on (a no-op otherwise)
      asm volatile("griddepcontrol.wait;" ::: "memory");
      int32_t cx[5] = {0, 0, 0, 0, 0}, cy[5] = {0, 0, 0, 0, 0};
      row_coords(cx, x0, p.xnr, p.xr_ext, p.xr_pos);
      row_coords(cy, y0 + (PAIR ? (int)rank * yrows_me : 0), p.ynr, p.yr_ext, p.yr_pos);
      int d0 = 0, d1 = 0;  // outer k digits of k-block kb0
      if (p.nko > 0) {
        d0 = (kb0 * KRN) % p.k_ext[0];
        d1 = (kb0 * KRN) / p.k_ext[0];
      }
      const uint32_t sbase = smem_u32(smem);
      // a pair's second Y half can lie wholly past NY (NY = 189: rows 192..255
      // of the second column tile): such a box faults (illegal instruction),
      // so it is not loaded — its columns are never stored
      const bool y_live = !PAIR || y0 + (int)rank * yrows_me < p.NY;
#ifdef GETT_KR_TRACE
      long long w_empty = 0;
#endif
      for (int r = 0; r < nkb * KRN; ++r) {
        const int s = r % SL, u = r / SL;
#ifdef GETT_KR_TRACE
        const long long c0 = clock64();
#endif
        if (u > 0) mbar_wait(smem_u32(lfree + s), (u - 1) & 1);
#ifdef GETT_KR_TRACE
        w_empty += clock64() - c0;
#endif
        const uint32_t fb = smem_u32(full + s);
        int32_t a[5], b[5];
#pragma unroll
        for (int j = 0; j < 5; ++j) {
          a[j] = cx[j] + (p.nko > 0 && p.xk_pos[0] == j ? d0 : 0) + (p.nko > 1 && p.xk_pos[1] == j ? d1 : 0);
          b[j] = cy[j] + (p.nko > 0 && p.yk_pos[0] == j ? d0 : 0) + (p.nko > 1 && p.yk_pos[1] == j ? d1 : 0);
        }
        if (GETT_KR_ABLATE & 1) {
          mbar_arrive(fb);
        } else {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb),
                       "r"((uint32_t)(p.x_rows * G::XP * 4) + (y_live ? tile_bytes : 0u))
                       : "memory");
          tma_load5(sbase + s * p.lslot_bytes, &p.mx, a, fb);
          if (y_live) tma_load5(sbase + s * p.lslot_bytes + G::XB_AL, &p.my, b, fb);
        }
        if (p.nko > 0 && ++d0 == p.k_ext[0]) {
          d0 = 0;
          ++d1;
        }
      }
#ifdef GETT_KR_TRACE
      if (blockIdx.x < 2) printf("KRROLE blk %d producer wait_lfree %lld\n", blockIdx.x, w_empty);
#endif
    }
  } else if (warp < 4) {
    // idle
  } else if (warp < MMA_WARP) {
    // ---------------- split warpgroups (alternate k-blocks), then epilogue ----------------
    const int h = (warp - 4) >> 2, wq = warp & 3, tw = (tid - WG) & (WG - 1);
    // this thread's Y blocks (chunk c of 4 k, row quad rq): source byte offset
    // in the [KR][NT] box, destination of the quad's first row in the K-major
    // tiles, store rotation
    constexpr int YU = (G::CHR * (NT_MAX / 4) + WG - 1) / WG;  // per run
    uint32_t y_src[YU], y_dst[YU];
    int y_rot[YU];
    const int nq = yrows_me >> 2;  // row quads of the box (rows % 4 == 0)
    int ny_units = 0;
    // (MIX: lanes l and l ^ 8 hold the two 4-k chunks of one 8-k step for the
    // same row quad and exchange halves, so each stores whole 16-byte bf16
    // chunks — the even chunk's lane the y_lo chunk, the odd one's the y chunk;
    // a quarter warp still covers 8 consecutive row quads of one chunk)
    bool y_ok[YU];
#pragma unroll
    for (int i = 0; i < YU; ++i) {
      const int uu = tw + WG * i;
      int c, rq;
      if (MIX) {
        const int pp = ((uu >> 4) << 3) | (uu & 7), e = (uu >> 3) & 1;
        const int cp = pp / nq;
        rq = pp - cp * nq;
        c = 2 * cp + e;
      } else {
        c = uu / nq;
        rq = uu - c * nq;
      }
      y_ok[i] = c < G::CHR;
      y_src[i] = (uint32_t)(4 * c * yrows_me * 4 + rq * 16);
      y_dst[i] = (uint32_t)(((4 * rq) >> 3) * G::SBO + c * 128 + ((4 * rq) & 7) * 16);
      y_rot[i] = (rq >> 1) & 3;
      if (y_ok[i]) ny_units = i + 1;
    }
    if (MIX) ny_units = __reduce_max_sync(0xffffffffu, ny_units);  // (warp-uniform: the exchange is a shuffle)
#ifdef GETT_KR_TRACE
    long long w_full = 0, w_lo = 0, t_x = 0, t_y = 0;
#endif
    for (int kb = h; kb < nkb; kb += 2) {
      const int so = kb % SO, sa = kb % TA;
#ifdef GETT_KR_TRACE
      long long c0 = clock64();
#endif
      // (first: see the ring comment above; SO == TA: one commit frees a
      // k-block's operand slot and TMEM slot)
      if (kb >= SO) mbar_wait(smem_u32(ofree + so), (kb / SO - 1) & 1);
      if (TA != SO && kb >= TA) mbar_wait(smem_u32(afree + sa), (kb / TA - 1) & 1);
#ifdef GETT_KR_TRACE
      w_lo += clock64() - c0;
#endif
      uint8_t* hi_t = smem + p.o_off + so * p.oslot_bytes;
      uint8_t* lo_t = hi_t + p.oslot_bytes / 2;
#pragma unroll
      for (int q = 0; q < KRN; ++q) {
        const int r = kb * KRN + q, sl = r % SL;
#ifdef GETT_KR_TRACE
        c0 = clock64();
#endif
        mbar_wait(smem_u32(full + sl), (r / SL) & 1);
#ifdef GETT_KR_TRACE
        w_full += clock64() - c0;
        c0 = clock64();
#endif
        const uint8_t* st = smem + sl * p.lslot_bytes;
        // X row -> TMEM hi / lo columns of slot sa (run q at columns q KR), 16
        // (then 8) columns at a time
        if (!(GETT_KR_ABLATE & 2)) {
          const int row = 32 * wq + lane;
          const float4* xr = reinterpret_cast<const float4*>(st + row * G::XP * 4);
          const uint32_t ta = tmem + ((uint32_t)(32 * wq) << 16) + (uint32_t)(p.a_col0 + sa * 2 * KE + q * KR);
#pragma unroll
          for (int c = 0; c < KR; c += 16) {
            constexpr int W = 16;
            const int n = KR - c >= W ? W : 8;
            uint32_t hv[W], lv[W];
#pragma unroll
            for (int q4 = 0; q4 < W / 4; ++q4) {
              if (4 * q4 < n) {
                const float4 v = xr[c / 4 + q4];
                const float f[4] = {v.x, v.y, v.z, v.w};
                if (MIX) {
                  float xl[4];
#pragma unroll
                  for (int j = 0; j < 4; ++j) {
                    const float xh = tf32_rn(f[j]);
                    hv[4 * q4 + j] = __float_as_uint(xh);
                    xl[j] = f[j] - xh;
                  }
                  // 8-k step g = q4 / 2: columns 8g + (0..3) bf16(x), 8g + (4..7) bf16(x_lo)
                  const int cb = 8 * (q4 >> 1) + 2 * (q4 & 1);
                  lv[cb] = bf16x2(f[0], f[1]);
                  lv[cb + 1] = bf16x2(f[2], f[3]);
                  lv[cb + 4] = bf16x2(xl[0], xl[1]);
                  lv[cb + 5] = bf16x2(xl[2], xl[3]);
                } else {
#pragma unroll
                  for (int j = 0; j < 4; ++j) {
                    hv[4 * q4 + j] = __float_as_uint(f[j]);
                    lv[4 * q4 + j] = __float_as_uint(tf32_lo(f[j]));
                  }
                }
              }
            }
            if (n == W) {
              tmemio::tst16(ta + c, hv);
              tmemio::tst16(ta + KE + c, lv);
            } else {
              tmemio::tst8(ta + c, hv);
              tmemio::tst8(ta + KE + c, lv);
            }
          }
        }
#ifdef GETT_KR_TRACE
        t_x += clock64() - c0;
        c0 = clock64();
#endif
        // Y [KR][NT] raw -> K-major hi + lo tiles of operand slot so (run q at
        // k chunks q KR/4 ...), in 4 k x 4 row blocks: four 16-byte row-quad
        // loads (one per k), a register transpose, and per row one 16-byte
        // store of 4 k to hi and to lo; the stores are rotated by the row quad
        // so a quarter warp covers the 8 rows of a core matrix (conflict-free)
        if (!(GETT_KR_ABLATE & 4)) {
          const uint8_t* yb = st + G::XB_AL;
#pragma unroll
          for (int i = 0; i < YU; ++i) {
            if (i < ny_units) {
              const bool ok = y_ok[i];
              float4 v[4];
#pragma unroll
              for (int j = 0; j < 4; ++j)
                v[j] = ok ? *reinterpret_cast<const float4*>(yb + y_src[i] + j * yrows_me * 4)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
              float4 rows[4];
              rows[0] = make_float4(v[0].x, v[1].x, v[2].x, v[3].x);
              rows[1] = make_float4(v[0].y, v[1].y, v[2].y, v[3].y);
              rows[2] = make_float4(v[0].z, v[1].z, v[2].z, v[3].z);
              rows[3] = make_float4(v[0].w, v[1].w, v[2].w, v[3].w);
              const int rot = y_rot[i];
              const uint32_t ob = y_dst[i] + q * (G::CHR * 128);
              if (MIX) {
                // hi rounded to tf32; this lane's half (2 words per row) of the
                // bf16 chunks: the partner's y_lo half goes to the even-chunk
                // lane, the partner's y half to the odd-chunk lane
                const bool odd = ((tw >> 3) & 1) != 0;
                uint2 mine[4], other[4];
#pragma unroll
                for (int r4 = 0; r4 < 4; ++r4) {
                  const float4 y = rows[r4];
                  const float4 yh = make_float4(tf32_rn(y.x), tf32_rn(y.y), tf32_rn(y.z), tf32_rn(y.w));
                  rows[r4] = yh;
                  const uint2 yb2 = make_uint2(bf16x2(y.x, y.y), bf16x2(y.z, y.w));
                  const uint2 yl2 = make_uint2(bf16x2(y.x - yh.x, y.y - yh.y), bf16x2(y.z - yh.z, y.w - yh.w));
                  mine[r4] = odd ? yb2 : yl2;
                  const uint2 send = odd ? yl2 : yb2;
                  other[r4].x = __shfl_xor_sync(0xffffffffu, send.x, 8);
                  other[r4].y = __shfl_xor_sync(0xffffffffu, send.y, 8);
                }
                if (ok) {
#pragma unroll
                  for (int q4 = 0; q4 < 4; ++q4) {
                    const int rq = (q4 + rot) & 3;
                    float4 rw = rows[0];
                    uint2 m2 = mine[0], o2 = other[0];
                    rw = rq == 1 ? rows[1] : rw;
                    m2 = rq == 1 ? mine[1] : m2;
                    o2 = rq == 1 ? other[1] : o2;
                    rw = rq == 2 ? rows[2] : rw;
                    m2 = rq == 2 ? mine[2] : m2;
                    o2 = rq == 2 ? other[2] : o2;
                    rw = rq == 3 ? rows[3] : rw;
                    m2 = rq == 3 ? mine[3] : m2;
                    o2 = rq == 3 ? other[3] : o2;
                    const uint32_t o = ob + rq * 16;
                    *reinterpret_cast<float4*>(hi_t + o) = rw;
                    // (k order inside the chunk: the even 4-k chunk first)
                    *reinterpret_cast<uint4*>(lo_t + o) =
                        odd ? make_uint4(o2.x, o2.y, m2.x, m2.y) : make_uint4(m2.x, m2.y, o2.x, o2.y);
                  }
                }
              } else {
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                  float4 rw = rows[0];
                  const int rq = (q4 + rot) & 3;
                  rw = rq == 1 ? rows[1] : rw;
                  rw = rq == 2 ? rows[2] : rw;
                  rw = rq == 3 ? rows[3] : rw;
                  const uint32_t o = ob + rq * 16;
                  *reinterpret_cast<float4*>(hi_t + o) = rw;
                  *reinterpret_cast<float4*>(lo_t + o) =
                      make_float4(tf32_lo(rw.x), tf32_lo(rw.y), tf32_lo(rw.z), tf32_lo(rw.w));
                }
              }
            }
          }
        }
        // the load slot is free once every warp of the group has read it
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(lfree + sl));
#ifdef GETT_KR_TRACE
        t_y += clock64() - c0;
#endif
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (PAIR) arrive_leader(smem_u32(ready + so));
        else mbar_arrive(smem_u32(ready + so));
      }
    }
#ifdef GETT_KR_TRACE
    if (blockIdx.x < 2 && (tid & 127) == 0)
      printf("KRROLE blk %d split%d wait_full %lld wait_slots %lld x %lld y %lld\n", blockIdx.x, h, w_full, w_lo, t_x, t_y);
#endif
    if (nkb > 0) mbar_wait(smem_u32(done), 0);
    else asm volatile("griddepcontrol.wait;" ::: "memory");  // (no producer ran: order the stores below)
    // the split-K reduce (or whatever follows as a programmatic dependent) may
    // be scheduled now; it waits for this grid's completion before reading
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#ifdef GETT_KR_TRACE
    tr_done = globaltimer();
#endif
    // ---------------- epilogue ----------------
    // (rows >= x_rows and columns >= y_rows of the accumulator hold garbage:
    // the boxes did not fill them)
    const int row = 32 * wq + lane, x = row < p.x_rows ? x0 + row : p.MX;
    const int half = p.NT >> 1, cbeg = h * half;
    uint32_t rr[64];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (8 * q < half)
        tmemio::tld8(tmem + ((uint32_t)(32 * wq) << 16) + (uint32_t)(cbeg + 8 * q), rr + 8 * q);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#ifdef GETT_KR_TRACE
    const unsigned long long tr_ld = globaltimer();
    unsigned long long tr_st = 0, tr_fe = 0, tr_a0 = 0;
#endif
    if (p.splits == 1) {
      if (x < p.MX) {
        const int64_t ox = p.gx.off(1, x);
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          const int y = y0 + cbeg + i;
          if (i < half && cbeg + i < p.y_rows && y < p.NY) {
            float* c = p.C + ox + p.gy.off(1, y);
            *c = epi(*c, nkb > 0 ? __uint_as_float(rr[i]) : -0.0f, p.neg);
          }
        }
      }
    } else {
      const int64_t mn = (int64_t)p.MX * p.NY;
      if (x < p.MX) {
        float* w = p.ws + split * mn + x;
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          const int y = y0 + cbeg + i;
          if (i < half && cbeg + i < p.y_rows && y < p.NY)
            __stcg(w + (int64_t)y * p.MX, nkb > 0 ? __uint_as_float(rr[i]) : -0.0f);
        }
      }
      if (p.cnt != nullptr) {
        // fused reduce: count in, then reduce the slices this CTA claims
        const int t = tid - WG;  // 0..255 over the two warpgroups
#ifdef GETT_KR_TRACE
        tr_st = globaltimer();
#endif
        __threadfence();
#ifdef GETT_KR_TRACE
        tr_fe = globaltimer();
#endif
        asm volatile("bar.sync 3, %0;" ::"n"(SPLIT) : "memory");
        uint32_t* claims = p.claim + (int64_t)tile * KR_MAX_SPLITS;
        if (t == 0) {
          // the generation before this launch's arrivals (the last arriver
          // bumps it only after every split, this one included, arrived)
          const uint32_t g0 = *reinterpret_cast<volatile uint32_t*>(p.gen + tile);
          uint32_t old;
          asm volatile("atom.acq_rel.gpu.global.inc.u32 %0, [%1], %2;" : "=r"(old) : "l"(p.cnt + tile), "r"((uint32_t)p.splits - 1) : "memory");
#ifdef GETT_KR_TRACE
          tr_a0 = globaltimer();
#endif
          int mine;
          if (old == (uint32_t)p.splits - 1) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p.gen + tile) : "memory");
            mine = 2;  // last arriver: own slice, then every unclaimed one
          } else {
            const unsigned long long t0 = globaltimer();
            while (ld_acquire_u32(p.gen + tile) == g0) {
              if (globaltimer() - t0 > (unsigned long long)p.spin_ns) break;
              __nanosleep(32);
            }
            mine = ld_acquire_u32(p.gen + tile) != g0 ? 1 : 0;
          }
          sh[0] = mine;
          sh[1] = (mine && claim_gen(claims + split, g0 + 1)) ? 1 : 0;
          sh[2] = (int)(g0 + 1);
        }
        asm volatile("bar.sync 3, %0;" ::"n"(SPLIT) : "memory");
        const int mine = sh[0];
        const uint32_t g1 = (uint32_t)sh[2];
#ifdef GETT_KR_TRACE
        tr_arr = globaltimer();
        tr_n = sh[1];
#endif
        if (sh[1]) reduce_slice(p, x0, y0, split, t, SPLIT);
#ifdef GETT_KR_TRACE
        tr_own = globaltimer();
#endif
        if (mine == 2) {
          // after its own slice, the last arriver claims every slice still
          // unclaimed (owners that timed out) in one parallel round: thread t
          // tries slice t, the winners' bits gather in shared memory
          uint32_t* won = reinterpret_cast<uint32_t*>(sh + 4);
          if (t < 8) won[t] = 0;
          asm volatile("bar.sync 3, %0;" ::"n"(SPLIT) : "memory");
          for (int sl = t; sl < p.splits; sl += SPLIT)
            if (sl != split && claim_gen(claims + sl, g1)) atomicOr(&won[(sl >> 5) & 7], 1u << (sl & 31));
          asm volatile("bar.sync 3, %0;" ::"n"(SPLIT) : "memory");
          for (int sl = 0; sl < p.splits && sl < 256; ++sl)
            if ((won[sl >> 5] >> (sl & 31)) & 1u) {
              reduce_slice(p, x0, y0, sl, t, SPLIT);
#ifdef GETT_KR_TRACE
              tr_n += 100;
#endif
            }
        }
#ifdef GETT_KR_TRACE
        if (t == 0)
          printf("KRTRACE blk %d tile %d split %d start %llu done %llu ld %llu st %llu fe %llu a0 %llu arr %llu own %llu end %llu mine %d n %d clk %lld\n",
                 blockIdx.x, tile, split, tr_start, tr_done, tr_ld, tr_st, tr_fe, tr_a0, tr_arr, tr_own, globaltimer(), mine, tr_n, clock64() - tr_c0);
#endif
      }
    }
  } else {
    // ---------------- MMA warp (pair: the leader's only) ----------------
    if (lane == 0 && nkb > 0 && rank == 0) {
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(p.NT >> 3) << 17) |
                             ((uint32_t)((PAIR ? 256 : 128) >> 4) << 24);
      // kind::f16 with bf16 operands (format 1), fp32 accumulate
      const uint32_t idesc_b = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(p.NT >> 3) << 17) |
                               ((uint32_t)((PAIR ? 256 : 128) >> 4) << 24);
      const uint32_t sbase = smem_u32(smem);
#ifdef GETT_KR_TRACE
      long long w_ready = 0, t_issue = 0;
      unsigned long long g_first = 0;
#endif
      for (int kb = 0; kb < nkb; ++kb) {
        const int so = kb % SO, sa = kb % TA;
#ifdef GETT_KR_TRACE
        long long c0 = clock64();
#endif
#ifndef GETT_KR_NOWAIT  // (tuning builds only: wrong results)
        if (PAIR) mbar_wait_cluster(smem_u32(ready + so), (kb / SO) & 1);
        else mbar_wait(smem_u32(ready + so), (kb / SO) & 1);
#endif
#ifdef GETT_KR_TRACE
        w_ready += clock64() - c0;
        c0 = clock64();
        if (kb == 0) g_first = globaltimer();
#endif
#ifndef GETT_KR_NOFENCE  // (tuning builds only)
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#endif
        const uint32_t hb = sbase + p.o_off + so * p.oslot_bytes;
        const uint32_t lb = hb + p.oslot_bytes / 2;
        const uint32_t ah0 = tmem + p.a_col0 + sa * 2 * KE;
#pragma unroll
        for (int j = 0; j < KE / 8; ++j) {
          const uint64_t bh = sdesc(hb + 256 * j, 128, G::SBO);
          const uint64_t bl = sdesc(lb + 256 * j, 128, G::SBO);
          const uint32_t ah = ah0 + 8 * j, al = ah + KE;
          // (hi*hi, hi*lo_Y, lo_X*hi: the tiled kernel's order when its TMEM
          // operand is this kernel's Y — c5 — so both give the same bits there)
          if (MIX) {
            if (PAIR) {
              mma_tf32_pair(tmem, ah, bh, idesc, (kb | j) != 0);
              mma_bf16_pair(tmem, al, bl, idesc_b, 1);
            } else {
              mma_tf32(tmem, ah, bh, idesc, (kb | j) != 0);
              mma_bf16(tmem, al, bl, idesc_b, 1);
            }
          } else if (PAIR) {
            mma_tf32_pair(tmem, ah, bh, idesc, (kb | j) != 0);
            mma_tf32_pair(tmem, ah, bl, idesc, 1);
            mma_tf32_pair(tmem, al, bh, idesc, 1);
          } else {
            mma_tf32(tmem, ah, bh, idesc, (kb | j) != 0);
            mma_tf32(tmem, ah, bl, idesc, 1);
            mma_tf32(tmem, al, bh, idesc, 1);
          }
        }
#ifdef GETT_KR_PLAIN_ARRIVE  // (tuning builds only: free the slots without tracking the MMAs)
        if (PAIR) {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(ofree + so)) : "memory");
          uint32_t rem;
          asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(rem) : "r"(smem_u32(ofree + so)));
          asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(rem) : "memory");
        } else {
          mbar_arrive(smem_u32(ofree + so));
        }
#else
        if (PAIR) {
          commit_pair(smem_u32(ofree + so));
          if (TA != SO) commit_pair(smem_u32(afree + sa));
        } else {
          commit(smem_u32(ofree + so));
          if (TA != SO) commit(smem_u32(afree + sa));
        }
#endif
#ifdef GETT_KR_TRACE
        t_issue += clock64() - c0;
#endif
      }
      if (PAIR) commit_pair(smem_u32(done));
      else commit(smem_u32(done));
#ifdef GETT_KR_TRACE
      if (blockIdx.x < 4) printf("KRROLE blk %d mma wait_ready %lld issue %lld nkb %d first_ready_ns %llu loop_ns %llu since_start_ns %llu\n", blockIdx.x, w_ready, t_issue, nkb,
                                 g_first - tr_start, globaltimer() - g_first, globaltimer() - tr_start);
#endif
    }
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (PAIR) {
    cluster_sync2();  // the peer's MMAs (issued by the leader) are done with this CTA's smem
    if (warp == MMA_WARP)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  } else if (warp == MMA_WARP) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

template <int KR, int KRN, bool MIX>
cudaError_t launch_t(const KrParams& p, bool pair, cudaStream_t s) {
  if (!pair) {
    auto k = sgett_kr_kernel<KR, KRN, false, MIX>;
    static unsigned long long configured = 0;
    cudaError_t e = ensure_dyn_smem(k, SMEM_MAX, configured);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(p.tiles_x * p.tiles_y * p.splits));
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = p.bar_off + BAR_BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = g_launch_pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, p);
  }
  auto k = sgett_kr_kernel<KR, KRN, true, MIX>;
  static unsigned long long configured2 = 0;
  cudaError_t e = ensure_dyn_smem(k, SMEM_MAX, configured2);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(p.tiles_x * p.tiles_y * p.splits));  // tiles_x even: 2 CTAs per X-tile pair
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = p.bar_off + BAR_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_launch_pdl ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, k, p);
}

template <bool MIX>
cudaError_t launch_m(const KrParams& p, int KR, int KRN, bool pair, cudaStream_t s) {
  if (KRN == 2) {
    switch (KR) {
      case 8: return launch_t<8, 2, MIX>(p, pair, s);
      case 16: return launch_t<16, 2, MIX>(p, pair, s);
      case 24: return launch_t<24, 2, MIX>(p, pair, s);
      case 32: return launch_t<32, 2, MIX>(p, pair, s);
      case 40: return launch_t<40, 2, MIX>(p, pair, s);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (KR) {
    case 8: return launch_t<8, 1, MIX>(p, pair, s);
    case 16: return launch_t<16, 1, MIX>(p, pair, s);
    case 24: return launch_t<24, 1, MIX>(p, pair, s);
    case 32: return launch_t<32, 1, MIX>(p, pair, s);
    case 40: return launch_t<40, 1, MIX>(p, pair, s);
    case 48: return launch_t<48, 1, MIX>(p, pair, s);
    case 56: return launch_t<56, 1, MIX>(p, pair, s);
    case 64: return launch_t<64, 1, MIX>(p, pair, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace kr

cudaError_t launch_sgett_kr(const KrParams& p, int KR, int KRN, bool pair, bool mix, cudaStream_t s) {
  return mix ? kr::launch_m<true>(p, KR, KRN, pair, s) : kr::launch_m<false>(p, KR, KRN, pair, s);
}

int sgett_kr_max_nt() { return kr::NT_MAX; }

}  // namespace gett
