// DGETT, warp-specialised: a producer warpgroup gathers the strided A'/B'
// tiles with cp.async into a 3-stage shared-memory ring (mbarrier full/empty
// handshakes, no block-wide barrier in the main loop); two consumer
// warpgroups run only shared-memory fragment loads + FP64 DMMA
// (mma.sync m8n8k4 -> DMMA.8x8x4) and the fused C += acc epilogue through the
// C offset tables (red.global.add.f64: one IEEE add per element at L2, no
// C loads on the SM).  setmaxnreg moves registers from the producer warpgroup
// (56) to the consumers (208): 2 consumer + 1 producer warp per SM sub-partition.
//
// Same semantics and layouts as gett_tiled_kernel<double> (kernels.cu): the
// tile is 128 x 128, BK 32; smem layouts follow the gmem fast dimension of each
// operand ([row][k] pitch 36 or [k][row] pitch 132 doubles, conflict-free DMMA
// fragment reads); K-tail padding is A' -0.0, B' +0.0 so signed zeros match the
// sequential reference loop (kernel.py:76); split-K writes partials.
#include <cstdint>
#include <cstdio>

#include "device.cuh"
#include "kernels.hpp"

namespace gett {
namespace ws {

// Optional per-role cycle accounting (tuning builds only: make variant
// EXTRA=-DGETT_WS_TRACE); blocks 0 and gridDim.x-1 printf their totals.
#ifdef GETT_WS_TRACE
__device__ __forceinline__ int smid() { int r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }
#define TR_DECL(...) long long __VA_ARGS__;
#define TR_T0() long long _tr0 = clock64();
#define TR_ADD(v) { long long _tr1 = clock64(); v += _tr1 - _tr0; _tr0 = _tr1; }
#define TR_PRINT(...) do { printf(__VA_ARGS__); } while (0)
#else
#define TR_DECL(...)
#define TR_T0()
#define TR_ADD(v)
#define TR_PRINT(...) do { } while (0)
#endif

// tuning builds only: skip the C += acc reductions (measures the epilogue's cost)
#ifndef GETT_WS_NO_EPI
#define GETT_WS_NO_EPI 0
#endif
#ifndef GETT_WS_GROUP_M
#define GETT_WS_GROUP_M 16  // c2: DRAM read 1.54 -> 1.28 GB per launch vs 8, same time
#endif
constexpr int BM = 128, BN = 128, BK = 32, STAGES = 3, PAD = 4, GROUP_M = GETT_WS_GROUP_M;
constexpr int CW = 8;                   // consumer warps (2 warpgroups), warp tile 64 x 32
constexpr int PW = 4;                   // producer warps (1 warpgroup)
constexpr int THREADS = (CW + PW) * 32;
constexpr int CONSUMER_REGS = 208, PRODUCER_REGS = 56;
constexpr int WARPS_N = 4, WARPS_M = CW / WARPS_N;
constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
constexpr int MI = WM / 8, NJ = WN / 8;
constexpr int KF_PITCH = BK + PAD;   // [row][k]: 36 doubles (= 4 mod 16: conflict-free frags)
constexpr int RF_PITCH = 128 + PAD;  // [k][row]: 132 doubles
constexpr int OPER_ELEMS = 128 * KF_PITCH > BK * RF_PITCH ? 128 * KF_PITCH : BK * RF_PITCH;
constexpr int STAGE_ELEMS = 2 * OPER_ELEMS;
constexpr int BAR_BYTES = 64;
constexpr int ROWOFF_BYTES = 2 * 128 * 8;
constexpr int SMEM_BYTES = STAGES * STAGE_ELEMS * 8 + BAR_BYTES + ROWOFF_BYTES;
// TMA-fed operands (both A' and B' affine boxes) land in exactly the padded
// layouts the gathers write — [row][k] pitch 36 or [k][row] pitch 132 — so the
// consumers are unchanged: each box is 4 elements wider than the tile along
// its fast dimension, and the host cuts that dimension into tile-sized
// digits, so the 4 extra columns are out of bounds and zero-filled.  (128B-
// swizzled dense boxes gave the DMMA fragment loads 2-way bank conflicts.)
// One thread issues one box per operand.
constexpr int T_KF_BYTES = 128 * KF_PITCH * 8;  // a k-fast box: 128 rows x 36
constexpr int T_RF_BYTES = BK * RF_PITCH * 8;   // a rows-fast box: 32 k x 132
// Bulk-add epilogue (p.c_bulk): each consumer warp stages its 64 x 32 block
// as 8-row chunks, [row][34] (the 16-byte row shift spreads a warp's
// fragment stores over all banks), and adds each 32-wide row run into C with
// one cp.reduce.async.bulk .add.f64 — done at L2 like red.add: one IEEE
// round-to-nearest add per element, the same result, and a 256-byte request
// instead of 32 scattered 8-byte ones.  The staging buffer is the ring slot
// after the tile's last k-block, which carries no data for it: the producer
// completes that slot's `full` phase once all consumer warps have released
// its previous k-block (so no warp still reads it — warps leave the k loop
// up to a k-block apart), and the consumers release it after the bulk reads.
// Four chunks per pass: 8 warps x 4 x 8 rows x 272 B fit a slot.
constexpr int EP_PITCH = 34;
constexpr int EP_CHUNKS = 4;
constexpr int EP_WARP_ELEMS = EP_CHUNKS * 8 * EP_PITCH;
static_assert(CW * EP_WARP_ELEMS <= STAGE_ELEMS, "bulk-add staging exceeds a stage");
static_assert(MI % EP_CHUNKS == 0 && WN == 32, "bulk-add staging shape");


// one lane of the (converged) warp: true for it, false for the others
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void mbar_init(uint32_t addr, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(addr), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t addr) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(addr)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_cpasync(uint32_t addr) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t"
      "}" ::"r"(addr),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Producer warp pw (0..PW-1): gather its share of one operand's 128 x BK tile
// for k-block [k0, k0+BK).  KF: smem [row][k] (gmem fast along k; the warp
// owns rows [32 pw, 32 pw + 32)), else [k][row] (the warp owns k-lines
// [8 pw, 8 pw + 8)).  VEC: 16-byte copies (2 doubles) along the fast dim.
template <bool KF, bool VEC, bool IS_A>
__device__ __forceinline__ void produce(double* s, const double* base, const int64_t* rowoff,
                                        int nrows_valid, const GroupDev& gk, int kt, int k0,
                                        int kend, int pw, int lane) {
  const double kpad = IS_A ? -0.0 : 0.0;
  constexpr int V = VEC ? 2 : 1;
  if (KF) {
    constexpr int CPL = BK / V;      // chunks per row: 16 or 32
    constexpr int RSTEP = 32 / CPL;  // rows per warp pass: 2 or 1
    const int c = lane % CPL;
    const int k = k0 + c * V;
    const bool kok = k < kend;
    const int64_t ko = kok ? gk.off(kt, k) : 0;
#pragma unroll 4
    for (int r = 32 * pw + lane / CPL; r < 32 * pw + 32; r += RSTEP) {
      double* dst = s + r * KF_PITCH + c * V;
      if (kok && r < nrows_valid) {
        const double* src = base + rowoff[r] + ko;
        if (VEC) cp_async_16(dst, src);
        else cp_async_8(dst, src);
      } else {
#pragma unroll
        for (int v = 0; v < V; ++v) dst[v] = kok ? 0.0 : kpad;
      }
    }
  } else {
    constexpr int CPK = 128 / V;  // chunks per k line: 64 or 128
    constexpr int KPW = BK / PW;  // k lines per producer warp: 8
    const int kl = k0 + KPW * pw + (lane % KPW);
    const int64_t my_ko = kl < kend ? gk.off(kt, kl) : 0;
#pragma unroll 1
    for (int j = 0; j < KPW; ++j) {
      const int kk = KPW * pw + j;
      const int64_t ko = __shfl_sync(0xffffffffu, my_ko, j);
      const bool kok = k0 + kk < kend;
#pragma unroll
      for (int q = 0; q < CPK / 32; ++q) {
        const int r = (lane + 32 * q) * V;
        double* dst = s + kk * RF_PITCH + r;
        if (kok && r < nrows_valid) {
          const double* src = base + rowoff[r] + ko;
          if (VEC) cp_async_16(dst, src);
          else cp_async_8(dst, src);
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v) dst[v] = kok ? 0.0 : kpad;
        }
      }
    }
  }
}

// One unit of work for a CTA: k-blocks [kb0, kb1) of tile `tile` (k-block kb
// covers k in [kbase + kb*BK, +BK) clipped to kend), and what the epilogue does
// with the accumulator.
enum SegKind : int {
  SEG_FULL = 0,    // whole tile: C += acc
  SEG_SPLITK = 1,  // split-K slice: partial -> workspace (gett_splitk_reduce_kernel)
  SEG_HEAD = 2,    // stream-K: first part of a tile; adds the tail's partial, then C += acc
  SEG_TAIL = 3,    // stream-K: last part of a tile; partial -> part[cta], flag[cta] = epoch
};
struct Seg {
  int tile, split, kbase, kend, kb0, kb1, kind;
  int rev;  // the producer walks the k-blocks downwards (serpentine k, see seg_next)
};

// Per-CTA work list, identical in the producer and consumer roles.
//   grid mode (sk.enabled == 0): one segment = tile blockIdx.x % ntiles, split
//     blockIdx.x / ntiles (the classic one-tile-per-CTA launch, split-K capable);
//   stream-K mode: the CTA first takes its equal share [c*U/G, (c+1)*U/G) of
//     the k-block units of the stream-K tiles (the last 1-2 waves' worth), then
//     the data-parallel tiles c, c+G, ...  Units are equal in length, so tile
//     boundaries fall at different times in different CTAs: the C epilogues of
//     concurrently running CTAs no longer hit HBM in one synchronized burst,
//     and the partial last wave disappears.  A tile cut by the CTA boundary c
//     is shared by CTA c-1 (head) and CTA c (tail); with fewer tiles than CTAs
//     the shares are shorter than a tile and a tile may also have middle
//     pieces (CTAs whose whole share lies inside it): they publish like tails
//     and the head adds all of them in CTA order.
struct SegIter {
  int64_t u, u_end;  // stream-K units still to take
  int dp;            // next data-parallel tile
  bool done;
};

__device__ __forceinline__ void seg_init(const TiledParams<double>& p, const SkParams& sk,
                                         SegIter& it) {
  it.done = false;
  if (!sk.enabled) {
    it.u = it.u_end = 0;
    it.dp = -1;
    return;
  }
  const int64_t G = gridDim.x, c = blockIdx.x;
  it.u = sk.sk_units * c / G;
  it.u_end = sk.sk_units * (c + 1) / G;
  it.dp = (int)c;
}

__device__ __forceinline__ bool seg_next(const TiledParams<double>& p, const SkParams& sk,
                                         SegIter& it, Seg& sg) {
  if (it.done) return false;
  sg.rev = 0;
  if (!sk.enabled) {
    const int ntiles = p.tiles_m * p.tiles_n;
    sg.tile = blockIdx.x % ntiles;
    sg.split = blockIdx.x / ntiles;
    sg.kbase = sg.split * p.k_chunk;
    sg.kend = min(p.K, sg.kbase + p.k_chunk);
    sg.kb0 = 0;
    sg.kb1 = sg.kend > sg.kbase ? (sg.kend - sg.kbase + BK - 1) / BK : 0;
    sg.kind = p.splits == 1 ? SEG_FULL : SEG_SPLITK;
    it.done = true;
    return true;
  }
  sg.split = 0;
  sg.kbase = 0;
  sg.kend = p.K;
  if (it.u < it.u_end) {
    const int nkb = sk.nkb;
    sg.tile = sk.sk_tile0 + (int)(it.u / nkb);
    sg.kb0 = (int)(it.u % nkb);
    sg.kb1 = (int)min((int64_t)nkb, sg.kb0 + (it.u_end - it.u));
    sg.kind = sg.kb0 == 0 ? (sg.kb1 == nkb ? SEG_FULL : SEG_HEAD) : SEG_TAIL;
    it.u += sg.kb1 - sg.kb0;
    return true;
  }
  if (it.dp < sk.sk_tile0) {
    sg.tile = it.dp;
    sg.kb0 = 0;
    sg.kb1 = sk.nkb;
    sg.kind = SEG_FULL;
    // serpentine k (l2hint bit 4): every other data-parallel tile of a CTA is
    // summed from its last k-block down, so a wave starts on the k slices the
    // previous wave (same tile rows, next columns) touched last — the part of
    // the shared row panels still in L2
    sg.rev = (sk.l2hint & 16) ? ((it.dp / (int)gridDim.x) & 1) : 0;
    it.dp += gridDim.x;
    return true;
  }
  it.done = true;
  return false;
}

// C += acc of this segment goes through the bulk-add epilogue, which takes
// one extra (data-less) ring slot after the segment's k-blocks
__device__ __forceinline__ bool bulk_epilogue(const TiledParams<double>& p, const Seg& sg) {
  return p.c_bulk && (sg.kind == SEG_FULL || sg.kind == SEG_HEAD) && sg.kb1 > sg.kb0;
}

__device__ __forceinline__ void tile_origin(const TiledParams<double>& p, int tile, int& m0,
                                            int& n0) {
  const int per_group = GROUP_M * p.tiles_n;
  const int group = tile / per_group;
  const int first_m = group * GROUP_M;
  const int gsize = min(p.tiles_m - first_m, GROUP_M);
  const int in_group = tile % per_group;
  m0 = (first_m + in_group % gsize) * BM;
  n0 = (in_group / gsize) * BN;
}

// TMA box coordinates of one operand for a tile and a k-block: the mixed-radix
// digits of the tile's first row over the row dims and of the k-block's first
// k over the k dims, placed at their tensor-map dims (TmaOperand, built by the
// host: capi.cu dgett_tma_layout)
__device__ __forceinline__ void dtma_coords(const TmaOperand& op, int row0, int k0, int32_t* c) {
#pragma unroll
  for (int j = 0; j < 5; ++j) c[j] = 0;
  int q = row0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
    if (i < op.nr) {
      const int v = q % op.r_ext[i];
      q /= op.r_ext[i];
#pragma unroll
      for (int j = 0; j < 5; ++j)
        if (op.r_pos[i] == j) c[j] = v;
    }
  q = k0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
    if (i < op.nk) {
      const int v = q % op.k_ext[i];
      q /= op.k_ext[i];
#pragma unroll
      for (int j = 0; j < 5; ++j)
        if (op.k_pos[i] == j) c[j] = v;
    }
}

__device__ __forceinline__ void dtma_load(uint32_t dst, const CUtensorMap* map, const int32_t* c, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void dtma_load_hint(uint32_t dst, const CUtensorMap* map, const int32_t* c, uint32_t bar,
                                               uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(dst),
      "l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

template <bool AKF, bool BKF, bool AVEC, bool BVEC, bool TMA>
__global__ void __launch_bounds__(THREADS, 1)
    dgett_ws_kernel(const __grid_constant__ TiledParams<double> p,
                    const __grid_constant__ SkParams sk, const __grid_constant__ TmaParams tp) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* sbase_ptr = smem_raw;
  double* smem = reinterpret_cast<double*>(sbase_ptr);
  constexpr int RING_BYTES = STAGES * STAGE_ELEMS * 8;
  constexpr int SOPER = OPER_ELEMS;    // doubles per operand tile
  constexpr int SSTAGE = STAGE_ELEMS;  // doubles per stage
  uint64_t* full = reinterpret_cast<uint64_t*>(sbase_ptr + RING_BYTES);
  uint64_t* empty = full + STAGES;
  int64_t* rowoff_a = reinterpret_cast<int64_t*>(sbase_ptr + RING_BYTES + BAR_BYTES);
  int64_t* rowoff_b = rowoff_a + 128;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    if (TMA) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tp.map[0]) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tp.map[1]) : "memory");
    }
    for (int s = 0; s < STAGES; ++s) {
      // per producer lane: cp.async + plain arrival; TMA: the expect_tx arrival
      mbar_init(smem_u32(full + s), TMA ? 1 : 2 * PW * 32);
      mbar_init(smem_u32(empty + s), CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  SegIter it;
  seg_init(p, sk, it);
  Seg sg;

  if (TMA && warp >= CW) {
    // ---------------- TMA producer: one thread, one box per operand ----------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PRODUCER_REGS));
    if (warp != CW || lane != 0) return;
    uint32_t g = 0;
    const uint32_t ring = smem_u32(smem);
    const uint64_t pol_last = policy_evict_last(), pol_first = policy_evict_first();
    const bool swap = (sk.l2hint & 8) != 0;
    const int hint_a = swap ? ((sk.l2hint & 2) ? 2 : 0) : ((sk.l2hint & 1) ? 1 : 0);  // 1 evict_last, 2 evict_first
    const int hint_b = swap ? ((sk.l2hint & 1) ? 1 : 0) : ((sk.l2hint & 2) ? 2 : 0);
    while (seg_next(p, sk, it, sg)) {
      int m0, n0;
      tile_origin(p, sg.tile, m0, n0);
      for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++g) {
        const int s = g % STAGES, u = g / STAGES;
        if (u > 0) mbar_wait(smem_u32(empty + s), (u - 1) & 1);
        const uint32_t fb = smem_u32(full + s);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb),
                     "r"((AKF ? T_KF_BYTES : T_RF_BYTES) + (BKF ? T_KF_BYTES : T_RF_BYTES))
                     : "memory");
        const int k0 = sg.kbase + (sg.rev ? sg.kb0 + sg.kb1 - 1 - kb : kb) * BK;
        int32_t c[5];
        dtma_coords(tp.op[0], m0, k0, c);
        if (hint_a) dtma_load_hint(ring + s * STAGE_ELEMS * 8, &tp.map[0], c, fb, hint_a == 1 ? pol_last : pol_first);
        else dtma_load(ring + s * STAGE_ELEMS * 8, &tp.map[0], c, fb);
        dtma_coords(tp.op[1], n0, k0, c);
        if (hint_b)
          dtma_load_hint(ring + s * STAGE_ELEMS * 8 + OPER_ELEMS * 8, &tp.map[1], c, fb,
                         hint_b == 1 ? pol_last : pol_first);
        else dtma_load(ring + s * STAGE_ELEMS * 8 + OPER_ELEMS * 8, &tp.map[1], c, fb);
      }
      if (bulk_epilogue(p, sg)) {
        // the epilogue's staging slot: completes its `full` phase without data
        // once the consumers have released the slot's previous k-block
        const int s = g % STAGES, u = g / STAGES;
        if (u > 0) mbar_wait(smem_u32(empty + s), (u - 1) & 1);
        mbar_arrive(smem_u32(full + s));
        ++g;
      }
    }
    return;
  }
  if (warp >= CW) {
    // ---------------- producer warpgroup ----------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PRODUCER_REGS));
    const int pw = warp - CW, ptid = tid - CW * 32;
    uint32_t g = 0;  // k-blocks produced so far (the stage ring runs across segments)
    while (seg_next(p, sk, it, sg)) {
      int m0, n0;
      tile_origin(p, sg.tile, m0, n0);
      const int mvalid = min(BM, p.M - m0), nvalid = min(BN, p.N - n0);
      // the previous segment's copies were issued with the old row offsets:
      // all producer warps pass before they are overwritten
      asm volatile("bar.sync 2, %0;" ::"n"(PW * 32) : "memory");
      for (int r = ptid; r < 128; r += PW * 32) {
        rowoff_a[r] = r < mvalid ? p.gm.off(0, m0 + r) : 0;
        rowoff_b[r] = r < nvalid ? p.gn.off(0, n0 + r) : 0;
      }
      asm volatile("bar.sync 2, %0;" ::"n"(PW * 32) : "memory");
      for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++g) {
        const int s = g % STAGES, u = g / STAGES;
        if (u > 0) mbar_wait(smem_u32(empty + s), (u - 1) & 1);
        double* sa = smem + s * SSTAGE;
        double* sb = sa + SOPER;
        const int k0 = sg.kbase + (sg.rev ? sg.kb0 + sg.kb1 - 1 - kb : kb) * BK;
        produce<AKF, AVEC, true>(sa, p.A, rowoff_a, mvalid, p.gk, 0, k0, sg.kend, pw, lane);
        produce<BKF, BVEC, false>(sb, p.B, rowoff_b, nvalid, p.gk, 1, k0, sg.kend, pw, lane);
        mbar_arrive_cpasync(smem_u32(full + s));  // fires when this lane's copies land
        mbar_arrive(smem_u32(full + s));          // publishes this lane's padding stores
      }
      if (bulk_epilogue(p, sg)) {
        // the epilogue's staging slot (see the TMA producer)
        const int s = g % STAGES, u = g / STAGES;
        if (u > 0) mbar_wait(smem_u32(empty + s), (u - 1) & 1);
        mbar_arrive(smem_u32(full + s));
        mbar_arrive(smem_u32(full + s));
        ++g;
      }
    }
    cp_async_wait<0>();
    return;
  }

  // ---------------- consumer warpgroups ----------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(CONSUMER_REGS));
  const int wm0 = (warp / WARPS_N) * WM, wn0 = (warp % WARPS_N) * WN;
  int aoff[MI], boff[NJ];
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    int r = wm0 + i * 8 + (lane >> 2);
    aoff[i] = AKF ? r * KF_PITCH + (lane & 3) : (lane & 3) * RF_PITCH + r;
  }
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    int c = wn0 + j * 8 + (lane >> 2);
    boff[j] = BKF ? c * KF_PITCH + (lane & 3) : (lane & 3) * RF_PITCH + c;
  }
  constexpr int AKS = AKF ? 4 : 4 * RF_PITCH;
  constexpr int BKS = BKF ? 4 : 4 * RF_PITCH;
  uint32_t g = 0;
  TR_DECL(cw = 0, cc = 0, ce = 0, cx = 0, e_slot = 0, e_st = 0, e_iss = 0, e_rd = 0, e_fin = 0, cw_first = 0, cw_seg0 = 0)
  TR_T0()
  int nseg = 0;
  while (seg_next(p, sk, it, sg)) {
    ++nseg;
#ifdef GETT_WS_TRACE_SEGS
    if (blockIdx.x == 0 && lane == 0 && (warp == 0 || warp == CW / 2) && nseg <= 12)
      printf("seg %d warp %d clk %lld kind %d kb %d..%d\n", nseg, warp, clock64(), (int)sg.kind, sg.kb0, sg.kb1);
#endif
    int m0, n0;
    tile_origin(p, sg.tile, m0, n0);
    double acc[MI][NJ][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = -0.0;

#pragma unroll 1
    for (int kb = sg.kb0; kb < sg.kb1; ++kb, ++g) {
      const int s = g % STAGES, u = g / STAGES;
      mbar_wait(smem_u32(full + s), u & 1);
#ifdef GETT_WS_TRACE
      if (g == 0) TR_ADD(cw_first)
      else if (kb == sg.kb0) TR_ADD(cw_seg0)
      else
#endif
      TR_ADD(cw)
      const double* As = smem + s * SSTAGE;
      const double* Bs = As + SOPER;
      double a[2][MI], b[2][NJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[0][i] = As[aoff[i]];
#pragma unroll
      for (int j = 0; j < NJ; ++j) b[0][j] = Bs[boff[j]];
#pragma unroll
      for (int ks = 0; ks < BK / 4; ++ks) {
        const int cur = ks & 1;
        if (ks + 1 < BK / 4) {
#pragma unroll
          for (int i = 0; i < MI; ++i) a[cur ^ 1][i] = As[aoff[i] + (ks + 1) * AKS];
#pragma unroll
          for (int j = 0; j < NJ; ++j) b[cur ^ 1][j] = Bs[boff[j] + (ks + 1) * BKS];
        }
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NJ; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[cur][i], b[cur][j]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(empty + s));
      TR_ADD(cc)
    }

    // epilogue: acc[i][j][e] is C'(m0+wm0+i*8+lane/4, n0+wn0+j*8+2*(lane%4)+e)
    if (sg.kind == SEG_TAIL) {
      // publish this part for the head's CTA (boundary blockIdx.x)
      double* w = sk.part + (int64_t)blockIdx.x * (BM * BN);
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j)
          __stcg(reinterpret_cast<double2*>(w + (wm0 + i * 8 + (lane >> 2)) * BN + wn0 + j * 8 +
                                            2 * (lane & 3)),
                 make_double2(acc[i][j][0], acc[i][j][1]));
      __threadfence();
      asm volatile("bar.sync 1, %0;" ::"n"(CW * 32) : "memory");
      if (tid == 0)
        asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(sk.flags + blockIdx.x),
                     "r"(sk.epoch)
                     : "memory");
      TR_ADD(cx)
      continue;
    }
    if (sg.kind == SEG_HEAD) {
      // the rest of the tile belongs to CTAs blockIdx.x + 1, ... (one, or more
      // when the shares are shorter than a tile); wait for each one's published
      // part and add them in CTA order: acc = head + p1 + p2 ..., the same
      // order for every element
      const int64_t G = gridDim.x;
      const int64_t tile_end = (int64_t)(sg.tile - sk.sk_tile0 + 1) * sk.nkb;
      for (int64_t c2 = blockIdx.x + 1; c2 < G && sk.sk_units * c2 / G < tile_end; ++c2) {
        const int* f = sk.flags + c2;
        int v;
        do {
          asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        } while (v != sk.epoch);
        const double* w = sk.part + c2 * (BM * BN);
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int j = 0; j < NJ; ++j) {
            const double2 t = __ldcg(reinterpret_cast<const double2*>(
                w + (wm0 + i * 8 + (lane >> 2)) * BN + wn0 + j * 8 + 2 * (lane & 3)));
            acc[i][j][0] = acc[i][j][0] + t.x;
            acc[i][j][1] = acc[i][j][1] + t.y;
          }
      }
    }
    if (bulk_epilogue(p, sg)) {
      // C's 32-wide row runs are contiguous and 16-byte aligned (host check).
      // The ring slot after the tile's last k-block carries no data: the
      // producer signals its `full` phase once every warp has released the
      // slot's previous k-block, so no warp still reads what is staged here.
      // Stage, then lane l adds row l of the pass with one bulk reduction.
      const int sx = g % STAGES;
      TR_ADD(ce)
      mbar_wait(smem_u32(full + sx), (g / STAGES) & 1);
      TR_ADD(e_slot)
      double* stg = smem + sx * SSTAGE + warp * EP_WARP_ELEMS;
      const uint32_t stg_u = smem_u32(stg);
      const int nb = n0 + wn0;
      const int64_t cb = nb < p.N ? p.gn.off(1, nb) : 0;
#pragma unroll
      for (int pass = 0; pass < MI / EP_CHUNKS; ++pass) {
        if (pass > 0) {
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
          TR_ADD(e_rd)
        }
#pragma unroll
        for (int ii = 0; ii < EP_CHUNKS; ++ii) {
          const int i = pass * EP_CHUNKS + ii;
#pragma unroll
          for (int j = 0; j < NJ; ++j) {
            const double x0 = p.neg ? -acc[i][j][0] : acc[i][j][0];
            const double x1 = p.neg ? -acc[i][j][1] : acc[i][j][1];
            *reinterpret_cast<double2*>(stg + (ii * 8 + (lane >> 2)) * EP_PITCH + j * 8 + 2 * (lane & 3)) =
                make_double2(x0, x1);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        TR_ADD(e_st)
        const int mf = m0 + wm0 + pass * EP_CHUNKS * 8;
        if (p.c_bulk & 2) {
          // rows mf .. mf+31 lie in one inner run of C's M group: row l's run
          // starts at row mf's + l * stride; one thread issues all the adds
          // from warp-uniform operands (no per-lane issue loop)
          const int nrows = __shfl_sync(0xffffffffu, min(32, p.M - mf), 0);
          const int64_t base = __shfl_sync(0xffffffffu, mf < p.M ? p.gm.off(1, mf) + cb : 0, 0);
          const uint32_t src = __shfl_sync(0xffffffffu, stg_u, 0);
          if (nb < p.N && !GETT_WS_NO_EPI && elect_one()) {
            const int64_t rs = p.gm.s_in[1];
            const double* dst = p.C + base;
            if (sk.l2hint & 4) {
              // C's lines are touched once per call: let them leave L2 first
              const uint64_t pol = policy_evict_first();
#pragma unroll 4
              for (int l = 0; l < nrows; ++l)
                asm volatile(
                    "cp.reduce.async.bulk.global.shared::cta.bulk_group.L2::cache_hint.add.f64 [%0], [%1], %2, %3;" ::"l"(
                        dst + l * rs),
                    "r"(src + l * EP_PITCH * 8), "n"(WN * 8), "l"(pol)
                    : "memory");
            } else {
#pragma unroll 4
              for (int l = 0; l < nrows; ++l)
                asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(
                                 dst + l * rs),
                             "r"(src + l * EP_PITCH * 8), "n"(WN * 8)
                             : "memory");
            }
          }
        } else {
          const int m = mf + lane;
          if (nb < p.N && m < p.M && !GETT_WS_NO_EPI) {
            const double* dst = p.C + p.gm.off(1, m) + cb;
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(dst),
                         "r"(stg_u + lane * EP_PITCH * 8), "n"(WN * 8)
                         : "memory");
          }
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        __syncwarp();
        TR_ADD(e_iss)
      }
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(empty + sx));
      ++g;
      TR_ADD(e_fin)
      continue;
    }
    const bool to_c = sg.kind != SEG_SPLITK;
    int64_t coff[NJ * 2];
    bool cok[NJ * 2];
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        int n = n0 + wn0 + j * 8 + 2 * (lane & 3) + e;
        cok[j * 2 + e] = n < p.N;
        coff[j * 2 + e] = (n < p.N) ? (to_c ? p.gn.off(1, n) : (int64_t)n) : 0;
      }
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      const int m = m0 + wm0 + i * 8 + (lane >> 2);
      if (m >= p.M) continue;
      if (to_c) {
        const int64_t ro = p.gm.off(1, m);
        // C += acc as fire-and-forget fp64 reductions at L2: one IEEE
        // round-to-nearest add per element (each element is updated by exactly
        // one thread), so the result equals C + acc and stays deterministic,
        // and the SM never waits for the C loads
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            if (cok[j * 2 + e] && !GETT_WS_NO_EPI)
              asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p.C + ro + coff[j * 2 + e]),
                           "d"(p.neg ? -acc[i][j][e] : acc[i][j][e])
                           : "memory");
      } else {
        double* w = p.ws + ((int64_t)sg.split * p.M + m) * p.N;
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            if (cok[j * 2 + e]) w[coff[j * 2 + e]] = acc[i][j][e];
      }
    }
    TR_ADD(ce)
  }
  if (p.c_bulk) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (warp == 0 && lane == 0)
    TR_PRINT("blk %d consumer0: segs %d wait_full %lld compute %lld epilogue %lld tail_publish %lld sm %d "
             "bulk: slot %lld store %lld issue %lld read %lld final %lld first_wait %lld seg0_wait %lld\n",
             blockIdx.x, nseg, cw, cc, ce, cx, smid(), e_slot, e_st, e_iss, e_rd, e_fin, cw_first, cw_seg0);
}

template <bool AKF, bool BKF, bool AV, bool BV, bool TMA>
cudaError_t launch5(const TiledParams<double>& p, const SkParams& sk, const TmaParams& tp,
                    unsigned grid, cudaStream_t s) {
  auto k = dgett_ws_kernel<AKF, BKF, AV, BV, TMA>;
  static unsigned long long configured = 0;
  constexpr int smem = SMEM_BYTES;
  cudaError_t e = ensure_dyn_smem(k, smem, configured);
  if (e != cudaSuccess) return e;
  k<<<grid, THREADS, smem, s>>>(p, sk, tp);
  return cudaGetLastError();
}

template <bool AKF, bool BKF>
cudaError_t launch2(const TiledParams<double>& p, const SkParams& sk, const TmaParams* tp,
                    unsigned grid, bool av, bool bv, cudaStream_t s) {
  if (tp) return launch5<AKF, BKF, false, false, true>(p, sk, *tp, grid, s);
  static const TmaParams none{};
  if (av && bv) return launch5<AKF, BKF, true, true, false>(p, sk, none, grid, s);
  if (av) return launch5<AKF, BKF, true, false, false>(p, sk, none, grid, s);
  if (bv) return launch5<AKF, BKF, false, true, false>(p, sk, none, grid, s);
  return launch5<AKF, BKF, false, false, false>(p, sk, none, grid, s);
}

}  // namespace ws

int dgett_ws_tiles_k(int K) { return (K + ws::BK - 1) / ws::BK; }

cudaError_t launch_dgett_ws(const TiledParams<double>& p, const SkParams& sk, const TmaParams* tp,
                            bool a_kf, bool b_kf, bool a_vec, bool b_vec, cudaStream_t s) {
  const unsigned grid = sk.enabled ? (unsigned)sk.grid
                                   : (unsigned)(p.tiles_m * p.tiles_n * p.splits);
  cudaError_t e;
  if (a_kf && b_kf) e = ws::launch2<true, true>(p, sk, tp, grid, a_vec, b_vec, s);
  else if (a_kf) e = ws::launch2<true, false>(p, sk, tp, grid, a_vec, b_vec, s);
  else if (b_kf) e = ws::launch2<false, true>(p, sk, tp, grid, a_vec, b_vec, s);
  else e = ws::launch2<false, false>(p, sk, tp, grid, a_vec, b_vec, s);
  if (e != cudaSuccess || p.splits == 1) return e;
  return launch_splitk_reduce<double>(p, s);
}

}  // namespace gett
