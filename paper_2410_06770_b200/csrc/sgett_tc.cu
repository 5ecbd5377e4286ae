// SGETT on the 5th-generation tensor cores: 3xTF32 with tcgen05.mma + TMEM.
//
// Replaces the fp32 hot loop (kernel.py:48-78 for sgett) for contractions big
// enough to tile.  Per 128x128 output tile and k-block of 16:
//   * 128 threads gather the A' (M x K) and B' (N x K) tiles straight from the
//     strided views with cp.async (row offsets from the planner's groups, k
//     offsets from a precomputed per-k table; 16-byte copies where the
//     planner proved 4-k contiguity) into the UMMA K-major no-swizzle layout
//     (8-row x 16-byte core matrices, LBO 128 B between k-chunks, SBO 512 B
//     between 8-row groups).  GETT_TC_STAGES-1 k-blocks are in flight, which
//     is what a latency-bound strided gather needs (SGETT c5 is HBM-bound);
//   * when a k-block lands, each thread splits its own elements in place:
//     hi = rna_tf32(x) (overwrites x), lo = x - hi (exact in fp32) into the lo
//     tile, then fence.proxy.async publishes both to the tensor core;
//   * one thread issues, per UMMA_K = 8 step, tcgen05.mma.kind::tf32 for
//     lo*hi, hi*lo, hi*hi into one fp32 accumulator in TMEM (128 lanes x 128
//     columns); tcgen05.commit frees the smem stage through an mbarrier;
//   * epilogue: tcgen05.ld 32x32b (thread = row), C += acc through the C
//     offset tables, or the split-K partial into the workspace.
// Accuracy: 3xTF32 products are within ~2^-22 relative, fp32 accumulation in
// TMEM; checked against the fp64 oracle and the reference (tests/).
#include <cstdint>

#include "device.cuh"
#include "kernels.hpp"

#ifndef GETT_TC_STAGES
#define GETT_TC_STAGES 2
#endif
#ifndef GETT_TC_SLACK
#define GETT_TC_SLACK 1
#endif

namespace gett {
namespace tc {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int BK = 16;
constexpr int CH = BK / 4;                     // 16-byte k-chunks per row
constexpr int STAGES = GETT_TC_STAGES;
constexpr int THREADS = 128;
constexpr int GROUP_M = 8;
constexpr int LBO = 128;                       // bytes between k-chunks
constexpr int SBO = CH * 128;                  // bytes between 8-row groups
constexpr int TILE_BYTES = 128 * BK * 4;       // one operand part (hi or lo): 8 KB
constexpr int STAGE_BYTES = 4 * TILE_BYTES;    // A hi, A lo, B hi, B lo
#ifndef GETT_TC_TCAP
#define GETT_TC_TCAP 256
#endif
constexpr int TCAP = GETT_TC_TCAP;             // outer k-table entries staged in smem
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 256 + 2 * TCAP * 8;
constexpr uint32_t TMEM_COLS = 128;

// instruction descriptor: D f32, A/B tf32, both K-major, N = 128, M = 128
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ uint32_t toff(int r, int c) {
  return (uint32_t)((r >> 3) * SBO + c * LBO + (r & 7) * 16);
}

// shared-memory matrix descriptor (sm_100: version 1 at bit 46), no swizzle
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(LBO >> 4) << 16) |
         ((uint64_t)(SBO >> 4) << 32) | (1ull << 46);
}

__device__ __forceinline__ void mbar_init(uint32_t addr, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(addr), "r"(count));
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

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(tmem),
      "l"(a), "l"(b), "r"(IDESC), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

__device__ __forceinline__ void split4(float4 x, float4& h, float4& l) {
  uint32_t t;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(x.x)); h.x = __uint_as_float(t); l.x = x.x - h.x;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(x.y)); h.y = __uint_as_float(t); l.y = x.y - h.y;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(x.z)); h.z = __uint_as_float(t); l.z = x.z - h.z;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(x.w)); h.w = __uint_as_float(t); l.w = x.w - h.w;
}

// k-group decoder for one operand: offset(k) = T[k / e_in] + (k % e_in) * s
struct KDec {
  const int64_t* T;
  int64_t s;
  FastDiv div;
};

// One operand's 128-row x BK gather with cp.async.  GKF: gmem fast along k
// (a thread owns one 16-byte k-chunk of 4 rows) else along rows (a thread
// owns one row, all chunks).  Units are (row, chunk) pairs.
template <bool GKF, bool VEC>
struct Gather {
  static constexpr int U = GKF ? 4 : CH;  // units per thread
  int64_t roff[GKF ? 4 : 1];
  bool rok[GKF ? 4 : 1];
  int chunk, row0;

  __device__ __forceinline__ int urow(int u) const { return GKF ? row0 + 32 * u : row0; }
  __device__ __forceinline__ int uchunk(int u) const { return GKF ? chunk : u; }

  __device__ __forceinline__ void setup(const GroupDev& g, int base_row, int nrows) {
    const int t = threadIdx.x;
    chunk = GKF ? (t & (CH - 1)) : 0;
    row0 = GKF ? t / CH : t;
#pragma unroll
    for (int i = 0; i < (GKF ? 4 : 1); ++i) {
      int r = base_row + row0 + 32 * i;
      rok[i] = r < nrows;
      roff[i] = rok[i] ? g.off(0, r) : 0;
    }
  }

  // k offsets of the next k-block, loaded ahead of the copies so the table
  // reads overlap (the cp.async issue would otherwise serialise on them)
  static constexpr int NKO = GKF ? (VEC ? 1 : 4) : BK;
  int64_t ko[NKO];
  int kk0, kkend;

  // k -> offset by stepping the group's (outer q, inner r) decode: one fast
  // divmod per k-block, and an outer-table read only when r wraps (the
  // table sits in shared memory when it fits)
  __device__ __forceinline__ void prep(const KDec& kd, int k0, int kend) {
    kk0 = k0;
    kkend = kend;
    const int kb = GKF ? k0 + 4 * chunk : k0;
    int q, r;
    kd.div.divmod(kb, q, r);
    int64_t t = kb < kend ? kd.T[q] : 0;
#pragma unroll
    for (int e = 0; e < NKO; ++e) {
      ko[e] = t + (int64_t)r * kd.s;
      if (++r == kd.div.d) {
        r = 0;
        ++q;
        t = (kb + e + 1 < kend) ? kd.T[q] : 0;
      }
    }
  }

  // issue the prepared k-block into the hi tile at smem address s
  __device__ __forceinline__ void issue(uint8_t* s, const float* base) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = urow(u), c = uchunk(u);
      const bool rv = rok[GKF ? u : 0];
      const int64_t ro = roff[GKF ? u : 0];
      uint8_t* dst = s + toff(r, c);
      const int k = kk0 + 4 * c;
      if (VEC) {
        if (rv && k < kkend) cp_async_16(dst, base + ro + ko[0]);
        else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int64_t o = GKF ? ko[e] : ko[4 * c + e];
          if (rv && k + e < kkend) cp_async_4(dst + 4 * e, base + ro + o);
          else *reinterpret_cast<float*>(dst + 4 * e) = 0.f;
        }
      }
    }
  }

  // split this thread's own landed elements: hi in place, lo into lo tile
  __device__ __forceinline__ void split(uint8_t* hi_s, uint8_t* lo_s) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t o = toff(urow(u), uchunk(u));
      float4 x = *reinterpret_cast<const float4*>(hi_s + o);
      float4 h, l;
      split4(x, h, l);
      *reinterpret_cast<float4*>(hi_s + o) = h;
      *reinterpret_cast<float4*>(lo_s + o) = l;
    }
  }
};

template <bool AKF, bool BKF, bool AVEC, bool BVEC>
__global__ void __launch_bounds__(THREADS, 1)
    sgett_tc_kernel(const __grid_constant__ TiledParams<float> p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);  // [STAGES] free, [1] done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + STAGES + 1);
  int64_t* ktabs = reinterpret_cast<int64_t*>(smem + STAGES * STAGE_BYTES + 256);  // [2][TCAP]
  const int tid = threadIdx.x;
  const int warp = tid >> 5;

  const int ntiles = p.tiles_m * p.tiles_n;
  const int tile = blockIdx.x % ntiles;
  const int split = blockIdx.x / ntiles;
  int tm, tn;
  {
    int per_group = GROUP_M * p.tiles_n;
    int group = tile / per_group;
    int first_m = group * GROUP_M;
    int gsize = min(p.tiles_m - first_m, GROUP_M);
    int in_group = tile % per_group;
    tm = first_m + in_group % gsize;
    tn = in_group / gsize;
  }
  const int m0 = tm * BM, n0 = tn * BN;
  const int kbeg = split * p.k_chunk;
  const int kend = min(p.K, kbeg + p.k_chunk);
  const int nkb = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;

  if (tid == 0) {
    for (int s = 0; s <= STAGES; ++s) mbar_init(smem_u32(bars + s), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  // the K group's outer offset tables, staged in shared memory when small
  const int n_outer = (p.gk.G + p.gk.e_in.d - 1) / p.gk.e_in.d;
  KDec kda{p.gk.T[0], p.gk.s_in[0], p.gk.e_in}, kdb{p.gk.T[1], p.gk.s_in[1], p.gk.e_in};
  if (n_outer <= TCAP) {
    for (int i = tid; i < n_outer; i += THREADS) {
      ktabs[i] = __ldg(p.gk.T[0] + i);
      ktabs[TCAP + i] = __ldg(p.gk.T[1] + i);
    }
    __syncthreads();
    kda.T = ktabs;
    kdb.T = ktabs + TCAP;
  }
  Gather<AKF, AVEC> ga;
  Gather<BKF, BVEC> gb;
  ga.setup(p.gm, m0, p.M);
  gb.setup(p.gn, n0, p.N);
  auto stage = [&](int s) { return smem + s * STAGE_BYTES; };

  // prefetch distance: DIST k-blocks of copies in flight; the stage being
  // refilled was read by the MMAs of k-block kb - (STAGES - DIST), issued
  // STAGES - DIST iterations earlier, so MMA latency stays off the loop
  constexpr int DIST = STAGES - GETT_TC_SLACK;
#pragma unroll 1
  for (int s = 0; s < DIST; ++s) {
    if (s < nkb) {
      ga.prep(kda, kbeg + s * BK, kend);
      gb.prep(kdb, kbeg + s * BK, kend);
      ga.issue(stage(s), p.A);
      gb.issue(stage(s) + 2 * TILE_BYTES, p.B);
    }
    cp_async_commit();
  }
  const uint32_t smem_base = smem_u32(smem);
#pragma unroll 1
  for (int kb = 0; kb < nkb; ++kb) {
    const int s = kb % STAGES;
    const int nk = kb + DIST;
    if (nk < nkb) {  // table reads for the refill, hidden behind this k-block's work
      ga.prep(kda, kbeg + nk * BK, kend);
      gb.prep(kdb, kbeg + nk * BK, kend);
    }
    cp_async_wait<DIST - 1>();
    uint8_t* st = stage(s);
#ifndef GETT_TC_NO_SPLIT
    ga.split(st, st + TILE_BYTES);
    gb.split(st + 2 * TILE_BYTES, st + 3 * TILE_BYTES);
#endif
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t sb = smem_base + s * STAGE_BYTES;
#pragma unroll
      for (int j = 0; j < BK / 8; ++j) {
        const uint64_t ah = sdesc(sb + 256 * j);
        const uint64_t al = sdesc(sb + TILE_BYTES + 256 * j);
        const uint64_t bh = sdesc(sb + 2 * TILE_BYTES + 256 * j);
        const uint64_t bl = sdesc(sb + 3 * TILE_BYTES + 256 * j);
        mma_tf32(tmem, ah, bh, (kb | j) != 0);  // first MMA of the tile overwrites D
#ifndef GETT_TC_NO_MMA
        mma_tf32(tmem, al, bh, 1);
        mma_tf32(tmem, ah, bl, 1);
#endif
      }
      commit(smem_u32(bars + s));
    }
    // refill the stage k-block kb - SLACK used, once its MMAs are done
    if (nk < nkb) {
      const int ns = nk % STAGES;
      const int prev = nk - STAGES;  // last k-block that used stage ns
      if (prev >= 0) mbar_wait(smem_u32(bars + ns), (prev / STAGES) & 1);
#ifndef GETT_TC_NO_LOAD
      ga.issue(stage(ns), p.A);
      gb.issue(stage(ns) + 2 * TILE_BYTES, p.B);
#endif
    }
    cp_async_commit();
  }
  if (tid == 0) commit(smem_u32(bars + STAGES));
  if (nkb > 0) mbar_wait(smem_u32(bars + STAGES), 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  // epilogue: thread tid owns accumulator row tid (TMEM lane = row)
  const int m = m0 + tid;
  const bool mok = m < p.M;
  const int64_t ro = (mok && p.splits == 1) ? p.gm.off(1, m) : 0;
  float* wrow = p.splits > 1 ? p.ws + ((int64_t)split * p.M + (mok ? m : 0)) * p.N : nullptr;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 16) {
    uint32_t r[16];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (!mok) continue;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int n = n0 + c0 + i;
      if (n >= p.N) break;
      const float acc = nkb > 0 ? __uint_as_float(r[i]) : -0.0f;
      if (p.splits == 1) {
        float* c = p.C + ro + p.gn.off(1, n);
        *c = epi(*c, acc, p.neg);
      } else {
        wrow[n] = acc;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

template <bool AKF, bool BKF, bool AV, bool BV>
cudaError_t launch4(const TiledParams<float>& p, cudaStream_t s) {
  auto k = sgett_tc_kernel<AKF, BKF, AV, BV>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  k<<<(unsigned)(p.tiles_m * p.tiles_n * p.splits), THREADS, SMEM_BYTES, s>>>(p);
  return cudaGetLastError();
}

template <bool AKF, bool BKF>
cudaError_t launch2(const TiledParams<float>& p, bool av, bool bv, cudaStream_t s) {
  if (av && bv) return launch4<AKF, BKF, true, true>(p, s);
  if (av) return launch4<AKF, BKF, true, false>(p, s);
  if (bv) return launch4<AKF, BKF, false, true>(p, s);
  return launch4<AKF, BKF, false, false>(p, s);
}

}  // namespace tc

cudaError_t launch_sgett_tc(const TiledParams<float>& p, bool a_kf, bool b_kf, bool a_vec, bool b_vec,
                            cudaStream_t s) {
  if (!a_kf) a_vec = false;  // vectors only along k
  if (!b_kf) b_vec = false;
  cudaError_t e;
  if (a_kf && b_kf) e = tc::launch2<true, true>(p, a_vec, b_vec, s);
  else if (a_kf) e = tc::launch2<true, false>(p, a_vec, b_vec, s);
  else if (b_kf) e = tc::launch2<false, true>(p, a_vec, b_vec, s);
  else e = tc::launch2<false, false>(p, a_vec, b_vec, s);
  if (e != cudaSuccess || p.splits == 1) return e;
  return launch_splitk_reduce<float>(p, s);
}

int tc_bm() { return tc::BM; }
int tc_bn() { return tc::BN; }
int tc_bk() { return tc::BK; }

}  // namespace gett
