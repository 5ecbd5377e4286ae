// SGETT on the 5th-generation tensor cores: 3xTF32 with tcgen05.mma + TMEM.
//
// Replaces the fp32 hot loop (kernel.py:48-78 for sgett) for contractions big
// enough to tile.  Per 128x128 output tile and k-block of 32:
//   * 128 threads gather the A' (M x K) and B' (N x K) tiles straight from the
//     strided views (row offsets from the planner's groups, k offsets from a
//     precomputed per-k table), split every value x = hi + lo with
//     hi = rna_tf32(x), lo = x - hi (exact in fp32), and store hi/lo tiles in
//     the UMMA K-major no-swizzle layout (8-row x 16-byte core matrices;
//     LBO 128 B between k-chunks, SBO 1 KB between 8-row groups);
//   * one thread issues, per UMMA_K=8 step, tcgen05.mma.kind::tf32 for
//     hi*hi, hi*lo, lo*hi into one fp32 accumulator in TMEM (128 lanes x 128
//     columns), and tcgen05.commit frees the smem stage through an mbarrier;
//   * the gathers of k-block kb+1 are in flight while the MMAs of kb run
//     (3-stage smem ring);
//   * epilogue: tcgen05.ld 32x32b (thread = row), C += acc through the C
//     offset tables, or the split-K partial into the workspace.
// Accuracy: the 3xTF32 product error is ~2^-22 relative per term, fp32
// accumulation in TMEM; checked against the fp64 oracle and the reference.
#include <cstdint>

#include "device.cuh"
#include "kernels.hpp"

namespace gett {
namespace tc {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int BK = 32;
constexpr int STAGES = 3;
constexpr int THREADS = 128;
constexpr int GROUP_M = 8;
constexpr int TILE_BYTES = 128 * BK * 4;       // one operand part (hi or lo): 16 KB
constexpr int STAGE_BYTES = 4 * TILE_BYTES;    // A hi, A lo, B hi, B lo
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024;
constexpr uint32_t TMEM_COLS = 128;

// instruction descriptor: D f32, A/B tf32, both K-major, N = 128, M = 128
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ uint32_t toff(int r, int c) {
  return (uint32_t)((r >> 3) * 1024 + c * 128 + (r & 7) * 16);
}

// shared-memory matrix descriptor (sm_100: version 1), no swizzle, K-major
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) |
         ((uint64_t)(1024u >> 4) << 32) | (1ull << 46);
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

__device__ __forceinline__ void tf32_split(float x, float& hi, float& lo) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  hi = __uint_as_float(h);
  lo = x - hi;
}

// One operand's 128-row x 32-k gather.  GKF: gmem fast along k (thread owns
// one 4-k chunk of 8 rows) else along rows (thread owns one row, all chunks).
template <bool GKF, bool VEC>
struct Gather {
  float v[8][4];
  int64_t roff[GKF ? 8 : 1];
  bool rok[GKF ? 8 : 1];
  int chunk, row0;

  __device__ __forceinline__ void setup(const GroupDev& g, int base_row, int nrows) {
    const int t = threadIdx.x;
    if (GKF) {
      chunk = t & 7;
      row0 = t >> 3;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        int r = base_row + row0 + 16 * i;
        rok[i] = r < nrows;
        roff[i] = rok[i] ? g.off(0, r) : 0;
      }
    } else {
      chunk = 0;
      row0 = t;
      int r = base_row + t;
      rok[0] = r < nrows;
      roff[0] = rok[0] ? g.off(0, r) : 0;
    }
  }

  __device__ __forceinline__ void load(const float* base, const int64_t* ktab, int k0, int kend) {
    if (GKF) {
      const int k = k0 + 4 * chunk;
      if (VEC) {
        const bool kok = k < kend;  // planner: K % 4 == 0 when VEC
        const int64_t ko = kok ? __ldg(ktab + k) : 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (kok && rok[i]) {
            float4 x = __ldg(reinterpret_cast<const float4*>(base + roff[i] + ko));
            v[i][0] = x.x; v[i][1] = x.y; v[i][2] = x.z; v[i][3] = x.w;
          } else {
            v[i][0] = v[i][1] = v[i][2] = v[i][3] = 0.f;
          }
        }
      } else {
        int64_t ko[4];
        bool kok[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          kok[e] = k + e < kend;
          ko[e] = kok[e] ? __ldg(ktab + k + e) : 0;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int e = 0; e < 4; ++e) v[i][e] = (kok[e] && rok[i]) ? __ldg(base + roff[i] + ko[e]) : 0.f;
      }
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int k = k0 + 4 * c + e;
          const bool ok = rok[0] && k < kend;
          v[c][e] = ok ? __ldg(base + roff[0] + __ldg(ktab + k)) : 0.f;
        }
    }
  }

  // split into hi/lo and store both tiles (byte offsets hi_s / lo_s in smem)
  __device__ __forceinline__ void store(uint8_t* hi_s, uint8_t* lo_s) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = GKF ? row0 + 16 * i : row0;
      const int c = GKF ? chunk : i;
      float4 h, l;
      tf32_split(v[i][0], h.x, l.x);
      tf32_split(v[i][1], h.y, l.y);
      tf32_split(v[i][2], h.z, l.z);
      tf32_split(v[i][3], h.w, l.w);
      const uint32_t o = toff(r, c);
      *reinterpret_cast<float4*>(hi_s + o) = h;
      *reinterpret_cast<float4*>(lo_s + o) = l;
    }
  }
};

template <bool AKF, bool BKF, bool AVEC, bool BVEC>
__global__ void __launch_bounds__(THREADS, 1)
    sgett_tc_kernel(const __grid_constant__ TiledParams<float> p, const int64_t* __restrict__ ktab_a,
                    const int64_t* __restrict__ ktab_b) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);  // [STAGES] free, [STAGES] done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + STAGES + 1);
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

  Gather<AKF, AVEC> ga;
  Gather<BKF, BVEC> gb;
  ga.setup(p.gm, m0, p.M);
  gb.setup(p.gn, n0, p.N);
  if (nkb > 0) {
    ga.load(p.A, ktab_a, kbeg, kend);
    gb.load(p.B, ktab_b, kbeg, kend);
  }
  const uint32_t smem_base = smem_u32(smem);
  for (int kb = 0; kb < nkb; ++kb) {
    const int s = kb % STAGES;
    const int use = kb / STAGES;
    if (use > 0) mbar_wait(smem_u32(bars + s), (use - 1) & 1);
    uint8_t* st = smem + s * STAGE_BYTES;
    ga.store(st, st + TILE_BYTES);
    gb.store(st + 2 * TILE_BYTES, st + 3 * TILE_BYTES);
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
        mma_tf32(tmem, al, bh, (kb | j) != 0);
        mma_tf32(tmem, ah, bl, 1);
        mma_tf32(tmem, ah, bh, 1);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(bars + s))
                   : "memory");
    }
    if (kb + 1 < nkb) {
      ga.load(p.A, ktab_a, kbeg + (kb + 1) * BK, kend);
      gb.load(p.B, ktab_b, kbeg + (kb + 1) * BK, kend);
    }
  }
  if (tid == 0) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bars + STAGES))
                 : "memory");
  }
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
        *c = *c + acc;
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
cudaError_t launch4(const TiledParams<float>& p, const int64_t* ka, const int64_t* kb, cudaStream_t s) {
  auto k = sgett_tc_kernel<AKF, BKF, AV, BV>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  k<<<(unsigned)(p.tiles_m * p.tiles_n * p.splits), THREADS, SMEM_BYTES, s>>>(p, ka, kb);
  return cudaGetLastError();
}

template <bool AKF, bool BKF>
cudaError_t launch2(const TiledParams<float>& p, const int64_t* ka, const int64_t* kb, bool av, bool bv,
                    cudaStream_t s) {
  if (av && bv) return launch4<AKF, BKF, true, true>(p, ka, kb, s);
  if (av) return launch4<AKF, BKF, true, false>(p, ka, kb, s);
  if (bv) return launch4<AKF, BKF, false, true>(p, ka, kb, s);
  return launch4<AKF, BKF, false, false>(p, ka, kb, s);
}

}  // namespace tc

cudaError_t launch_sgett_tc(const TiledParams<float>& p, const int64_t* ktab_a, const int64_t* ktab_b,
                            bool a_kf, bool b_kf, bool a_vec, bool b_vec, cudaStream_t s) {
  if (!a_kf) a_vec = false;  // vectors only along k
  if (!b_kf) b_vec = false;
  cudaError_t e;
  if (a_kf && b_kf) e = tc::launch2<true, true>(p, ktab_a, ktab_b, a_vec, b_vec, s);
  else if (a_kf) e = tc::launch2<true, false>(p, ktab_a, ktab_b, a_vec, b_vec, s);
  else if (b_kf) e = tc::launch2<false, true>(p, ktab_a, ktab_b, a_vec, b_vec, s);
  else e = tc::launch2<false, false>(p, ktab_a, ktab_b, a_vec, b_vec, s);
  if (e != cudaSuccess || p.splits == 1) return e;
  return launch_splitk_reduce<float>(p, s);
}

int tc_bm() { return tc::BM; }
int tc_bn() { return tc::BN; }
int tc_bk() { return tc::BK; }

}  // namespace gett
