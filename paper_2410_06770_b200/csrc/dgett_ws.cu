// DGETT, warp-specialised: a producer warpgroup gathers the strided A'/B'
// tiles with cp.async into a 3-stage shared-memory ring (mbarrier full/empty
// handshakes, no block-wide barrier in the main loop); two consumer
// warpgroups run only shared-memory fragment loads + FP64 DMMA
// (mma.sync m8n8k4 -> DMMA.8x8x4) and the fused C += acc epilogue through the
// C offset tables.  setmaxnreg moves registers from the producer warpgroup
// (56) to the consumers (208): 2 consumer + 1 producer warp per SM sub-partition.
//
// Same semantics and layouts as gett_tiled_kernel<double> (kernels.cu): the
// tile is 128 x 128, BK 32; smem layouts follow the gmem fast dimension of each
// operand ([row][k] pitch 36 or [k][row] pitch 132 doubles, conflict-free DMMA
// fragment reads); K-tail padding is A' -0.0, B' +0.0 so signed zeros match the
// sequential reference loop (kernel.py:76); split-K writes partials.
#include <cstdint>

#include "device.cuh"
#include "kernels.hpp"

namespace gett {
namespace ws {

constexpr int BM = 128, BN = 128, BK = 32, STAGES = 3, PAD = 4, GROUP_M = 8;
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

template <bool AKF, bool BKF, bool AVEC, bool BVEC>
__global__ void __launch_bounds__(THREADS, 1)
    dgett_ws_kernel(const __grid_constant__ TiledParams<double> p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* smem = reinterpret_cast<double*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + STAGES * STAGE_ELEMS * 8);
  uint64_t* empty = full + STAGES;
  int64_t* rowoff_a = reinterpret_cast<int64_t*>(smem_raw + STAGES * STAGE_ELEMS * 8 + BAR_BYTES);
  int64_t* rowoff_b = rowoff_a + 128;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
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
  const int mvalid = min(128, p.M - m0), nvalid = min(128, p.N - n0);

  // row offsets of this tile's A' rows and B' rows (one decode per row)
  for (int r = tid; r < 128; r += THREADS) {
    rowoff_a[r] = r < mvalid ? p.gm.off(0, m0 + r) : 0;
    rowoff_b[r] = r < nvalid ? p.gn.off(0, n0 + r) : 0;
  }
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(full + s), 2 * PW * 32);  // per producer lane: cp.async + plain arrival
      mbar_init(smem_u32(empty + s), CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp >= CW) {
    // ---------------- producer warpgroup ----------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PRODUCER_REGS));
    const int pw = warp - CW;
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES, u = kb / STAGES;
      if (u > 0) mbar_wait(smem_u32(empty + s), (u - 1) & 1);
      double* sa = smem + s * STAGE_ELEMS;
      double* sb = sa + OPER_ELEMS;
      const int k0 = kbeg + kb * BK;
      produce<AKF, AVEC, true>(sa, p.A, rowoff_a, mvalid, p.gk, 0, k0, kend, pw, lane);
      produce<BKF, BVEC, false>(sb, p.B, rowoff_b, nvalid, p.gk, 1, k0, kend, pw, lane);
      mbar_arrive_cpasync(smem_u32(full + s));  // fires when this lane's copies land
      mbar_arrive(smem_u32(full + s));          // publishes this lane's padding stores
    }
    cp_async_wait<0>();
    return;
  }

  // ---------------- consumer warpgroups ----------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(CONSUMER_REGS));
  const int wm0 = (warp / WARPS_N) * WM, wn0 = (warp % WARPS_N) * WN;
  double acc[MI][NJ][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = -0.0;
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

  for (int kb = 0; kb < nkb; ++kb) {
    const int s = kb % STAGES, u = kb / STAGES;
    mbar_wait(smem_u32(full + s), u & 1);
    const double* As = smem + s * STAGE_ELEMS;
    const double* Bs = As + OPER_ELEMS;
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
  }

  // epilogue: acc[i][j][e] is C'(m0+wm0+i*8+lane/4, n0+wn0+j*8+2*(lane%4)+e)
  int64_t coff[NJ * 2];
  bool cok[NJ * 2];
#pragma unroll
  for (int j = 0; j < NJ; ++j)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      int n = n0 + wn0 + j * 8 + 2 * (lane & 3) + e;
      cok[j * 2 + e] = n < p.N;
      coff[j * 2 + e] = (n < p.N) ? (p.splits == 1 ? p.gn.off(1, n) : (int64_t)n) : 0;
    }
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int m = m0 + wm0 + i * 8 + (lane >> 2);
    if (m >= p.M) continue;
    if (p.splits == 1) {
      const int64_t ro = p.gm.off(1, m);
      double cv[NJ][2];  // all loads of the row first, then the stores
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) cv[j][e] = cok[j * 2 + e] ? p.C[ro + coff[j * 2 + e]] : 0.0;
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (cok[j * 2 + e]) p.C[ro + coff[j * 2 + e]] = epi(cv[j][e], acc[i][j][e], p.neg);
    } else {
      double* w = p.ws + ((int64_t)split * p.M + m) * p.N;
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (cok[j * 2 + e]) w[coff[j * 2 + e]] = acc[i][j][e];
    }
  }
}

template <bool AKF, bool BKF, bool AV, bool BV>
cudaError_t launch4(const TiledParams<double>& p, cudaStream_t s) {
  auto k = dgett_ws_kernel<AKF, BKF, AV, BV>;
  static unsigned long long configured = 0;
  cudaError_t e = ensure_dyn_smem(k, SMEM_BYTES, configured);
  if (e != cudaSuccess) return e;
  k<<<(unsigned)(p.tiles_m * p.tiles_n * p.splits), THREADS, SMEM_BYTES, s>>>(p);
  return cudaGetLastError();
}

template <bool AKF, bool BKF>
cudaError_t launch2(const TiledParams<double>& p, bool av, bool bv, cudaStream_t s) {
  if (av && bv) return launch4<AKF, BKF, true, true>(p, s);
  if (av) return launch4<AKF, BKF, true, false>(p, s);
  if (bv) return launch4<AKF, BKF, false, true>(p, s);
  return launch4<AKF, BKF, false, false>(p, s);
}

}  // namespace ws

cudaError_t launch_dgett_ws(const TiledParams<double>& p, bool a_kf, bool b_kf, bool a_vec,
                            bool b_vec, cudaStream_t s) {
  cudaError_t e;
  if (a_kf && b_kf) e = ws::launch2<true, true>(p, a_vec, b_vec, s);
  else if (a_kf) e = ws::launch2<true, false>(p, a_vec, b_vec, s);
  else if (b_kf) e = ws::launch2<false, true>(p, a_vec, b_vec, s);
  else e = ws::launch2<false, false>(p, a_vec, b_vec, s);
  if (e != cudaSuccess || p.splits == 1) return e;
  return launch_splitk_reduce<double>(p, s);
}

}  // namespace gett
