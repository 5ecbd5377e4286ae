// sm_100a kernels for the B200 xGETT.
//
//   gett_tiled_kernel<double>  DGETT: gathers strided M/K and K/N tiles straight
//       from HBM into shared memory (cp.async, 16 B vectors where the planner
//       proved contiguity), FP64 DMMA (mma.sync m8n8k4 -> DMMA.8x8x4; on
//       sm_100a FP64 has no tcgen05 kind and DMMA reaches the FP64 pipe peak,
//       profiles/peaks_r01.jsonl), fused epilogue C += acc through the C
//       offset tables.  Replaces the hot loop kernel.py:48-78.
//   gett_tiled_kernel<float>   SGETT: same gathers, register-tiled FFMA.
//   gett_ref_kernel            one thread per output, K in reference order,
//       unfused mul then add: bitwise equal to the reference on all data.
//   gett_serial_kernel         the literal reference loop on one thread (used
//       only when output coordinates may alias, which the reference permits).
//   gett_splitk_reduce_kernel  deterministic ordered sum of split-K partials,
//       then C += sum.
//   gett_zero_kernel           zero_view (kernel.py:111-113) on the device.
//
// Signed zeros: tiles accumulate from -0.0 and K-tail padding contributes
// (-0.0)*(+0.0) = -0.0, the additive identity, so C + acc reproduces the
// reference's sequential signed-zero outcomes.
#include <cstdio>
#include <type_traits>

#include "device.cuh"
#include "kernels.hpp"

namespace gett {
namespace tiled {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int PAD = 4;
#ifndef GETT_REDUCE_T
#define GETT_REDUCE_T 1  // transposed-partials reduce through a shared-memory tile (0: element per thread)
#endif
#ifndef GETT_GROUP_M
#define GETT_GROUP_M 8
#endif
#ifndef GETT_D_BK
#define GETT_D_BK 32
#endif
#ifndef GETT_D_STAGES
#define GETT_D_STAGES 3
#endif
#ifndef GETT_D_THREADS
#define GETT_D_THREADS 512
#endif
constexpr int GROUP_M = GETT_GROUP_M;
constexpr int ROWS = 128;  // BM == BN

// Per element type: k-block depth and pipeline stages.  f64: BK 32 x 3 stages
// (216 KB smem, halves the per-k-block barrier/issue overhead of the DMMA
// loop); f32 FFMA: BK 16 x 4 stages.
template <typename T>
struct Cfg {
  static constexpr int BK = sizeof(T) == 8 ? GETT_D_BK : 16;
  static constexpr int STAGES = sizeof(T) == 8 ? GETT_D_STAGES : 4;
  static constexpr int THREADS = sizeof(T) == 8 ? GETT_D_THREADS : 256;
  // DMMA warp grid: 8 warps -> 2 x 4 (warp tile 64 x 32); 16 warps -> 4 x 4 (32 x 32)
  static constexpr int WARPS_M = THREADS / 32 / 4;
  static constexpr int WARPS_N = 4;
  static constexpr int KF_PITCH = BK + PAD;    // [row][k] layout (f64: 36 = 4 mod 16)
  static constexpr int RF_PITCH = ROWS + PAD;  // [k][row] layout (132 = 4 mod 16)
  static constexpr int STAGE_ELEMS =
      ROWS * KF_PITCH > BK * RF_PITCH ? ROWS * KF_PITCH : BK * RF_PITCH;
};

template <typename T>
constexpr size_t smem_bytes() {
  return (size_t)Cfg<T>::STAGES * 2 * Cfg<T>::STAGE_ELEMS * sizeof(T);
}

// Loads one operand's ROWS x BK tile per stage.
//   GKF:  gmem fast along k (else along rows)
//   VEC:  16-byte copies along the fast dimension (planner-proven)
//   SKF:  smem layout [row][k] (else [k][row])
//   IS_A: K-tail pad value -0.0 (A') or +0.0 (B')
template <typename T, bool GKF, bool VEC, bool SKF, bool IS_A>
struct Loader {
  static constexpr int BK = Cfg<T>::BK;
  static constexpr int KF_PITCH = Cfg<T>::KF_PITCH;
  static constexpr int RF_PITCH = Cfg<T>::RF_PITCH;
  static constexpr int V = VEC ? (int)(16 / sizeof(T)) : 1;
  static constexpr int FAST = GKF ? BK : ROWS;        // extent of the fast dim
  static constexpr int CPL = FAST / V;                // chunks per line
  static constexpr int THREADS = Cfg<T>::THREADS;
  static constexpr int LSTEP = THREADS / CPL;         // lines per pass
  static constexpr int SLOW = GKF ? ROWS : BK;        // extent of the slow dim
  static constexpr int PER = SLOW / LSTEP;            // passes per thread
  static_assert(THREADS % CPL == 0 && SLOW % LSTEP == 0, "loader mapping");

  int fast0;                  // this thread's offset along the fast dim
  int line0;                  // first line (slow dim) of this thread
  int64_t roff[GKF ? PER : 1];
  bool rok[GKF ? PER : 1];

  __device__ __forceinline__ void setup(const GroupDev& g, int row0, int nrows) {
    const int t = threadIdx.x;
    fast0 = (t % CPL) * V;
    line0 = t / CPL;
    if (GKF) {
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        int r = row0 + line0 + i * LSTEP;
        rok[i] = r < nrows;
        roff[i] = rok[i] ? g.off(0, r) : 0;
      }
    } else {
      int r = row0 + fast0;
      rok[0] = r < nrows;
      roff[0] = rok[0] ? g.off(0, r) : 0;
    }
  }

  __device__ __forceinline__ void store_pad(T* s, int r, int k, T v) {
    if (SKF) s[r * KF_PITCH + k] = v;
    else s[k * RF_PITCH + r] = v;
  }

  __device__ __forceinline__ void copy(T* s, int r, int k, const T* src) {
    T* dst = SKF ? (s + r * KF_PITCH + k) : (s + k * RF_PITCH + r);
    if (V == 1) {
      if (sizeof(T) == 8) cp_async_8(dst, src);
      else cp_async_4(dst, src);
    } else {
      cp_async_16(dst, src);
    }
  }

  // kt: index of this operand in gk (0 = A', 1 = B')
  __device__ __forceinline__ void load(T* s, const T* base, const GroupDev& gk, int kt, int k0,
                                       int kend) {
    const T kpad = IS_A ? T(-0.0) : T(0.0);
    if (GKF) {
      int k = k0 + fast0;
      bool kok = k < kend;
      int64_t ko = kok ? gk.off(kt, k) : 0;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        int r = line0 + i * LSTEP;
        if (kok && rok[i]) {
          copy(s, r, fast0, base + roff[i] + ko);
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v) store_pad(s, r, fast0 + v, kok ? T(0) : kpad);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        int kk = line0 + i * LSTEP;
        int k = k0 + kk;
        bool kok = k < kend;
        if (kok && rok[0]) {
          copy(s, fast0, kk, base + roff[0] + gk.off(kt, k));
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v) store_pad(s, fast0 + v, kk, kok ? T(0) : kpad);
        }
      }
    }
  }
};

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void tile_coords(int tiles_m, int tiles_n, int tile, int& tm, int& tn) {
  int per_group = GROUP_M * tiles_n;
  int group = tile / per_group;
  int first_m = group * GROUP_M;
  int gsize = min(tiles_m - first_m, GROUP_M);
  int in_group = tile % per_group;
  tm = first_m + in_group % gsize;
  tn = in_group / gsize;
}

// T = double: DMMA core, warps 2 (M) x 4 (N), warp tile 64 x 32.
// T = float : FFMA core, 16 x 16 threads, thread tile 8 x 8 (rows ty*4+i,
//             64+ty*4+i; cols tx*4+j, 64+tx*4+j).
template <typename T, bool AKF, bool BKF, bool AVEC, bool BVEC>
__global__ void __launch_bounds__(Cfg<T>::THREADS, 1) gett_tiled_kernel(const __grid_constant__ TiledParams<T> p) {
  constexpr bool IS_D = sizeof(T) == 8;
  constexpr int BK = Cfg<T>::BK;
  constexpr int STAGES = Cfg<T>::STAGES;
  constexpr int KF_PITCH = Cfg<T>::KF_PITCH;
  constexpr int RF_PITCH = Cfg<T>::RF_PITCH;
  constexpr int STAGE_ELEMS = Cfg<T>::STAGE_ELEMS;
  // smem layouts: DMMA follows the gmem fast dimension; FFMA always [k][row]
  constexpr bool ASKF = IS_D ? AKF : false;
  constexpr bool BSKF = IS_D ? BKF : false;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* smem = reinterpret_cast<T*>(smem_raw);

  const int ntiles = p.tiles_m * p.tiles_n;
  const int tile = blockIdx.x % ntiles;
  const int split = blockIdx.x / ntiles;
  int tm, tn;
  tile_coords(p.tiles_m, p.tiles_n, tile, tm, tn);
  const int m0 = tm * BM, n0 = tn * BN;
  const int kbeg = split * p.k_chunk;
  const int kend = min(p.K, kbeg + p.k_chunk);
  const int nkb = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;

  Loader<T, AKF, AVEC, ASKF, true> la;
  Loader<T, BKF, BVEC, BSKF, false> lb;
  la.setup(p.gm, m0, p.M);
  lb.setup(p.gn, n0, p.N);

  auto sA = [&](int st) { return smem + (size_t)st * 2 * STAGE_ELEMS; };
  auto sB = [&](int st) { return smem + (size_t)st * 2 * STAGE_ELEMS + STAGE_ELEMS; };

#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < nkb) {
      la.load(sA(st), p.A, p.gk, 0, kbeg + st * BK, kend);
      lb.load(sB(st), p.B, p.gk, 1, kbeg + st * BK, kend);
    }
    cp_async_commit();
  }

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;

  if constexpr (IS_D) {
    constexpr int WM = BM / Cfg<T>::WARPS_M, WN = BN / Cfg<T>::WARPS_N;
    constexpr int MI = WM / 8, NJ = WN / 8;
    const int wm0 = (warp / Cfg<T>::WARPS_N) * WM;
    const int wn0 = (warp % Cfg<T>::WARPS_N) * WN;
    double acc[MI][NJ][2];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[i][j][0] = acc[i][j][1] = -0.0;

    // fragment offsets within a stage (k-step 0); k-step ks adds 4*ks along k
    int aoff[MI], boff[NJ];
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      int r = wm0 + i * 8 + (lane >> 2);
      aoff[i] = ASKF ? r * KF_PITCH + (lane & 3) : (lane & 3) * RF_PITCH + r;
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      int c = wn0 + j * 8 + (lane >> 2);
      boff[j] = BSKF ? c * KF_PITCH + (lane & 3) : (lane & 3) * RF_PITCH + c;
    }
    constexpr int AKS = ASKF ? 4 : 4 * RF_PITCH;  // k-step stride in smem
    constexpr int BKS = BSKF ? 4 : 4 * RF_PITCH;

    for (int kb = 0; kb < nkb; ++kb) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      const double* As = sA(kb % STAGES);
      const double* Bs = sB(kb % STAGES);
      // register double buffer: fragments of k-step ks+1 load under the DMMAs of ks
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
        if (ks == 0) {
          // issue the next stage's gathers while the first k-step's DMMAs drain
          int nk = kb + STAGES - 1;
          if (nk < nkb) {
            la.load(sA(nk % STAGES), p.A, p.gk, 0, kbeg + nk * BK, kend);
            lb.load(sB(nk % STAGES), p.B, p.gk, 1, kbeg + nk * BK, kend);
          }
          cp_async_commit();
        }
      }
    }
    cp_async_wait<0>();

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
    if (p.splits == 1) {
      // all C loads first (many in flight), then the stores: C += acc
      int64_t ro[MI];
      bool rok[MI];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        int m = m0 + wm0 + i * 8 + (lane >> 2);
        rok[i] = m < p.M;
        ro[i] = rok[i] ? p.gm.off(1, m) : 0;
      }
      constexpr int IH = 1;  // rows per batch (bounds live registers)
#pragma unroll
      for (int i0 = 0; i0 < MI; i0 += IH) {
        double cv[IH][NJ][2];
#pragma unroll
        for (int i = 0; i < IH; ++i)
#pragma unroll
          for (int j = 0; j < NJ; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              cv[i][j][e] = (rok[i0 + i] && cok[j * 2 + e]) ? p.C[ro[i0 + i] + coff[j * 2 + e]] : 0.0;
#pragma unroll
        for (int i = 0; i < IH; ++i)
#pragma unroll
          for (int j = 0; j < NJ; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              if (rok[i0 + i] && cok[j * 2 + e])
                p.C[ro[i0 + i] + coff[j * 2 + e]] = epi(cv[i][j][e], acc[i0 + i][j][e], p.neg);
      }
    }
#pragma unroll
    for (int i = 0; i < MI; ++i) {
      int m = m0 + wm0 + i * 8 + (lane >> 2);
      if (m >= p.M) continue;
      if (p.splits == 1) {
        continue;
      } else {
        double* w = p.ws + ((int64_t)split * p.M + m) * p.N;
#pragma unroll
        for (int j = 0; j < NJ; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            if (cok[j * 2 + e]) w[coff[j * 2 + e]] = acc[i][j][e];
      }
    }
  } else {
    const int tx = threadIdx.x & 15;
    const int ty = threadIdx.x >> 4;
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = -0.0f;

    for (int kb = 0; kb < nkb; ++kb) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      {
        int nk = kb + STAGES - 1;
        if (nk < nkb) {
          la.load(sA(nk % STAGES), p.A, p.gk, 0, kbeg + nk * BK, kend);
          lb.load(sB(nk % STAGES), p.B, p.gk, 1, kbeg + nk * BK, kend);
        }
        cp_async_commit();
      }
      const float* As = sA(kb % STAGES);
      const float* Bs = sB(kb % STAGES);
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        float4 a0 = *reinterpret_cast<const float4*>(As + kk * RF_PITCH + ty * 4);
        float4 a1 = *reinterpret_cast<const float4*>(As + kk * RF_PITCH + 64 + ty * 4);
        float4 b0 = *reinterpret_cast<const float4*>(Bs + kk * RF_PITCH + tx * 4);
        float4 b1 = *reinterpret_cast<const float4*>(Bs + kk * RF_PITCH + 64 + tx * 4);
        float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
    }
    cp_async_wait<0>();

    int64_t coff[8];
    bool cok[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      cok[j] = n < p.N;
      coff[j] = (n < p.N) ? (p.splits == 1 ? p.gn.off(1, n) : (int64_t)n) : 0;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
      if (m >= p.M) continue;
      if (p.splits == 1) {
        int64_t ro = p.gm.off(1, m);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (cok[j]) {
            float* c = p.C + ro + coff[j];
            *c = epi(*c, acc[i][j], p.neg);
          }
      } else {
        float* w = p.ws + ((int64_t)split * p.M + m) * p.N;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (cok[j]) w[coff[j]] = acc[i][j];
      }
    }
  }
}

}  // namespace tiled

// ---------------------------------------------------------------------------

__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }

template <typename T>
__global__ void __launch_bounds__(256) gett_ref_kernel(const __grid_constant__ RefParams<T> p) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)p.M * p.N) return;
  int32_t n = (int32_t)(idx % p.N);
  int32_t m = (int32_t)(idx / p.N);
  int64_t fa, ca, fb, cb;
  p.gm.off2(m, fa, ca);
  p.gn.off2(n, fb, cb);
  T* c = p.C + ca + cb;
  T acc = *c;
  const T* A = p.A + fa;
  const T* B = p.B + fb;
  for (int32_t q = 0; q < p.k_outer; ++q) {
    const T* a = A + __ldg(p.kta + q);
    const T* b = B + __ldg(p.ktb + q);
    for (int32_t r = 0; r < p.k_inner; ++r)
      acc = add_rn(acc, mul_rn(__ldg(a + (int64_t)r * p.k_sa), __ldg(b + (int64_t)r * p.k_sb)));
  }
  *c = acc;
}

// Few outputs, long K (c1: 960 outputs x K 1280): one warp per output, lanes
// stride the K range (reference order decode), a fixed xor-butterfly sum, then
// C + acc.  Accumulators start at -0.0 like the tiled kernels; the order is
// fixed, so results are deterministic (not bitwise equal to the sequential
// loop except on exactly representable data).
constexpr int DOT_TAB = 1024;  // outer K entries staged in smem per block

template <typename T>
__global__ void __launch_bounds__(256) gett_dot_kernel(const __grid_constant__ RefParams<T> p) {
  __shared__ int64_t ta_s[DOT_TAB], tb_s[DOT_TAB];
  const int64_t* kta = p.kta;
  const int64_t* ktb = p.ktb;
  if (p.k_outer <= DOT_TAB) {  // block-uniform: stage the outer K tables once
    for (int i = threadIdx.x; i < p.k_outer; i += blockDim.x) {
      ta_s[i] = __ldg(p.kta + i);
      tb_s[i] = __ldg(p.ktb + i);
    }
    __syncthreads();
    kta = ta_s;
    ktb = tb_s;
  }
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= (int64_t)p.M * p.N) return;  // warp-uniform
  const int32_t n = (int32_t)(w % p.N);
  const int32_t m = (int32_t)(w / p.N);
  int64_t fa, ca, fb, cb;
  p.gm.off2(m, fa, ca);
  p.gn.off2(n, fb, cb);
  const T* A = p.A + fa;
  const T* B = p.B + fb;
  T acc = T(-0.0);
  const int32_t K = p.k_inner * p.k_outer;
  // independent iterations (one fast division each), so the loads of several
  // k steps are in flight at once
#pragma unroll 4
  for (int32_t k = lane; k < K; k += 32) {
    int32_t q, r;
    p.kdiv.divmod(k, q, r);
    acc = add_rn(acc, mul_rn(__ldg(A + kta[q] + (int64_t)r * p.k_sa),
                             __ldg(B + ktb[q] + (int64_t)r * p.k_sb)));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc = add_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
  if (lane == 0) {
    T* c = p.C + ca + cb;
    *c = add_rn(*c, acc);
  }
}

// Few outputs, long K: block = one staged row (of A' or B') x 8 streamed rows,
// one warp per output.  The staged row's K values are gathered once into
// shared memory in gk's order, with the streamed operand's k offsets beside
// them; lanes then walk k = lane, lane+32, ... so the streamed operand is read
// along its unit-stride inner k mode (coalesced) and the staged values without
// bank conflicts.  Per output: lane-sequential unfused sums from -0.0, a fixed
// xor butterfly, C + acc: deterministic.
template <typename T>
__global__ void __launch_bounds__(256) gett_dot_staged_kernel(const __grid_constant__ DotParams<T> p) {
  extern __shared__ __align__(16) unsigned char dsm[];
  T* sv = reinterpret_cast<T*>(dsm);                                   // [K] staged values
  int64_t* ko = reinterpret_cast<int64_t*>(dsm + ((size_t)p.K * sizeof(T) + 15) / 16 * 16);  // [K]
  const bool sa = p.stream_a != 0;
  const GroupDev& gs = sa ? p.gn : p.gm;  // staged rows
  const GroupDev& gr = sa ? p.gm : p.gn;  // streamed rows
  const T* S = sa ? p.B : p.A;
  const T* R = sa ? p.A : p.B;
  const int ts = sa ? 1 : 0, tr = sa ? 0 : 1;
  const int NR = sa ? p.M : p.N;
  const int nrb = (NR + 7) / 8;
  const int rs = blockIdx.x / nrb;
  const T* srow = S + gs.off(0, rs);
  for (int k = threadIdx.x; k < p.K; k += blockDim.x) {
    int64_t os, orr;
    p.gk.off2(k, os, orr);
    sv[k] = __ldg(srow + (ts ? orr : os));
    ko[k] = tr ? orr : os;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rr = (blockIdx.x % nrb) * 8 + warp;
  if (rr >= NR) return;  // warp-uniform
  const T* rrow = R + gr.off(0, rr);
  T acc = T(-0.0);
  int k = lane;
  // loads of 8 k steps issued before their (sequential) accumulation
  for (; k + 32 * 7 < p.K; k += 32 * 8) {
    T v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldg(rrow + ko[k + 32 * j]);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc = add_rn(acc, mul_rn(v[j], sv[k + 32 * j]));
  }
  for (; k < p.K; k += 32) acc = add_rn(acc, mul_rn(__ldg(rrow + ko[k]), sv[k]));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc = add_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
  if (lane == 0) {
    const int m = sa ? rr : rs, n = sa ? rs : rr;
    T* c = p.C + p.gm.off(1, m) + p.gn.off(1, n);
    *c = add_rn(*c, acc);
  }
}

// kernel.py:48-78 verbatim on one thread (odometer order, c read each MAC)
template <typename T>
__global__ void gett_serial_kernel(const __grid_constant__ SerialParams<T> p) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const int nf = p.num_free, nc = p.num_cont;
  const int64_t* out_inc = p.tab;
  const int64_t* src_inc = p.tab + nf;
  const int64_t* from_a = p.tab + 2 * nf;
  const int64_t* ext_free = p.tab + 3 * nf;
  const int64_t* inc_ca = p.tab + 4 * nf;
  const int64_t* inc_cb = p.tab + 4 * nf + nc;
  const int64_t* ext_cont = p.tab + 4 * nf + 2 * nc;
  int64_t cf[64], cc[64];
  for (int j = 0; j < nf; ++j) cf[j] = 0;
  for (int64_t f = 0; f < p.size_free; ++f) {
    int64_t ic = 0, ia0 = 0, ib0 = 0;
    for (int j = 0; j < nf; ++j) {
      ic += out_inc[j] * cf[j];
      if (from_a[j]) ia0 += src_inc[j] * cf[j];
      else ib0 += src_inc[j] * cf[j];
    }
    for (int k = 0; k < nc; ++k) cc[k] = 0;
    for (int64_t q = 0; q < p.size_cont; ++q) {
      int64_t ia = ia0, ib = ib0;
      for (int k = 0; k < nc; ++k) {
        ia += inc_ca[k] * cc[k];
        ib += inc_cb[k] * cc[k];
      }
      volatile T* c = p.C + ic;
      *c = add_rn(*c, mul_rn(p.A[ia], p.B[ib]));
      for (int k = 0; k < nc; ++k) {
        cc[k] = (cc[k] + 1) % ext_cont[k];
        if (cc[k] != 0) break;
      }
    }
    for (int j = 0; j < nf; ++j) {
      cf[j] = (cf[j] + 1) % ext_free[j];
      if (cf[j] != 0) break;
    }
  }
}

// Complex (cgett / zgett, kernel.py:187-200): R is the real type, buffers are
// interleaved (re, im) pairs and all offsets are in complex elements.  The
// product is numba's complex multiply, unfused: re = ar*br - ai*bi,
// im = ar*bi + ai*br, then c = c + prod componentwise, K in reference order.
template <typename R>
__device__ __forceinline__ void cmac(R& cr, R& ci, const R* a, const R* b) {
  const R ar = __ldg(a), ai = __ldg(a + 1), br = __ldg(b), bi = __ldg(b + 1);
  const R pr = add_rn(mul_rn(ar, br), -mul_rn(ai, bi));
  const R pi = add_rn(mul_rn(ar, bi), mul_rn(ai, br));
  cr = add_rn(cr, pr);
  ci = add_rn(ci, pi);
}

template <typename R>
__global__ void __launch_bounds__(256) gett_ref_kernel_c(const __grid_constant__ RefParams<R> p) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)p.M * p.N) return;
  int32_t n = (int32_t)(idx % p.N);
  int32_t m = (int32_t)(idx / p.N);
  int64_t fa, ca, fb, cb;
  p.gm.off2(m, fa, ca);
  p.gn.off2(n, fb, cb);
  R* c = p.C + 2 * (ca + cb);
  R cr = c[0], ci = c[1];
  const R* A = p.A + 2 * fa;
  const R* B = p.B + 2 * fb;
  for (int32_t q = 0; q < p.k_outer; ++q) {
    const R* a = A + 2 * __ldg(p.kta + q);
    const R* b = B + 2 * __ldg(p.ktb + q);
    for (int32_t r = 0; r < p.k_inner; ++r) cmac(cr, ci, a + 2 * r * p.k_sa, b + 2 * r * p.k_sb);
  }
  c[0] = cr;
  c[1] = ci;
}

template <typename R>
__global__ void gett_serial_kernel_c(const __grid_constant__ SerialParams<R> p) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const int nf = p.num_free, nc = p.num_cont;
  const int64_t* out_inc = p.tab;
  const int64_t* src_inc = p.tab + nf;
  const int64_t* from_a = p.tab + 2 * nf;
  const int64_t* ext_free = p.tab + 3 * nf;
  const int64_t* inc_ca = p.tab + 4 * nf;
  const int64_t* inc_cb = p.tab + 4 * nf + nc;
  const int64_t* ext_cont = p.tab + 4 * nf + 2 * nc;
  int64_t cf[64], cc[64];
  for (int j = 0; j < nf; ++j) cf[j] = 0;
  for (int64_t f = 0; f < p.size_free; ++f) {
    int64_t ic = 0, ia0 = 0, ib0 = 0;
    for (int j = 0; j < nf; ++j) {
      ic += out_inc[j] * cf[j];
      if (from_a[j]) ia0 += src_inc[j] * cf[j];
      else ib0 += src_inc[j] * cf[j];
    }
    for (int k = 0; k < nc; ++k) cc[k] = 0;
    for (int64_t q = 0; q < p.size_cont; ++q) {
      int64_t ia = ia0, ib = ib0;
      for (int k = 0; k < nc; ++k) {
        ia += inc_ca[k] * cc[k];
        ib += inc_cb[k] * cc[k];
      }
      volatile R* c = p.C + 2 * ic;
      R cr = c[0], ci = c[1];
      const R ar = p.A[2 * ia], ai = p.A[2 * ia + 1], br = p.B[2 * ib], bi = p.B[2 * ib + 1];
      cr = add_rn(cr, add_rn(mul_rn(ar, br), -mul_rn(ai, bi)));
      ci = add_rn(ci, add_rn(mul_rn(ar, bi), mul_rn(ai, br)));
      c[0] = cr;
      c[1] = ci;
      for (int k = 0; k < nc; ++k) {
        cc[k] = (cc[k] + 1) % ext_cont[k];
        if (cc[k] != 0) break;
      }
    }
    for (int j = 0; j < nf; ++j) {
      cf[j] = (cf[j] + 1) % ext_free[j];
      if (cf[j] != 0) break;
    }
  }
}

// C[m, n] += sum_s ws[s][m][n], s ascending, sum started at -0.0
template <typename T>
__global__ void __launch_bounds__(256) gett_splitk_reduce_kernel(const __grid_constant__ TiledParams<T> p) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t mn = (int64_t)p.M * p.N;
  if (idx >= mn) return;
  int32_t n, m;
  if (p.ws_t) {  // [splits][N][M]: consecutive threads read consecutive m
    m = (int32_t)(idx % p.M);
    n = (int32_t)(idx / p.M);
  } else {
    n = (int32_t)(idx % p.N);
    m = (int32_t)(idx / p.N);
  }
  // launched as a programmatic dependent of the split-K kernel: wait for its
  // partials (no-op for an ordinary launch)
  // C's element (offset tables, then its value) does not depend on the
  // partials: fetched first, so its two round trips overlap the partials'
  T* c = p.C + p.gm.off(1, m) + p.gn.off(1, n);
  // (safe before the wait: the split-K kernel triggers this grid only after its
  // own wait for whatever preceded it, and it never writes C)
  const T c0 = *c;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // the slices' partials in a fixed order; loads batched 8 at a time so their
  // latencies overlap
  T s = T(-0.0);
  int sp = 0;
  for (; sp + 8 <= p.splits; sp += 8) {
    T v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldcg(p.ws + (sp + j) * mn + idx);
#pragma unroll
    for (int j = 0; j < 8; ++j) s = s + v[j];
  }
  for (; sp < p.splits; ++sp) s = s + __ldcg(p.ws + sp * mn + idx);
  *c = epi(c0, s, p.neg);
}

// The same sum for transposed partials [splits][N][M] (the SGETT tcgen05
// kernel's layout) when C's smallest stride is in N (the planner's choice):
// a 32 m x 8 n tile per block, partials read m-fastest, staged through shared
// memory, C read and written n-fastest (8 consecutive n: one 32 B sector per
// row for fp32 instead of one per element).  Same order, same bits.
template <typename T>
__global__ void __launch_bounds__(256) gett_splitk_reduce_t_kernel(const __grid_constant__ TiledParams<T> p) {
  __shared__ T tile[8][33];
  const int t = threadIdx.x;
  const int n0 = blockIdx.x * 8, m0 = blockIdx.y * 32;
  const int64_t mn = (int64_t)p.M * p.N;
  const int mw = m0 + t / 8, nw = n0 + t % 8;
  const bool okw = mw < p.M && nw < p.N;
  T* c = okw ? p.C + p.gm.off(1, mw) + p.gn.off(1, nw) : nullptr;
  // C does not depend on the partials: fetched before the wait, so its round
  // trip overlaps the split-K kernel's tail (that kernel never writes C, and it
  // triggers this grid only after its own wait for whatever preceded it).  A
  // programmatic dependent of this grid may be scheduled right away: it waits
  // for this grid's completion itself.
  const T c0 = okw ? *c : T(0);
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int mr = m0 + t % 32, nr = n0 + t / 32;
  if (mr < p.M && nr < p.N) {
    const int64_t idx = (int64_t)nr * p.M + mr;
    T s = T(-0.0);
    // every partial of a chunk of 32 splits in flight before the in-order sum
    // (one L2 round trip for c5's 24 splits instead of three)
    for (int sp0 = 0; sp0 < p.splits; sp0 += 32) {
      T v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = sp0 + j < p.splits ? __ldcg(p.ws + (sp0 + j) * mn + idx) : T(0);
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (sp0 + j < p.splits) s = s + v[j];
    }
    tile[t / 32][t % 32] = s;
  }
  __syncthreads();
  if (okw) *c = epi(c0, tile[t % 8][t / 8], p.neg);
}

template <typename T>
__global__ void __launch_bounds__(256) gett_zero_kernel(T* base, const __grid_constant__ GroupDev g) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.G; i += stride)
    base[g.off(0, (int32_t)i)] = T(0);
}

template <typename T>
__global__ void __launch_bounds__(256) gett_accum_view_kernel(const __grid_constant__ AccumParams<T> p) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.g.G; i += stride) {
    const int64_t o = p.g.off(0, (int32_t)i);
    T s = __ldcv(p.P[0] + o);  // volatile: peer memory written by another device's kernel
    for (int j = 1; j < p.n; ++j) s = s + __ldcv(p.P[j] + o);
    p.C[o] = p.C[o] + s;
  }
}

template <typename E, bool SMALL>
__global__ void __launch_bounds__(256) gett_pack_kernel(const __grid_constant__ PackParams p) {
  const E* src = static_cast<const E*>(p.src);
  E* dst = static_cast<E*>(p.dst);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.n; i += stride) {
    int64_t off = 0;
    if (SMALL) {
      int32_t rem = (int32_t)i;
      for (int d = 0; d < p.rank; ++d) {
        int32_t q, r;
        p.div[d].divmod(rem, q, r);
        off += (int64_t)r * p.inc[d];
        rem = q;
      }
    } else {
      int64_t rem = i;
      for (int d = 0; d < p.rank; ++d) {
        const int64_t q = rem / p.ext[d];
        off += (rem - q * p.ext[d]) * p.inc[d];
        rem = q;
      }
    }
    dst[i] = src[off];
  }
}

// ---------------------------------------------------------------------------
// launchers

namespace {
template <typename T, bool AKF, bool BKF, bool AV, bool BV>
cudaError_t launch_t(const TiledParams<T>& p, cudaStream_t s) {
  auto k = tiled::gett_tiled_kernel<T, AKF, BKF, AV, BV>;
  constexpr size_t smem = tiled::smem_bytes<T>();
  static unsigned long long configured = 0;
  cudaError_t e = ensure_dyn_smem(k, (int)smem, configured);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)(p.tiles_m * p.tiles_n * p.splits));
  k<<<grid, tiled::Cfg<T>::THREADS, smem, s>>>(p);
  return cudaGetLastError();
}

template <typename T, bool AKF, bool BKF>
cudaError_t launch_v(const TiledParams<T>& p, bool av, bool bv, cudaStream_t s) {
  if (av && bv) return launch_t<T, AKF, BKF, true, true>(p, s);
  if (av) return launch_t<T, AKF, BKF, true, false>(p, s);
  if (bv) return launch_t<T, AKF, BKF, false, true>(p, s);
  return launch_t<T, AKF, BKF, false, false>(p, s);
}
}  // namespace

template <typename T>
cudaError_t launch_tiled(const TiledParams<T>& p, bool a_kf, bool b_kf, bool a_vec, bool b_vec,
                         cudaStream_t s) {
  if (sizeof(T) == 4) {  // FFMA core keeps [k][row] smem: k-fast gathers are scalar
    if (a_kf) a_vec = false;
    if (b_kf) b_vec = false;
  }
  cudaError_t e;
  if (a_kf && b_kf) e = launch_v<T, true, true>(p, a_vec, b_vec, s);
  else if (a_kf) e = launch_v<T, true, false>(p, a_vec, b_vec, s);
  else if (b_kf) e = launch_v<T, false, true>(p, a_vec, b_vec, s);
  else e = launch_v<T, false, false>(p, a_vec, b_vec, s);
  if (e != cudaSuccess || p.splits == 1) return e;
  return launch_splitk_reduce<T>(p, s);
}

template <typename T>
cudaError_t launch_splitk_reduce(const TiledParams<T>& p, cudaStream_t s) {
  // programmatic dependent launch: the reduce grid is scheduled while the
  // split-K kernel drains and waits on griddepcontrol.wait for its partials
  int64_t mn = (int64_t)p.M * p.N;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((mn + 255) / 256));
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_launch_pdl ? 1 : 0;
  const int64_t mt = (p.M + 31) / 32;
  if (GETT_REDUCE_T && p.ws_t && mt <= 65535) {
    cfg.gridDim = dim3((unsigned)((p.N + 7) / 8), (unsigned)mt);
    return cudaLaunchKernelEx(&cfg, gett_splitk_reduce_t_kernel<T>, p);
  }
  return cudaLaunchKernelEx(&cfg, gett_splitk_reduce_kernel<T>, p);
}

template <typename T>
cudaError_t launch_ref(const RefParams<T>& p, cudaStream_t s) {
  int64_t n = (int64_t)p.M * p.N;
  gett_ref_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_dot(const RefParams<T>& p, cudaStream_t s) {
  const int64_t threads = (int64_t)p.M * p.N * 32;
  gett_dot_kernel<T><<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(p);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_dot_staged(const DotParams<T>& p, cudaStream_t s) {
  const int NR = p.stream_a ? p.M : p.N, NS = p.stream_a ? p.N : p.M;
  const size_t smem = ((size_t)p.K * sizeof(T) + 15) / 16 * 16 + (size_t)p.K * sizeof(int64_t);
  auto k = gett_dot_staged_kernel<T>;
  if (smem > 48 * 1024) {
    static unsigned long long configured = 0;
    cudaError_t e = ensure_dyn_smem(k, (int)smem, configured);
    if (e != cudaSuccess) return e;
  }
  k<<<(unsigned)(NS * ((NR + 7) / 8)), 256, smem, s>>>(p);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_serial(const SerialParams<T>& p, cudaStream_t s) {
  gett_serial_kernel<T><<<1, 1, 0, s>>>(p);
  return cudaGetLastError();
}

template <typename R>
cudaError_t launch_ref_c(const RefParams<R>& p, cudaStream_t s) {
  int64_t n = (int64_t)p.M * p.N;
  gett_ref_kernel_c<R><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p);
  return cudaGetLastError();
}

template <typename R>
cudaError_t launch_serial_c(const SerialParams<R>& p, cudaStream_t s) {
  gett_serial_kernel_c<R><<<1, 1, 0, s>>>(p);
  return cudaGetLastError();
}
template cudaError_t launch_ref_c<double>(const RefParams<double>&, cudaStream_t);
template cudaError_t launch_ref_c<float>(const RefParams<float>&, cudaStream_t);
template cudaError_t launch_serial_c<double>(const SerialParams<double>&, cudaStream_t);
template cudaError_t launch_serial_c<float>(const SerialParams<float>&, cudaStream_t);

// Real embedding of a complex operand: one thread per element, the modes
// walked fastest first so the two pair stores of neighbouring threads are
// contiguous.
template <typename R>
__global__ void __launch_bounds__(256) gett_expand_complex_kernel(const __grid_constant__ ExpandParams<R> p) {
  using V2 = typename std::conditional<sizeof(R) == 8, double2, float2>::type;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = i, src = 0, dst = 0;
    for (int d = 0; d < p.n; ++d) {
      const int64_t e = p.ext[d], x = rem % e;
      rem /= e;
      src += x * p.inc[d];
      dst += x * p.dst_st[d];
    }
    const R re = p.src[2 * src], im = p.src[2 * src + 1];
    V2 v0, v1;
    v0.x = re; v0.y = im;
    v1.x = -im; v1.y = re;
    *reinterpret_cast<V2*>(p.dst + dst) = v0;
    *reinterpret_cast<V2*>(p.dst + dst + p.q) = v1;
  }
}

template <typename R>
cudaError_t launch_expand_complex(const ExpandParams<R>& p, cudaStream_t s) {
  int64_t blocks = (p.total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  gett_expand_complex_kernel<R><<<(unsigned)blocks, 256, 0, s>>>(p);
  return cudaGetLastError();
}
template cudaError_t launch_expand_complex<float>(const ExpandParams<float>&, cudaStream_t);
template cudaError_t launch_expand_complex<double>(const ExpandParams<double>&, cudaStream_t);

template <typename T>
cudaError_t launch_zero(T* base, const GroupDev& g, cudaStream_t s) {
  int64_t blocks = (g.G + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  gett_zero_kernel<T><<<(unsigned)blocks, 256, 0, s>>>(base, g);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_accum(const AccumParams<T>& p, cudaStream_t s) {
  if (p.n < 1) return cudaSuccess;
  int64_t blocks = (p.g.G + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  gett_accum_view_kernel<T><<<(unsigned)blocks, 256, 0, s>>>(p);
  return cudaGetLastError();
}
template cudaError_t launch_accum<double>(const AccumParams<double>&, cudaStream_t);
template cudaError_t launch_accum<float>(const AccumParams<float>&, cudaStream_t);

cudaError_t launch_pack(const PackParams& p, int elem_bytes, cudaStream_t s) {
  if (p.n <= 0) return cudaSuccess;
  int64_t blocks = (p.n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  const bool small = p.n < (1LL << 31);
  switch (elem_bytes) {
    case 4:
      if (small) gett_pack_kernel<uint32_t, true><<<(unsigned)blocks, 256, 0, s>>>(p);
      else gett_pack_kernel<uint32_t, false><<<(unsigned)blocks, 256, 0, s>>>(p);
      break;
    case 8:
      if (small) gett_pack_kernel<uint64_t, true><<<(unsigned)blocks, 256, 0, s>>>(p);
      else gett_pack_kernel<uint64_t, false><<<(unsigned)blocks, 256, 0, s>>>(p);
      break;
    case 16:
      if (small) gett_pack_kernel<ulonglong2, true><<<(unsigned)blocks, 256, 0, s>>>(p);
      else gett_pack_kernel<ulonglong2, false><<<(unsigned)blocks, 256, 0, s>>>(p);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

int tiled_bm() { return tiled::BM; }
int tiled_bn() { return tiled::BN; }
int tiled_bk(int elt_bytes) { return elt_bytes == 8 ? tiled::Cfg<double>::BK : tiled::Cfg<float>::BK; }

template cudaError_t launch_tiled<double>(const TiledParams<double>&, bool, bool, bool, bool, cudaStream_t);
template cudaError_t launch_tiled<float>(const TiledParams<float>&, bool, bool, bool, bool, cudaStream_t);
template cudaError_t launch_splitk_reduce<double>(const TiledParams<double>&, cudaStream_t);
template cudaError_t launch_splitk_reduce<float>(const TiledParams<float>&, cudaStream_t);
template cudaError_t launch_ref<double>(const RefParams<double>&, cudaStream_t);
template cudaError_t launch_ref<float>(const RefParams<float>&, cudaStream_t);
template cudaError_t launch_dot<double>(const RefParams<double>&, cudaStream_t);
template cudaError_t launch_dot<float>(const RefParams<float>&, cudaStream_t);
template cudaError_t launch_dot_staged<double>(const DotParams<double>&, cudaStream_t);
template cudaError_t launch_dot_staged<float>(const DotParams<float>&, cudaStream_t);
template cudaError_t launch_serial<double>(const SerialParams<double>&, cudaStream_t);
template cudaError_t launch_serial<float>(const SerialParams<float>&, cudaStream_t);
template cudaError_t launch_zero<double>(double*, const GroupDev&, cudaStream_t);
template cudaError_t launch_zero<float>(float*, const GroupDev&, cudaStream_t);

}  // namespace gett
