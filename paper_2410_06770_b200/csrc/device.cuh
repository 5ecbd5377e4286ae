// Device-side types shared by the xGETT kernels (sm_100a).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace gett {

// cudaFuncSetAttribute is per device: opt a kernel into `bytes` of dynamic
// shared memory once per device (bit d of `mask`).  Calls on different devices
// may run concurrently (per-device API locks), so the mask is read and set
// atomically; a race only repeats the (idempotent) attribute call.
template <class Kern>
inline cudaError_t ensure_dyn_smem(Kern k, int bytes, unsigned long long& mask) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 64 && ((__atomic_load_n(&mask, __ATOMIC_ACQUIRE) >> dev) & 1ull)) return cudaSuccess;
  e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && dev < 64) __atomic_fetch_or(&mask, 1ull << dev, __ATOMIC_RELEASE);
  return e;
}


// Division by a runtime-invariant positive int32 with one mul.hi + shift
// (round-up reciprocal; valid for 0 <= n < 2^31, 1 <= d < 2^31).
struct FastDiv {
  int32_t d;
  uint32_t mul;
  uint32_t shr;

  __host__ static FastDiv make(int32_t d) {
    FastDiv f;
    f.d = d;
    if (d == 1) {
      f.mul = 0;
      f.shr = 0;
    } else {
      uint32_t l = 0;
      while ((1ull << l) < (uint64_t)d) ++l;  // ceil(log2 d)
      uint32_t p = 31 + l;
      f.mul = (uint32_t)(((1ull << p) + (uint64_t)d - 1) / (uint64_t)d);
      f.shr = p - 32;
    }
    return f;
  }

  __device__ __forceinline__ void divmod(int32_t n, int32_t& q, int32_t& r) const {
    q = (d == 1) ? n : (int32_t)(__umulhi((uint32_t)n, mul) >> shr);
    r = n - q * d;
  }
};

// One folded mode group on the device: element g of the group sits at
//   T[t][g / e_in] + (g % e_in) * s_in[t]   in tensor t.
struct GroupDev {
  int32_t G;
  FastDiv e_in;
  int64_t s_in[2];
  const int64_t* T[2];

  __device__ __forceinline__ int64_t off(int t, int32_t g) const {
    int32_t q, r;
    e_in.divmod(g, q, r);
    return __ldg(T[t] + q) + (int64_t)r * s_in[t];
  }
  __device__ __forceinline__ void off2(int32_t g, int64_t& o0, int64_t& o1) const {
    int32_t q, r;
    e_in.divmod(g, q, r);
    o0 = __ldg(T[0] + q) + (int64_t)r * s_in[0];
    o1 = __ldg(T[1] + q) + (int64_t)r * s_in[1];
  }
};

// Tiled GETT launch parameters.  Roles are the kernel's: A' (rows m) and B'
// (columns n); gm = (A', C), gn = (B', C), gk = (A', B').
template <typename T>
struct TiledParams {
  const T* A;
  const T* B;
  T* C;
  GroupDev gm, gn, gk;
  int32_t M, N, K;
  int32_t tiles_m, tiles_n;
  int32_t splits;   // split-K factor (1 = fused C += acc epilogue)
  int32_t k_chunk;  // K per split, a multiple of the k-block
  T* ws;            // [splits][M][N] partial tiles when splits > 1 ([splits][N][M] if ws_t)
  int32_t neg = 0;  // epilogue C += -acc (the a.im*b.im term of a complex contraction)
  int32_t ws_t = 0; // split-K workspace transposed (tcgen05 SGETT epilogue: m fastest)
  int32_t c_bulk = 0; // DGETT bulk-add epilogue (dgett_ws.cu), bits: 1 = C's N group has a unit
                      // inner stride and an inner extent a multiple of 32, every offset even and
                      // C 16-B aligned; 2 = also C's M group's inner extent a multiple of 32 (32
                      // consecutive rows from a 32-aligned start are affine: one thread issues
                      // their adds)
  // wide SGETT kernel, tail split (sgett_tc.cu): the pair tiles [tail_tile0,
  // tail_tile0 + tail_tiles) of the raster — the partial last wave — are cut
  // in two K halves (k_chunk) whose partials go to the compact workspace
  // ws [2][tail_tiles][256 n][256 m]; every other tile runs its whole K with the
  // fused epilogue.  tail_tiles == 0: off.
  int32_t tail_tile0 = 0, tail_tiles = 0;
};

// Persistent stream-K schedule of the DGETT kernel (dgett_ws.cu); enabled == 0
// launches one CTA per tile (and split-K slice).
struct SkParams {
  int32_t enabled = 0;
  int32_t grid = 0;       // persistent CTAs (one per SM)
  int32_t nkb = 0;        // k-blocks per tile
  int32_t sk_tile0 = 0;   // tiles [sk_tile0, ntiles) are shared out by k-block units
  int64_t sk_units = 0;   // (ntiles - sk_tile0) * nkb
  double* part = nullptr; // [grid][128*128] tail partials
  int32_t* flags = nullptr;  // [grid] "part published" epochs
  int32_t epoch = 0;
  // L2 cache-policy hints (TMA producer, bulk-add epilogue): bit 0 A' boxes
  // evict_last, bit 1 B' boxes evict_first, bit 2 the C bulk adds evict_first,
  // bit 3 exchanges the A' / B' policies; bit 4 (the default): serpentine k —
  // every other data-parallel tile of a CTA is summed from its last k-block down
  int32_t l2hint = 0;
};


// TMA-fed operands of the SGETT kernel (sgett_tc.cu), built by the host when a
// tile's rows and a k-block's k values are boxes of an affine (<= 5-D,
// positive-stride) view: one rank-5 tensor map per operand (unused dims have
// extent 1).  K-major operands (kf) put the inner k mode in TMA dim 0 and load
// 8-float boxes with SWIZZLE_32B (the UMMA K-major SW32 layout, 4 KB per 8 k);
// rows-major operands put the rows first and load [8 k][128 rows] boxes (the
// [k][row] staging of the cp.async path).  The row index (k index) is the
// mixed radix of its dims' coordinates, inner first, at TMA dims r_pos (k_pos).
struct TmaOperand {
  int32_t kf;
  int32_t nr, nk;
  int32_t r_ext[3], r_pos[3];
  int32_t k_ext[3], k_pos[3];
};
struct TmaParams {
  CUtensorMap map[2];   // A', B'
  TmaOperand op[2];
};

// SGETT "k-run" kernel (sgett_kr.cu): the TMEM operand X has a contiguous
// inner k run of KR floats (KR % 8 == 0, <= 64) — one k-block is one whole
// run, loaded as a dense [rows][KR] TMA box (long contiguous lines instead of
// 32 B SW32 boxes) and split straight into TMEM; Y is rows-major ([KR k][NT
// rows] boxes) and transposed into K-major hi/lo tiles for the MMA's B.  The
// accumulator is [128 X rows][NT Y rows].  With split-K the partials land in
// ws [splits][NY][MX] (x fastest) and, when epoch != 0, the CTAs of a tile
// reduce them themselves (each its slice, in split order), else the separate
// reduce kernel does (CUDA-graph capture: the epoch would be baked in).
constexpr int KR_MAX_SPLITS = 256;
constexpr int KR_MAX_TILES = 256;  // fused split-K reduce: tiles of one call
struct KrParams {
  float* C;
  GroupDev gx, gy;  // tensor 1 = C offsets of X rows / Y rows
  int32_t MX, NY, NT;
  int32_t x_rows, y_rows;  // rows one X / Y box covers (<= 128 / <= NT; a multiple of the inner row extent)
  int32_t tiles_x, tiles_y;
  int32_t nkb, kpc, splits;  // k-blocks (k runs) in all, per split, splits
  float* ws;
  // fused split-K reduce (null: the separate reduce kernel): per tile an
  // arrival counter that wraps to 0 after `splits` arrivals (atomicInc), a
  // generation bumped by the last arriver, and per slice the generation it
  // was last claimed for — self-resetting, so CUDA-graph replays are safe
  uint32_t* cnt;    // [tiles]
  uint32_t* gen;    // [tiles]
  uint32_t* claim;  // [tiles][KR_MAX_SPLITS]: slot (t, s) only ever holds tile t's generations
  int32_t neg;
  int64_t spin_ns;  // bounded wait of a split for its tile's other splits
  // shared-memory / TMEM layout (host-computed for this NT): lslots load
  // slots [X raw 128 x (KR+4) | Y raw KR x NT] of lslot_bytes from 0,
  // oslots operand slots [Y hi | Y lo] of oslot_bytes from o_off, barriers
  // at bar_off; aslots TMEM A slots of 2 KR columns from a_col0 (after the NT
  // accumulator columns)
  int32_t lslots, oslots, aslots, lslot_bytes, oslot_bytes, o_off, bar_off, a_col0;
  int32_t xnr, ynr, nko;                   // row dims of X / Y, outer k dims
  int32_t xr_ext[3], xr_pos[3], yr_ext[3], yr_pos[3];
  int32_t k_ext[2], xk_pos[2], yk_pos[2];  // outer k digits (inner first)
  CUtensorMap mx, my;
};

// the fused epilogue's update: C + acc, or C + (-acc) == C - acc for neg
template <typename T>
__device__ __forceinline__ T epi(T c, T acc, int32_t neg) {
  return neg ? c - acc : c + acc;
}

// Reference-order kernel parameters: one thread per output, K in the
// reference order (pair 0 fastest) with unfused multiply then add.
template <typename T>
struct RefParams {
  const T* A;
  const T* B;
  T* C;
  GroupDev gm, gn;      // as in TiledParams
  int32_t M, N;
  int32_t k_inner;      // reference-order K: inner affine extent ...
  int64_t k_sa, k_sb;   // ... and its strides in A', B'
  int32_t k_outer;      // outer table length
  const int64_t* kta;   // outer offsets in A'
  const int64_t* ktb;   // outer offsets in B'
  FastDiv kdiv;         // division by k_inner (dot kernel)
};

// Staged dot kernel (few outputs, long K): one operand's row is staged in
// shared memory in the K order of gk, the other ("streamed") is read along its
// unit-stride inner k mode, one warp per output.  stream_a: A' rows are
// streamed (k tensor 0) and B' rows staged, else the reverse.
template <typename T>
struct DotParams {
  const T* A;
  const T* B;
  T* C;
  GroupDev gm, gn, gk;
  int32_t M, N, K;
  int32_t stream_a;
};

// Serial kernel: the literal reference loop (kernel.py:48-78) on one thread,
// used when distinct output coordinates may address the same C element.
template <typename T>
struct SerialParams {
  const T* A;
  const T* B;
  T* C;
  int32_t num_free, num_cont;
  int64_t size_free, size_cont;
  const int64_t* tab;  // [out_inc | src_inc | from_a | ext_free] x num_free,
                       // [inc_ca | inc_cb | ext_cont] x num_cont
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void cp_async_8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async_4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async_16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

}  // namespace gett
