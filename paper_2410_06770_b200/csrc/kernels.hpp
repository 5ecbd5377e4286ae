// Host-side launchers for the xGETT kernels (kernels.cu).
#pragma once

#include <cuda_runtime.h>

#include "device.cuh"

namespace gett {

// Programmatic dependent launch (capi.cu; GETT_PDL / gett_set_pdl): the k-run
// SGETT kernel and the split-K reduce are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so each is scheduled while
// its predecessor in the stream drains (both wait on griddepcontrol.wait before
// touching global memory the predecessor may still use).
extern int g_launch_pdl;

template <typename T>
cudaError_t launch_tiled(const TiledParams<T>& p, bool a_kf, bool b_kf, bool a_vec, bool b_vec,
                         cudaStream_t s);
template <typename T>
cudaError_t launch_ref(const RefParams<T>& p, cudaStream_t s);
template <typename T>
cudaError_t launch_serial(const SerialParams<T>& p, cudaStream_t s);
template <typename T>
cudaError_t launch_dot(const RefParams<T>& p, cudaStream_t s);  // warp per output
template <typename T>
cudaError_t launch_dot_staged(const DotParams<T>& p, cudaStream_t s);  // staged row, warp per output
constexpr int kDotStagedMaxK = 4096;
template <typename T>
cudaError_t launch_zero(T* base, const GroupDev& g, cudaStream_t s);

// Multi-device split-K reduce: for every element of the C view (folded as
// one group, g.T[0] / g.s_in[0]), C[o] = C[o] + (P[0][o] + ... + P[n-1][o]) in
// that order.  The partial pointers may be peer-device memory (NVLink loads).
constexpr int kMaxParts = 63;
template <typename T>
struct AccumParams {
  T* C;
  const T* P[kMaxParts];
  int n;
  GroupDev g;
};
template <typename T>
cudaError_t launch_accum(const AccumParams<T>& p, cudaStream_t s);

// pack (testkit.pack, /root/reference/pkg/src/gett/testkit.py:101-103): dst[i]
// = src[offset of packed index i], i in canonical order (dimension 0 fastest),
// a bit-exact copy of elem_bytes (4, 8 or 16) per element.
constexpr int kPackMaxRank = 32;
struct PackParams {
  const void* src;  // at the view's coordinate (0, ..., 0)
  void* dst;
  int rank;
  int64_t n;
  int64_t ext[kPackMaxRank], inc[kPackMaxRank];
  FastDiv div[kPackMaxRank];  // used when n < 2^31
};
cudaError_t launch_pack(const PackParams& p, int elem_bytes, cudaStream_t s);

template <typename T>
cudaError_t launch_splitk_reduce(const TiledParams<T>& p, cudaStream_t s);

// complex (interleaved re/im, offsets in complex elements): R = float / double
template <typename R>
cudaError_t launch_ref_c(const RefParams<R>& p, cudaStream_t s);
template <typename R>
cudaError_t launch_serial_c(const SerialParams<R>& p, cudaStream_t s);

// Real embedding of one complex operand (run_complex in capi.cu): for each
// element b of the strided view, dst[o] = (re b, im b) and dst[o + q] =
// (-im b, re b), o = sum idx_d * dst_st[d] (modes fastest first).
constexpr int kExpandMaxModes = 24;
template <typename R>
struct ExpandParams {
  const R* src;  // interleaved (re, im) at the view's base element
  R* dst;
  int n;          // modes
  int64_t total;  // elements of the view
  int64_t q;      // real offset of the (-im, re) pair
  int64_t ext[kExpandMaxModes], inc[kExpandMaxModes], dst_st[kExpandMaxModes];  // inc in complex elements
};
template <typename R>
cudaError_t launch_expand_complex(const ExpandParams<R>& p, cudaStream_t s);

// DGETT warp-specialised (producer warp + DMMA consumer warps), dgett_ws.cu
// tp != nullptr: both operands TMA-fed (128B-swizzled boxes; capi.cu dgett_tma)
cudaError_t launch_dgett_ws(const TiledParams<double>& p, const SkParams& sk, const TmaParams* tp,
                            bool a_kf, bool b_kf, bool a_vec, bool b_vec, cudaStream_t s);
int dgett_ws_tiles_k(int K);  // k-blocks per tile

// SGETT 3xTF32 on tcgen05 (sgett_tc.cu); tp != nullptr: both operands TMA-fed
cudaError_t launch_sgett_tc(const TiledParams<float>& p, const TmaParams* tp, bool a_kf, bool b_kf,
                            bool a_vec, bool b_vec, cudaStream_t s);

// CTA-pair SGETT (M = 256 per pair, N <= 128 split across the pair; both
// operands TMA-fed: A' K-major, B' rows-major with NBH-row boxes); split-K
cudaError_t launch_sgett_tc_pair(const TiledParams<float>& p, const TmaParams& tp, cudaStream_t s);

// wide CTA-pair SGETT (256 x 256 tile per pair; both operands TMA-fed);
// p.tiles_m / tiles_n count pair tiles; split-K partials [split][N][M]
// mix: per 8 k one tf32 MMA (hi * hi) + one bf16 MMA (both cross terms) instead
// of three tf32 MMAs
// k16: tp's K-major operands are one [16 k][128 rows] SWIZZLE_64B box per
// k-block (capi.cu sgett_tma64) instead of two SW32 boxes
cudaError_t launch_sgett_tc_wide(const TiledParams<float>& p, const TmaParams& tp, bool a_kf, bool b_kf,
                                 bool mix, bool k16, cudaStream_t s);

// k-run SGETT (sgett_kr.cu); KR in {8, 16, ..., 64}
// pair: clusters of 2 (cta_group::2, M = 256; tiles_x even, y_rows == NT)
// KRN: k runs per k-block (1, or 2 for KR <= 40)
// mix: per 8 k one tf32 MMA (hi * hi) + one bf16 MMA (both cross terms)
// instead of three tf32 MMAs
cudaError_t launch_sgett_kr(const KrParams& p, int KR, int KRN, bool pair, bool mix, cudaStream_t s);
int sgett_kr_max_nt();

int tiled_bm();
int tiled_bn();
int tiled_bk(int elt_bytes);
int tc_bm();
int tc_bn();
int tc_bk();

}  // namespace gett
