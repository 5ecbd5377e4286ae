/*
 * gett_b200.h — C ABI of the B200-native xGETT (arXiv 2410.06770).
 *
 * One binary tensor contraction, C += contract(A, B), over strided views of
 * flat buffers, with the argument order of the thesis's xGETT
 * and the semantics of the reference Python package:
 *
 *   gett_dgett / gett_sgett   replace  gett.kernel.dgett / sgett
 *                             (/root/reference/pkg/src/gett/kernel.py:158-184,
 *                              via _gett kernel.py:124-155)
 *   gett_validate             replaces gett.plan.validate (plan.py:162-234)
 *                             plus the phase-2 output footprint check
 *                             (kernel.py:149-153, plan.py:237-241)
 *   gett_derive_output_extents replaces plan.derive_output_extents (plan.py:119-127)
 *   gett_zero_view_{d,s}      replaces gett.kernel.zero_view (kernel.py:111-113)
 *
 * Conventions
 *   - A view is (rank, ext[rank], inc[rank]) over a buffer of `len` elements,
 *     its coordinate (0,...,0) at element `offset` (the reference's offset_x
 *     keywords, README.md:56-59).  Increments may be negative or zero.
 *   - PERM maps free index -> output position (plan.py:10-12); free indices
 *     are A's free dims ascending, then B's (plan.py:113-116).
 *   - C is accumulated: C += A·B (kernel.py:76).  Output extents are derived.
 *   - Value problems are returned as coded errors, in the reference's order
 *     (plan.py:179-232), with C untouched and no kernel launched.
 *   - Structural problems that the reference raises as TypeError/ValueError
 *     (kernel.py:132-140, layout.py:71-84, plan.py:62-72) are the caller's
 *     (the Python shim's) job; in C the array lengths are implied by the
 *     ranks, except perm_len and inc_c_len, which the reference validates
 *     as values (PermLengthWrong, IncCLengthWrong).
 *
 * Return value: number of validation errors (>= 0; 0 = the contraction ran),
 * or a negative GETT_E_* status (CUDA failure, bad argument, out of memory).
 * err_codes[i] / err_info[6*i .. 6*i+5] receive the first max_errs errors.
 *
 * Host entry points (gett_dgett, gett_sgett, gett_zero_view_*) take HOST
 * buffers, copy the addressed spans to the device, run on the current CUDA
 * device and copy C's span back before returning (synchronous, like the
 * reference).  *_device entry points take DEVICE pointers and are
 * stream-ordered on `stream` (a cudaStream_t; NULL = legacy default stream).
 */
#ifndef GETT_B200_H_
#define GETT_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* validation error codes: gett.plan.ErrorCode (plan.py:23-32) */
enum gett_error_code {
  GETT_EXTENT_MISMATCH = 1,
  GETT_CONT_INDEX_OUT_OF_RANGE = 2,
  GETT_CONT_INDEX_DUPLICATE = 3,
  GETT_PERM_LENGTH_WRONG = 4,
  GETT_PERM_NOT_BIJECTION = 5,
  GETT_INC_C_LENGTH_WRONG = 6,
  GETT_OUTPUT_WRITE_ALIASING = 7,
  GETT_FOOTPRINT_OUT_OF_BOUNDS = 8,
  GETT_NEGATIVE_EXTENT = 9
};

/* err_info layout per error (6 x int64), used to rebuild the reference's
 * messages:
 *   NEGATIVE_EXTENT          [tensor(0=A,1=B,2=C), dim, extent, 0, 0, 0]
 *   CONT_INDEX_OUT_OF_RANGE  [tensor, k, d, rank, 0, 0]
 *   CONT_INDEX_DUPLICATE     [tensor, k, d, 0, 0, 0]
 *   EXTENT_MISMATCH          [-1, k, ext_a, dim_a, ext_b, dim_b]
 *   PERM_LENGTH_WRONG        [-1, perm_len, rank_c, 0, 0, 0]
 *   PERM_NOT_BIJECTION       [-1, rank_c, 0, 0, 0, 0]
 *   INC_C_LENGTH_WRONG       [-1, inc_c_len, rank_c, 0, 0, 0]
 *   OUTPUT_WRITE_ALIASING    [2, dim, extent, 0, 0, 0]
 *   FOOTPRINT_OUT_OF_BOUNDS  [tensor, lowest offset, highest offset, buffer len, 0, 0]
 */
#define GETT_ERR_INFO_WORDS 6

/* negative status codes */
#define GETT_E_CUDA (-1)
#define GETT_E_INVALID_ARG (-2)
#define GETT_E_NOMEM (-3)
#define GETT_E_UNSUPPORTED (-4)

/* ---- xGETT, host buffers (synchronous drop-in) ---- */
int gett_dgett(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const double* a,
               int64_t offset_a, int64_t len_a,
               int rank_b, const int64_t* ext_b, const int64_t* inc_b, const double* b,
               int64_t offset_b, int64_t len_b,
               int conts, const int64_t* cont_a, const int64_t* cont_b,
               int perm_len, const int64_t* perm,
               int inc_c_len, const int64_t* inc_c, double* c, int64_t offset_c, int64_t len_c,
               int32_t* err_codes, int64_t* err_info, int max_errs);

int gett_sgett(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const float* a,
               int64_t offset_a, int64_t len_a,
               int rank_b, const int64_t* ext_b, const int64_t* inc_b, const float* b,
               int64_t offset_b, int64_t len_b,
               int conts, const int64_t* cont_a, const int64_t* cont_b,
               int perm_len, const int64_t* perm,
               int inc_c_len, const int64_t* inc_c, float* c, int64_t offset_c, int64_t len_c,
               int32_t* err_codes, int64_t* err_info, int max_errs);

/* ---- xGETT, device buffers (stream-ordered; zero-copy) ---- */
int gett_dgett_device(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const double* a,
                      int64_t offset_a, int64_t len_a,
                      int rank_b, const int64_t* ext_b, const int64_t* inc_b, const double* b,
                      int64_t offset_b, int64_t len_b,
                      int conts, const int64_t* cont_a, const int64_t* cont_b,
                      int perm_len, const int64_t* perm,
                      int inc_c_len, const int64_t* inc_c, double* c, int64_t offset_c,
                      int64_t len_c, void* stream,
                      int32_t* err_codes, int64_t* err_info, int max_errs);

int gett_sgett_device(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const float* a,
                      int64_t offset_a, int64_t len_a,
                      int rank_b, const int64_t* ext_b, const int64_t* inc_b, const float* b,
                      int64_t offset_b, int64_t len_b,
                      int conts, const int64_t* cont_a, const int64_t* cont_b,
                      int perm_len, const int64_t* perm,
                      int inc_c_len, const int64_t* inc_c, float* c, int64_t offset_c,
                      int64_t len_c, void* stream,
                      int32_t* err_codes, int64_t* err_info, int max_errs);

/* ---- xGETT over several devices, host buffers (synchronous) ----
 * One call drives the listed CUDA devices (the reference's
 * concurrency rule: calls writing disjoint C
 * footprints may run concurrently):
 *   - slabs:   C's outermost free mode (largest |INCC|, disjoint spans) is
 *              split into one row range per device; each device copies its
 *              slabs of the owner operand and of C over its own PCIe link and
 *              computes them; the other operand crosses PCIe once in total
 *              (device j uploads chunk j, the devices exchange chunks over
 *              NVLink).  No collective.  Each slab is the same xGETT a
 *              one-device call on that sub-view computes (a free-mode slice).
 *   - split-K: when the free extents cannot fill the devices (e.g. c5), the
 *              contracted pair with the largest extent is split; device 0
 *              computes C += A_0·B_0, device j > 0 computes P_j = A_j·B_j,
 *              and device 0 adds C += (P_1 + ... + P_{n-1}) in that order,
 *              loading the partials from the peers over NVLink.
 *   - small calls (< 2^27 MACs per device) and self-overlapping C views run
 *     on devices[0] alone.
 * A device may be listed more than once (each occurrence is a separate lane
 * with its own streams and staging), so devices = {0, 0} runs the whole
 * multi-device path on one GPU.  Validation, errors and return values are
 * those of gett_dgett / gett_sgett.  Replaces: kernel.py:158-184 (the same
 * call; the reference is single-threaded on one CPU core). */
int gett_dgett_multi(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const double* a,
                     int64_t offset_a, int64_t len_a,
                     int rank_b, const int64_t* ext_b, const int64_t* inc_b, const double* b,
                     int64_t offset_b, int64_t len_b,
                     int conts, const int64_t* cont_a, const int64_t* cont_b,
                     int perm_len, const int64_t* perm,
                     int inc_c_len, const int64_t* inc_c, double* c, int64_t offset_c,
                     int64_t len_c, int n_dev, const int32_t* devices,
                     int32_t* err_codes, int64_t* err_info, int max_errs);
int gett_sgett_multi(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const float* a,
                     int64_t offset_a, int64_t len_a,
                     int rank_b, const int64_t* ext_b, const int64_t* inc_b, const float* b,
                     int64_t offset_b, int64_t len_b,
                     int conts, const int64_t* cont_a, const int64_t* cont_b,
                     int perm_len, const int64_t* perm,
                     int inc_c_len, const int64_t* inc_c, float* c, int64_t offset_c,
                     int64_t len_c, int n_dev, const int32_t* devices,
                     int32_t* err_codes, int64_t* err_info, int max_errs);
/* Default device list of gett_dgett / gett_sgett (the unchanged drop-in
 * signature then runs multi-device); n_dev = 0 restores the current device.
 * Returns 0 or GETT_E_INVALID_ARG (ordinal out of range). */
int gett_set_devices(int n_dev, const int32_t* devices);
/* Multi-device strategy: 0 = automatic (default), 1 = always slabs,
 * 2 = always split-K (when the call allows it; for tests); + 4 = the split-K
 * reduce stages the partials with cudaMemcpyPeerAsync instead of loading them
 * over NVLink (also GETT_MULTI_STAGE=1). */
int gett_set_multi(int strategy);
/* Description of the last host call's multi-device schedule ("none" when it
 * ran on one device), e.g. "slabs x2 (...)", "split-K x2 (pair 2, peer-load reduce)". */
const char* gett_last_multi(void);

/* The multi-device schedule gett_{d,s}gett_multi would run for this call on
 * n_dev devices, computed on the host (no CUDA) — also the partition a
 * one-process-per-GPU launcher (torchrun) gives its ranks.  strategy: 0 =
 * automatic, 1 = slabs, 2 = split-K when the call allows it (as
 * gett_set_multi, for this query only).  sched receives
 * 4 + 2*n_dev int64:
 *   [0] strategy: 0 = one device, 1 = slabs, 2 = split-K
 *   [1] lanes used (n <= n_dev; lane i is devices[i])
 *   [2] slabs: the operand owning the cut mode (0 = A, 1 = B); else -1
 *   [3] slabs: that operand's dimension; split-K: the contracted pair; else -1
 *   [4 + 2i], [5 + 2i]: lane i's range [lo, hi) of that dimension / pair.
 * Returns the validation error count (> 0: sched untouched) or a negative
 * status.  Replaces: shard.py's Python mode choice (round 1). */
int gett_multi_schedule(int rank_a, const int64_t* ext_a, const int64_t* inc_a, int64_t offset_a,
                        int64_t len_a,
                        int rank_b, const int64_t* ext_b, const int64_t* inc_b, int64_t offset_b,
                        int64_t len_b,
                        int conts, const int64_t* cont_a, const int64_t* cont_b,
                        int perm_len, const int64_t* perm, int inc_c_len, const int64_t* inc_c,
                        int64_t offset_c, int64_t len_c, int n_dev, int strategy,
                        int64_t* sched, int32_t* err_codes, int64_t* err_info, int max_errs);

/* ---- complex xGETT: cgett / zgett (kernel.py:187-200) ----
 * Buffers are interleaved (re, im) pairs (numpy complex64 / complex128 memory);
 * offsets, lengths and increments count complex elements.  Products follow the
 * reference's complex multiply: re = a.re*b.re - a.im*b.im, im = a.re*b.im + a.im*b.re. */
int gett_zgett(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const double* a,
               int64_t offset_a, int64_t len_a,
               int rank_b, const int64_t* ext_b, const int64_t* inc_b, const double* b,
               int64_t offset_b, int64_t len_b,
               int conts, const int64_t* cont_a, const int64_t* cont_b,
               int perm_len, const int64_t* perm,
               int inc_c_len, const int64_t* inc_c, double* c, int64_t offset_c, int64_t len_c,
               int32_t* err_codes, int64_t* err_info, int max_errs);
int gett_cgett(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const float* a,
               int64_t offset_a, int64_t len_a,
               int rank_b, const int64_t* ext_b, const int64_t* inc_b, const float* b,
               int64_t offset_b, int64_t len_b,
               int conts, const int64_t* cont_a, const int64_t* cont_b,
               int perm_len, const int64_t* perm,
               int inc_c_len, const int64_t* inc_c, float* c, int64_t offset_c, int64_t len_c,
               int32_t* err_codes, int64_t* err_info, int max_errs);
int gett_zgett_device(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const double* a,
                      int64_t offset_a, int64_t len_a,
                      int rank_b, const int64_t* ext_b, const int64_t* inc_b, const double* b,
                      int64_t offset_b, int64_t len_b,
                      int conts, const int64_t* cont_a, const int64_t* cont_b,
                      int perm_len, const int64_t* perm,
                      int inc_c_len, const int64_t* inc_c, double* c, int64_t offset_c,
                      int64_t len_c, void* stream,
                      int32_t* err_codes, int64_t* err_info, int max_errs);
int gett_cgett_device(int rank_a, const int64_t* ext_a, const int64_t* inc_a, const float* a,
                      int64_t offset_a, int64_t len_a,
                      int rank_b, const int64_t* ext_b, const int64_t* inc_b, const float* b,
                      int64_t offset_b, int64_t len_b,
                      int conts, const int64_t* cont_a, const int64_t* cont_b,
                      int perm_len, const int64_t* perm,
                      int inc_c_len, const int64_t* inc_c, float* c, int64_t offset_c,
                      int64_t len_c, void* stream,
                      int32_t* err_codes, int64_t* err_info, int max_errs);

/* ---- plan once, execute many (d and s) ----
 * gett_plan_create validates a descriptor exactly like gett_dgett (same
 * codes; the C view is footprint-checked against offset_c / len_c) and, when
 * it is valid, returns a handle holding the device plan.  gett_execute (host
 * buffers, synchronous) and gett_execute_device (device pointers, stream-
 * ordered) then run C += contract(A, B) on buffers of the planned lengths at
 * the planned offsets, without validation, descriptor hashing or plan lookup:
 * the per-call host cost of a small contraction.  The same call semantics
 * as the reference's dgett/sgett (kernel.py:158-184) minus its per-call
 * argument processing (kernel.py:124-155).  dtype: 'd' or 's'.  Returns the
 * validation error count (> 0: *out = NULL) or a negative status; a handle
 * with an empty iteration space executes to nothing.  n_dev/devices: as
 * gett_dgett_multi (0 = the current device).  A handle may be executed from
 * any thread; destroy it once. */
typedef struct gett_plan_s* gett_plan_t;
int gett_plan_create(char dtype, int rank_a, const int64_t* ext_a, const int64_t* inc_a, int64_t offset_a,
                     int64_t len_a, int rank_b, const int64_t* ext_b, const int64_t* inc_b,
                     int64_t offset_b, int64_t len_b, int conts, const int64_t* cont_a,
                     const int64_t* cont_b, int perm_len, const int64_t* perm, int inc_c_len,
                     const int64_t* inc_c, int64_t offset_c, int64_t len_c, int n_dev,
                     const int32_t* devices, gett_plan_t* out, int32_t* err_codes, int64_t* err_info,
                     int max_errs);
int gett_execute(gett_plan_t plan, const void* a, const void* b, void* c);
int gett_execute_device(gett_plan_t plan, const void* a, const void* b, void* c, void* stream);
void gett_plan_destroy(gett_plan_t plan);

/* ---- planning helpers ---- */
/* Validation only.  c_mode selects how the output view takes part:
 *   GETT_CHECK_C_NONE     plan.validate(a, b, spec, inc_c)           (plan.py:162-234)
 *   GETT_CHECK_C_DERIVED  xGETT's two phases: the C view (derived extents, inc_c,
 *                         offset_c, len_c) is footprint-checked only when
 *                         everything else is clean                    (kernel.py:146-153)
 *   GETT_CHECK_C_EXPLICIT plan.validate(..., c_view) with the explicit view
 *                         (rank_cv, ext_cv, inc_cv, offset_c, len_c)  (plan.py:179-232) */
#define GETT_CHECK_C_NONE 0
#define GETT_CHECK_C_DERIVED 1
#define GETT_CHECK_C_EXPLICIT 2
int gett_validate(int rank_a, const int64_t* ext_a, const int64_t* inc_a, int64_t offset_a,
                  int64_t len_a,
                  int rank_b, const int64_t* ext_b, const int64_t* inc_b, int64_t offset_b,
                  int64_t len_b,
                  int conts, const int64_t* cont_a, const int64_t* cont_b,
                  int perm_len, const int64_t* perm, int inc_c_len, const int64_t* inc_c,
                  int c_mode, int rank_cv, const int64_t* ext_cv, const int64_t* inc_cv,
                  int64_t offset_c, int64_t len_c,
                  int32_t* err_codes, int64_t* err_info, int max_errs);

/* ext_c[perm[i]] = extent of free index i; requires a valid spec.
 * Returns rank_c, or GETT_E_INVALID_ARG. */
int gett_derive_output_extents(int rank_a, const int64_t* ext_a, int rank_b, const int64_t* ext_b,
                               int conts, const int64_t* cont_a, const int64_t* cont_b,
                               const int64_t* perm, int64_t* ext_c_out);

/* ---- zero_view: set every addressed element to 0, nothing else ---- */
int gett_zero_view_d(int rank, const int64_t* ext, const int64_t* inc, int64_t offset,
                     int64_t len, double* buf);
int gett_zero_view_s(int rank, const int64_t* ext, const int64_t* inc, int64_t offset,
                     int64_t len, float* buf);
int gett_zero_view_d_device(int rank, const int64_t* ext, const int64_t* inc, int64_t offset,
                            int64_t len, double* buf, void* stream);
int gett_zero_view_s_device(int rank, const int64_t* ext, const int64_t* inc, int64_t offset,
                            int64_t len, float* buf, void* stream);

/* ---- pack: the addressed elements of a view in canonical packed order
 * (dimension 0 fastest), a bit-exact copy of elem_bytes = 4, 8 or 16 per
 * element (f32, f64 / c64, c128).  Replaces testkit.pack
 * (/root/reference/pkg/src/gett/testkit.py:101-103, buf[view_offsets(view)]).
 * gett_pack: host src (the whole buffer, view at `offset`) and host dst of
 * prod(ext) elements; gett_pack_device: device pointers, stream-ordered.
 * Returns 0 or GETT_E_INVALID_ARG (rank > 32, negative extent, footprint
 * outside [0, len)). */
int gett_pack(int rank, const int64_t* ext, const int64_t* inc, int64_t offset, int64_t len,
              int elem_bytes, const void* src, void* dst);
int gett_pack_device(int rank, const int64_t* ext, const int64_t* inc, int64_t offset, int64_t len,
                     int elem_bytes, const void* src, void* dst, void* stream);

/* ---- runtime control ---- */
/* Kernel selection: "auto" (default), "ref" (reference-order kernel, bitwise
 * equal to the reference on all data), "tiled" (tensor-core / register-tiled
 * kernel), "dot" (one warp per output: few outputs, long K), "ffma" (SGETT on
 * the FP32 FFMA core instead of tcgen05), "serial" (one GPU thread, literal
 * reference loop).  Also set by the environment variable GETT_KERNEL.
 * Returns 0 or GETT_E_INVALID_ARG. */
int gett_set_kernel(const char* name);
/* Force the split-K factor of the tiled kernel (0 = automatic). */
int gett_set_split_k(int split);
/* Host entry points only: overlap H2D / compute / D2H by cutting C's outermost
 * free mode into `slabs` sub-contractions (-1 = automatic for calls moving
 * >= 64 MB, 0 = off, n >= 2 = always n slabs).  Also GETT_PIPELINE. */
int gett_set_pipeline(int slabs);
/* DGETT persistent stream-K schedule (1 = on when the tiles exceed one wave,
 * the default; 0 = one CTA per tile).  Also GETT_STREAM_K. */
int gett_set_stream_k(int on);
/* SGETT operands fed by TMA tensor maps when both views are affine boxes
 * (1 = on, the default; 0 = cp.async gathers only).  Also GETT_TMA. */
int gett_set_tma(int on);
/* DGETT epilogue C += acc as bulk shared->global f64 add reductions of whole
 * 32-element C row runs (cp.reduce.async.bulk; 1 = when C's N runs are
 * contiguous, even-aligned and C is 16-byte aligned, the default; 0 = one
 * red.add per element).  Both add each element once at L2: bitwise equal
 * results.  Also GETT_DGETT_BULK. */
int gett_set_bulk(int on);
/* SGETT wide CTA-pair kernel (tcgen05.mma.cta_group::2, a 256 x 256 output
 * tile per cluster of 2, half the shared-memory traffic per MAC of the
 * 128 x 128 kernel): 0 = off, 1 = automatic (tilings that fill at least half
 * the SMs, the default), 2 = whenever both operands are TMA-fed and M, N >=
 * 256; + 4 = the mixed split (one tf32 MMA hi * hi + one bf16 MMA carrying
 * both cross terms per 8 k, as the k-run kernel's; see gett_set_kr) instead of
 * the default three tf32 MMAs (3xTF32 truncation split, bitwise equal to the
 * 128 x 128 kernel without split-K): same accuracy, no faster while the
 * kernel is tensor-bound at the power cap and split-latency bound above it;
 * + 8 = no tail split (by default a partial last wave of at most half the
 * pair slots runs as two K halves per tile, summed by a small reduce kernel:
 * 4096^3 takes 3.5 instead of 4 waves' time).  Also GETT_WIDE / GETT_WIDE_MIX /
 * GETT_WIDE_TAIL / GETT_WIDE_K16 (K-major operands as one 16-k SWIZZLE_64B box
 * per k-block, default 1). */
int gett_set_wide(int mode);
/* Programmatic dependent launch of the k-run SGETT kernel and of the split-K
 * reduce kernels (cudaLaunchAttributeProgrammaticStreamSerialization): each is
 * scheduled while its predecessor in the stream drains — barrier / TMEM set-up
 * and launch latency overlap the predecessor's tail — and executes
 * griddepcontrol.wait before it touches global memory.  1 = on (the default),
 * 0 = ordinary launches.  Also GETT_PDL.  c5 back to back 38.5 -> 35.1 us. */
int gett_set_pdl(int on);
/* SGETT CTA-pair kernel (tcgen05.mma.cta_group::2, M = 256 per pair) for
 * split-K shapes with a K-major operand of >= 256 rows and a rows-major one of
 * <= 128 (e.g. c5); 0 = off (the default), 1 = on.  Also GETT_PAIR. */
int gett_set_pair(int on);
/* SGETT k-run kernel (one k-block = the TMEM operand's whole contiguous inner
 * k run, <= 64 floats; dense TMA boxes; split-K reduced inside the kernel):
 * 0 = off, 1 = automatic (runs < 64 on fewer tiles than SMs, the default),
 * 2 = whenever it applies; + 4 = split-K partials reduced inside the kernel
 * (tile counters; graph-replay safe) instead of by the separate reduce kernel
 * (the default); + 8 = never as CTA pairs (by default pairs of X tiles run as
 * cta_group::2 clusters, each CTA holding half of the other operand, with two
 * k runs per k-block when they fit); + 16 = three tf32 MMAs per 8 k (3xTF32,
 * truncation split) instead of the default mixed split: one tf32 MMA hi * hi
 * (hi rounded to tf32) and one bf16 MMA carrying both cross terms
 * ([bf16(x) | bf16(x_lo)] . [bf16(y_lo) ; bf16(y)]) — at least as accurate
 * (tools/umma_mixed_test.cu) at two thirds of the tensor work.  Also GETT_KR /
 * GETT_KR_FUSED / GETT_KR_PAIR / GETT_KR_MIX. */
int gett_set_kr(int mode);
/* cgett / zgett on the tensor-core kernels: 1 = one real GETT on a real
 * embedding of the smaller operand (the default), 0 = four real GETTs on the
 * re/im sub-views.  Also GETT_COMPLEX_EMBED. */
int gett_set_complex_embed(int on);
/* Name of the kernel the last call launched ("none" if none). */
const char* gett_last_kernel(void);
/* Text of the last CUDA / internal failure. */
const char* gett_last_error(void);
/* Number of kernels launched by this library since load (evidence counter). */
int64_t gett_launch_count(void);
/* Release cached device buffers and plans. */
void gett_release_caches(void);
/* ABI version: major*100 + minor. */
int gett_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* GETT_B200_H_ */
