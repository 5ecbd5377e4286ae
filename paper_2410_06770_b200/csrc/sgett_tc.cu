// SGETT on the 5th-generation tensor cores: 3xTF32 with tcgen05.mma + TMEM,
// warp-specialised.
//
// Replaces the fp32 hot loop (kernel.py:48-78 for sgett) for contractions big
// enough to tile.  Per 128x128 output tile, k-blocks of 16, STAGES-deep ring
// of (A' staging, B' raw) plus a LO_BUFS-deep ring of B' lo tiles:
//   * loads — TMA (TMA=true, both operands affine boxes, capi.cu tma_layout):
//     four lanes of the producer warp issue one cp.async.bulk.tensor box each
//     per k-block (K-major operands as SWIZZLE_32B [128 rows][8 k] boxes =
//     the UMMA K-major SW32 layout; rows-major operands as [8 k][128 rows]);
//     gathers (otherwise): the producer warpgroup cp.asyncs the tiles straight
//     from the strided views (16 B along k into the no-swizzle K-major core
//     layout, or along rows into [k][row] staging, else 4 B; zero fill past
//     the view; k offsets decoded lane-parallel from the staged K table);
//   * split warpgroups (warps 4-11, alternate k-blocks): the tensor core reads
//     a raw fp32 operand as tf32 by truncation, so the raw value is the hi
//     part and only lo = x - trunc(x) (exact) is produced: A' hi/lo go to TMEM
//     (tcgen05.st, lane = row, column = k: A' never returns to shared memory);
//     a K-major B' tile is used in place as B' hi and its lo written to the lo
//     ring; a rows-major B' is transposed into K-major hi (in place) and lo;
//   * MMA warp (warp 12): one thread issues, per UMMA_K = 8 step,
//     tcgen05.mma.cta_group::1.kind::tf32 for hi*hi, lo*hi, hi*lo into one fp32
//     accumulator in TMEM (128 lanes x 128 columns); tcgen05.commit frees the
//     stage (smem + its TMEM A slot) and, separately, the lo tile;
//   * epilogue (split warpgroups; warp w reads TMEM lane quarter w%4, columns
//     64h..64h+63 for warpgroup h): tcgen05.ld 32x32b -> C += acc through the C
//     offset tables, or the split-K partial (transposed, coalesced) into the
//     workspace.
// Shared memory traffic per k-block: 16 KB loaded, 16 KB read by the split,
// 8 KB of B' lo written, 24 KB of B' read by the MMAs.
// Accuracy: each product misses lo*lo and lo's own truncation (< 2^-19
// relative), fp32 accumulation in TMEM; checked against the fp64 oracle and
// the reference (tests/).
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <type_traits>

#include "device.cuh"
#include "kernels.hpp"

// tuning builds only: skip the loads (1), the split (2), the MMAs (4), or B''s
// lo tile and its MMA (8)
#ifndef GETT_TC_ABLATE
#define GETT_TC_ABLATE 0
#endif
#ifndef GETT_TC_STAGES
#define GETT_TC_STAGES 8
#endif
#ifndef GETT_TC_LO
#define GETT_TC_LO 3
#endif

namespace gett {
namespace tc {

// accumulator bits, or -0.0 (the additive identity) when the CTA had no k-blocks
__device__ __forceinline__ uint32_t r_or_zero(uint32_t r, int nkb) { return nkb > 0 ? r : 0x80000000u; }

// Optional per-role cycle accounting (tuning builds only: make variant
// EXTRA=-DGETT_TC_TRACE); blocks 0 and gridDim.x-1 printf their totals.
#ifdef GETT_TC_TRACE
#define TR_DECL(...) long long __VA_ARGS__;
#define TR_T0() long long _tr0 = clock64();
#define TR_ADD(v) { long long _tr1 = clock64(); v += _tr1 - _tr0; _tr0 = _tr1; }
#define TR_PRINT(...) do { if (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) printf(__VA_ARGS__); } while (0)
#else
#define TR_DECL(...)
#define TR_T0()
#define TR_ADD(v)
#define TR_PRINT(...) do { } while (0)
#endif

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int BK = 16;
constexpr int CH = BK / 4;                     // 16-byte k-chunks per row
constexpr int STAGES = GETT_TC_STAGES;
constexpr int WG = 128;                        // threads per warpgroup
constexpr int SPLIT = 2 * WG;                  // split/epilogue threads (two warpgroups)
constexpr int MMA_WARP = (WG + SPLIT) / 32;    // warp 12
constexpr int THREADS = WG + SPLIT + 32;       // producer WG, 2 split/epilogue WGs, MMA warp
constexpr int GROUP_M = 8;
constexpr int LBO = 128;                       // bytes between k-chunks
constexpr int SBO = CH * 128;                  // bytes between 8-row groups
constexpr int TILE_BYTES = 128 * BK * 4;       // one operand part: 8 KB
constexpr int STAGE_BYTES = 2 * TILE_BYTES;    // A fp32 staging, B raw (= B hi)
// B' lo tiles live in a short ring of their own: a stage's raw data must stay
// until its MMAs finish, but lo only from the split to the MMAs, so the loads
// can run STAGES k-blocks ahead with LO_BUFS lo tiles
constexpr int LO_BUFS = GETT_TC_LO;
constexpr int TCAP = 256;                      // outer k-table entries staged in smem
constexpr int BAR_BYTES = 512;
constexpr int LO_OFF = STAGES * STAGE_BYTES;   // lo ring
constexpr int EPI_PITCH = 65;                  // epilogue staging (floats per row)
constexpr int EPI_ROWS = 8;                    // rows in flight per warp in the epilogue
static_assert(2 * BM * EPI_PITCH * 4 <= STAGES * STAGE_BYTES, "epilogue staging fits the stage ring");
constexpr int BAR_OFF = LO_OFF + LO_BUFS * TILE_BYTES;
constexpr int SMEM_BYTES = BAR_OFF + BAR_BYTES + 2 * TCAP * 8;
constexpr uint32_t ACC_COLS = BN;              // fp32 accumulator columns
constexpr uint32_t A_COLS = 2 * BK;            // per stage: A hi (BK cols), A lo (BK cols)
constexpr uint32_t TMEM_COLS = 512;            // power of two >= ACC_COLS + STAGES * A_COLS
static_assert(ACC_COLS + STAGES * A_COLS <= TMEM_COLS, "TMEM budget");
static_assert(3 * STAGES + 2 + LO_BUFS <= BAR_BYTES / 8, "barrier area");
static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");

// instruction descriptor: D f32, A/B tf32, both K-major, N = 128, M = 128
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);
__device__ __forceinline__ uint32_t toff(int r, int c) {
  return (uint32_t)((r >> 3) * SBO + c * LBO + (r & 7) * 16);
}

// shared-memory matrix descriptor (sm_100: version 1 at bit 46), no swizzle
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo = LBO, uint32_t sbo = SBO) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(lbo >> 4) << 16) |
         ((uint64_t)(sbo >> 4) << 32) | (1ull << 46);
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

// A from TMEM (lane = row, 32-bit column = k), B from shared memory
__device__ __forceinline__ void mma_tf32_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(IDESC), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

// 3xTF32 split with the tensor core's own rounding: kind::tf32 reads the top
// 19 bits of a 32-bit operand (truncation, tools/tf32_trunc_test.cu), so a raw
// fp32 value IS its hi part and only lo = x - trunc_tf32(x) (exact in fp32)
// has to be produced.  hi*hi + lo*hi + hi*lo then misses lo*lo and lo's own
// truncation: < 2^-19 relative per product (accuracy checked in tests/).
__device__ __forceinline__ float tf32_lo(float x) {
  return x - __uint_as_float(__float_as_uint(x) & 0xffffe000u);
}
// Mixed split (tools/umma_mixed_test.cu; MIX kernels): per 8 k one tf32 MMA
// hi * hi plus ONE kind::f16 (bf16) MMA whose 16 k are [bf16(x) | bf16(x_lo)]
// against [bf16(y_lo) ; bf16(y)] — both cross terms at the bf16 rate, two MMAs
// per 8 k instead of three, at least as accurate as the truncation split.
// hi = x rounded to tf32 where the split writes it (TMEM A', transposed B'),
// the raw value (truncated by the tensor core) where a landed tile is used in
// place; lo = x - hi exactly either way.
__device__ __forceinline__ float tf32_rn(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}
__device__ __forceinline__ uint32_t bf16x2(float a, float b) {  // a in the low half (the first k)
  const __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&v);
}

// cp.async with zero fill: sz = 0 writes zeros and reads nothing (the source
// address is still kept inside the view)
__device__ __forceinline__ void cp_async_16z(uint32_t dst, const void* src, uint32_t sz) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(sz));
}
__device__ __forceinline__ void cp_async_4z(uint32_t dst, const void* src, uint32_t sz) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(sz));
}

// k-group decoder for both operands: offset_t(k) = T_t[k / e_in] + (k % e_in)
// * s_t, in bytes.  The CTA's slice of the outer tables is staged in shared
// memory when it fits (STAGED), else read from global memory.
struct KDec {
  const int64_t* T[2];  // global outer tables (element offsets)
  uint32_t Ts[2];       // shared-memory addresses of the staged slices (bytes)
  int q0;               // first staged entry
  int64_t s[2];         // inner strides, bytes
  FastDiv div;
};

// Lane-parallel k offsets for one k-block: lane l looks up operand l/16 at
// k = k0 + l%16 (0 past kend), so a warp decodes all 2 x BK offsets of the
// k-block with one divmod + one table load per lane; the gathers then take the
// ones they need with shuffles (kofs).
template <bool STAGED>
__device__ __forceinline__ int64_t klane(const KDec& kd, int k0, int kend, int lane) {
  const int t = lane >> 4, k = k0 + (lane & 15);
  if (k >= kend) return 0;
  int q, r;
  kd.div.divmod(k, q, r);
  int64_t tb;
  if (STAGED) {
    const uint32_t a = (t ? kd.Ts[1] : kd.Ts[0]) + 8u * (uint32_t)(q - kd.q0);
    asm volatile("ld.shared.s64 %0, [%1];" : "=l"(tb) : "r"(a));
  } else {
    tb = __ldg((t ? kd.T[1] : kd.T[0]) + q) * 4;
  }
  return tb + (int64_t)r * (t ? kd.s[1] : kd.s[0]);
}
static_assert(BK == 16, "klane covers 16 k per operand");

// offset of operand t at k-block-relative k (0..15) from the klane values
__device__ __forceinline__ int64_t kofs(int64_t v, int t, int kk) {
  return __shfl_sync(0xffffffffu, v, 16 * t + kk);
}

// One operand's 128-row x BK gather with cp.async by the producer warpgroup.
// Warp w owns row groups 4w..4w+3 (8 rows each).  One warp instruction covers
// 8 consecutive rows x 4 k: lane l -> row 8g + l%8 and, for 16-byte copies
// (VEC: 4 contiguous k per row), chunk l/8 (8 rows x 64 B of gmem, four
// conflict-free 128 B smem wavefronts); for 4-byte copies, k = 4c + l/8 of
// chunk c (32 distinct smem banks; 8 rows x 4 k of gmem).  Row base pointers
// are decoded once per tile; a copy is one 64-bit add + cp.async (zero fill
// for rows past the view and the K tail).
template <bool VEC>
struct Gather {
  const char* rp[4];
  uint32_t rsz[4];  // copy size for the row (0 past the view)
  uint32_t dst0;    // this thread's unit in a tile (bytes)
  int le;
  int64_t ko[2][VEC ? 1 : CH];  // k offsets (bytes; 0 in the K tail) ...
  uint32_t km[2][VEC ? 1 : CH];  // ... and copy-size masks (0 in the K tail)

  __device__ __forceinline__ void setup(int warp, int lane, const GroupDev& g, const float* base,
                                        int base_row, int nrows) {
    const int lr = lane & 7;
    le = lane >> 3;
    const char* r0 = reinterpret_cast<const char*>(base + g.off(0, 0));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int r = base_row + 8 * (4 * warp + i) + lr;
      const bool ok = r < nrows;
      rp[i] = ok ? reinterpret_cast<const char*>(base + g.off(0, r)) : r0;
      rsz[i] = ok ? (VEC ? 16u : 4u) : 0u;
    }
    dst0 = toff(8 * (4 * warp) + lr, VEC ? le : 0) + (VEC ? 0 : 4 * le);
  }

  // take this k-block's offsets of operand t from the warp's klane values
  template <int P>
  __device__ __forceinline__ void prep(int64_t kl, int t, int k0, int kend) {
    if (VEC) {
      ko[P][0] = kofs(kl, t, 4 * le);
      km[P][0] = k0 + 4 * le < kend ? ~0u : 0u;
    } else {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        ko[P][c] = kofs(kl, t, 4 * c + le);
        km[P][c] = k0 + 4 * c + le < kend ? ~0u : 0u;
      }
    }
  }

  template <int P>
  __device__ __forceinline__ void issue(uint32_t s) {
    // row group i is 8 rows = SBO bytes further on
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (VEC) {
        cp_async_16z(s + dst0 + i * SBO, rp[i] + ko[P][0], rsz[i] & km[P][0]);
      } else {
#pragma unroll
        for (int c = 0; c < CH; ++c)
          cp_async_4z(s + dst0 + i * SBO + c * LBO, rp[i] + ko[P][c], rsz[i] & km[P][c]);
      }
    }
  }
};

// Rows-contiguous operand with 16-byte row chunks (unit-stride inner row mode,
// extent and all offsets divisible by 4): staged MN-major, [k][128 rows] fp32
// (512 B per k), and transposed by the split warpgroup (split_a_tmem /
// split_tile_rv) — the tf32 UMMA reads K-major only.  Warp w, instruction i
// copies k = 4w + i: lane l -> rows 4l..4l+3, so one warp instruction moves
// 512 contiguous bytes of gmem into 512 contiguous bytes of smem.
struct GatherRV {
  const char* rp;
  uint32_t rsz;
  uint32_t dst0;
  int w;
  int64_t ko[2][4];
  uint32_t km[2][4];

  __device__ __forceinline__ void setup(int warp, int lane, const GroupDev& g, const float* base,
                                        int base_row, int nrows) {
    w = warp;
    const int r = base_row + 4 * lane;
    const bool ok = r < nrows;
    rp = reinterpret_cast<const char*>(base + g.off(0, ok ? r : 0));
    rsz = ok ? 16u : 0u;
    dst0 = (uint32_t)(4 * w * 512 + lane * 16);
  }

  template <int P>
  __device__ __forceinline__ void prep(int64_t kl, int t, int k0, int kend) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      ko[P][i] = kofs(kl, t, 4 * w + i);
      km[P][i] = k0 + 4 * w + i < kend ? ~0u : 0u;
    }
  }

  template <int P>
  __device__ __forceinline__ void issue(uint32_t s) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      cp_async_16z(s + dst0 + i * 512, rp + ko[P][i], rsz & km[P][i]);
    }
  }
};

template <bool KF, bool VEC>
struct GatherSel {
  using type = Gather<VEC>;
};
template <>
struct GatherSel<false, true> {
  using type = GatherRV;
};
template <>
struct GatherSel<false, false> {
  using type = Gather<false>;
};

// The split warpgroups take alternate k-blocks: warpgroup h (threads tw =
// 0..127 of it, warps wq = 0..3) prepares all of k-block kb = h, h+2, ...

// transpose one MN-major staged tile ([k][row] fp32) into the K-major hi tile
// (same 8 KB, in place: the raw value is the hi part) and the lo tile.  The
// tile is 16 blocks of 4 k x 8 row-chunks; warp wq takes blocks 4wq..4wq+3:
// lane l reads the unit (k = 4kg + l/8, rows 4rc..4rc+3 with rc = 8rcg + l%8)
// — each 8-lane phase reads 128 contiguous bytes.  After a barrier over the
// warpgroup (the writes land on other threads' inputs) it stores the 4 values
// rotated by s = (l/2)%4, so at each store the 32 lanes cover all 8 (row % 8)
// x 4 (k % 4) positions = 32 distinct banks.
__device__ __forceinline__ void split_tile_rv(uint8_t* hi_s, uint8_t* lo_s, int tw, int h) {
  constexpr int NB = 4;
  const int wq = tw >> 5, l = tw & 31;
  float4 x[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const int b = wq * NB + i, k = 4 * (b >> 2) + (l >> 3), rc = 8 * (b & 3) + (l & 7);
    x[i] = *reinterpret_cast<const float4*>(hi_s + k * 512 + rc * 16);
  }
  asm volatile("bar.sync %0, %1;" ::"r"(1 + h), "n"(WG) : "memory");
  const int rot = (l >> 1) & 3;
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const int b = wq * NB + i, k = 4 * (b >> 2) + (l >> 3), rc = 8 * (b & 3) + (l & 7);
    float hv[4] = {x[i].x, x[i].y, x[i].z, x[i].w};
    // rotate left by rot with selects (no dynamic register indexing)
    if (rot & 1) {
      float th = hv[0];
      hv[0] = hv[1]; hv[1] = hv[2]; hv[2] = hv[3]; hv[3] = th;
    }
    if (rot & 2) {
      float th0 = hv[0], th1 = hv[1];
      hv[0] = hv[2]; hv[1] = hv[3]; hv[2] = th0; hv[3] = th1;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int row = 4 * rc + ((j + rot) & 3);
      const uint32_t o = toff(row, k >> 2) + (k & 3) * 4;
      *reinterpret_cast<float*>(hi_s + o) = hv[j];
      *reinterpret_cast<float*>(lo_s + o) = tf32_lo(hv[j]);
    }
  }
}

// lo part of one landed K-major tile (8 KB; the tile itself is the hi part):
// 512 dense 16-byte units, thread tw handles units tw + 128 i (consecutive
// threads -> consecutive 16 B: conflict-free); layout-agnostic
__device__ __forceinline__ void split_tile(const uint8_t* hi_s, uint8_t* lo_s, int tw) {
#pragma unroll
  for (int i = 0; i < 512 / WG; ++i) {
    const uint32_t o = (uint32_t)(tw + WG * i) * 16;
    const float4 x = *reinterpret_cast<const float4*>(hi_s + o);
    *reinterpret_cast<float4*>(lo_s + o) =
        make_float4(tf32_lo(x.x), tf32_lo(x.y), tf32_lo(x.z), tf32_lo(x.w));
  }
}

// byte offset of (row r, 16-byte k chunk c = k / 4) in one SWIZZLE_64B box of
// 128 rows x 16 floats: row r's 64 B at 64 r, its chunk index XORed with
// (r >> 1) & 3 (address bits 4-5 ^ bits 7-8) — the TMA SW64 write pattern and
// the UMMA K-major SW64 layout
__device__ __forceinline__ uint32_t sw64_off(int r, int c) {
  return (uint32_t)(r * 64 + ((c ^ (r >> 1)) & 3) * 16);
}
// SWIZZLE_64B K-major descriptor: SBO 512 B (8 rows x 64 B), LBO unused; the
// 8-k steps of a box start 32 B apart (the swizzle applies to absolute
// shared-memory address bits, the box is 512 B aligned)
__device__ __forceinline__ uint64_t sdesc_sw64(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         (1ull << 46) | (4ull << 61);
}

// MIX, K-major B' landed as ONE SW64 box [16 k][128 rows]: the box stays the
// tf32 hi operand; the bf16 tile is written in the SW32 geometry of
// split_tile_mix (one 4 KB box per 8-k step).  Thread tw takes row tw; a
// quarter warp's reads of one logical chunk cover 8 distinct 16-byte bank
// groups (4 (r & 1) + (c ^ (r >> 1) & 3)).
__device__ __forceinline__ void split_tile_mix64(const uint8_t* hi_s, uint8_t* lo_s, int tw) {
  const uint32_t sw = (uint32_t)((tw >> 2) & 1) << 4;
#pragma unroll
  for (int j = 0; j < BK / 8; ++j) {
    const float4 a = *reinterpret_cast<const float4*>(hi_s + sw64_off(tw, 2 * j));      // k 0-3 of the step
    const float4 b = *reinterpret_cast<const float4*>(hi_s + sw64_off(tw, 2 * j + 1));  // k 4-7
    const uint4 yl = make_uint4(bf16x2(tf32_lo(a.x), tf32_lo(a.y)), bf16x2(tf32_lo(a.z), tf32_lo(a.w)),
                                bf16x2(tf32_lo(b.x), tf32_lo(b.y)), bf16x2(tf32_lo(b.z), tf32_lo(b.w)));
    const uint4 yy = make_uint4(bf16x2(a.x, a.y), bf16x2(a.z, a.w), bf16x2(b.x, b.y), bf16x2(b.z, b.w));
    const uint32_t o = 4096u * j + 32u * tw;
    *reinterpret_cast<uint4*>(lo_s + o + sw) = yl;
    *reinterpret_cast<uint4*>(lo_s + o + (sw ^ 16)) = yy;
  }
}

// MIX, K-major B' landed as two TMA SW32 boxes (k 0-7, k 8-15; row r's 32 B at
// 32 r, its two 16-byte halves exchanged when (r >> 2) is odd): the boxes stay
// the tf32 hi operand (truncated by the tensor core); the second tile gets, in
// the same SW32 geometry, row r's bf16 operand [bf16(y_lo) x 8 | bf16(y) x 8].
// Thread tw takes row tw of both boxes; reading / writing the logical first
// half first makes a quarter warp cover 8 distinct 16-byte bank groups.
__device__ __forceinline__ void split_tile_mix(const uint8_t* hi_s, uint8_t* lo_s, int tw) {
  const uint32_t sw = (uint32_t)((tw >> 2) & 1) << 4;
#pragma unroll
  for (int j = 0; j < BK / 8; ++j) {
    const uint32_t o = 4096u * j + 32u * tw;
    const float4 a = *reinterpret_cast<const float4*>(hi_s + o + sw);         // k 0-3 of the step
    const float4 b = *reinterpret_cast<const float4*>(hi_s + o + (sw ^ 16));  // k 4-7
    const uint4 yl = make_uint4(bf16x2(tf32_lo(a.x), tf32_lo(a.y)), bf16x2(tf32_lo(a.z), tf32_lo(a.w)),
                                bf16x2(tf32_lo(b.x), tf32_lo(b.y)), bf16x2(tf32_lo(b.z), tf32_lo(b.w)));
    const uint4 yy = make_uint4(bf16x2(a.x, a.y), bf16x2(a.z, a.w), bf16x2(b.x, b.y), bf16x2(b.z, b.w));
    *reinterpret_cast<uint4*>(lo_s + o + sw) = yl;
    *reinterpret_cast<uint4*>(lo_s + o + (sw ^ 16)) = yy;
  }
}

// MIX, rows-major B' staged [k][row]: thread tw takes one 4-k x 4-row unit
// (chunk c of 4 k, row quad rq; lanes l and l ^ 8 hold the two chunks of one
// 8-k step), transposes it in registers, and after the warpgroup barrier (the
// K-major hi tile overwrites the staged tile) stores per row the 16-byte chunk
// of tf32-rounded hi values and — after exchanging halves with its partner — a
// whole 16-byte bf16 chunk: the even chunk's lane the y_lo chunk, the odd
// one's the y chunk; stores rotated by the row quad (conflict-free).
__device__ __forceinline__ void split_tile_rv_mix(uint8_t* hi_s, uint8_t* lo_s, int tw, int h) {
  const int e = (tw >> 3) & 1, pp = ((tw >> 4) << 3) | (tw & 7);
  const int c = 2 * (pp >> 5) + e, rq = pp & 31;
  float4 v[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) v[j] = *reinterpret_cast<const float4*>(hi_s + (4 * c + j) * 512 + rq * 16);
  asm volatile("bar.sync %0, %1;" ::"r"(1 + h), "n"(WG) : "memory");
  float4 rows[4];
  rows[0] = make_float4(v[0].x, v[1].x, v[2].x, v[3].x);
  rows[1] = make_float4(v[0].y, v[1].y, v[2].y, v[3].y);
  rows[2] = make_float4(v[0].z, v[1].z, v[2].z, v[3].z);
  rows[3] = make_float4(v[0].w, v[1].w, v[2].w, v[3].w);
  const bool odd = e != 0;
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
  const int rot = (rq >> 1) & 3;
#pragma unroll
  for (int q4 = 0; q4 < 4; ++q4) {
    const int r4 = (q4 + rot) & 3;
    float4 rw = rows[0];
    uint2 m2 = mine[0], o2 = other[0];
    rw = r4 == 1 ? rows[1] : rw;
    m2 = r4 == 1 ? mine[1] : m2;
    o2 = r4 == 1 ? other[1] : o2;
    rw = r4 == 2 ? rows[2] : rw;
    m2 = r4 == 2 ? mine[2] : m2;
    o2 = r4 == 2 ? other[2] : o2;
    rw = r4 == 3 ? rows[3] : rw;
    m2 = r4 == 3 ? mine[3] : m2;
    o2 = r4 == 3 ? other[3] : o2;
    const uint32_t o = toff(4 * rq + r4, c);
    *reinterpret_cast<float4*>(hi_s + o) = rw;
    *reinterpret_cast<uint4*>(lo_s + o) = odd ? make_uint4(o2.x, o2.y, m2.x, m2.y) : make_uint4(m2.x, m2.y, o2.x, o2.y);
  }
}

// byte offset of (row r, k) in one SWIZZLE_32B box of 128 rows x 8 floats
// (the TMA SW32 write pattern = the UMMA K-major SW32 layout; checked by
// tools/umma_tma_test.cu)
__device__ __forceinline__ uint32_t sw32_off(int r, int k) {
  return (uint32_t)(r * 32 + ((((k >> 2) ^ (r >> 2)) & 1) << 4) + (k & 3) * 4);
}

// A' k-block -> TMEM: thread (warp wq of the warpgroup, lane l) owns row
// 32 wq + l (TMEM lane quarter wq = warp % 4) and all BK k of the k-block,
// read from the staging tile — LAYOUT 0: K-major no-swizzle core matrices (4
// 16-byte chunks), 1: [k][row] (16 words, consecutive lanes on consecutive
// words), 2: two TMA SW32 boxes, 3: one TMA SW64 box — and writes the raw values (hi) and lo with
// tcgen05.st into the stage's A columns.
template <int LAYOUT, bool MIX = false>
__device__ __forceinline__ void split_a_tmem(const uint8_t* st, uint32_t tmem, uint32_t col, int wq,
                                             int lane) {
  const int row = 32 * wq + lane;
  float v[BK];
  if (LAYOUT == 1) {
#pragma unroll
    for (int i = 0; i < BK; ++i) v[i] = *reinterpret_cast<const float*>(st + i * 512 + row * 4);
  } else {
#pragma unroll
    for (int c = 0; c < BK / 4; ++c) {
      const uint32_t o = LAYOUT == 0   ? toff(row, c)
                         : LAYOUT == 3 ? sw64_off(row, c)
                                       : 4096 * (c >> 1) + sw32_off(row, 4 * (c & 1));
      const float4 x = *reinterpret_cast<const float4*>(st + o);
      v[4 * c] = x.x; v[4 * c + 1] = x.y; v[4 * c + 2] = x.z; v[4 * c + 3] = x.w;
    }
  }
  uint32_t hi[BK], lo[BK];
  if (MIX) {
    // lo columns of 8-k step g: 8g + (0..3) bf16(x) pairs, 8g + (4..7) bf16(x_lo) pairs
    float xl[BK];
#pragma unroll
    for (int i = 0; i < BK; ++i) {
      const float xh = tf32_rn(v[i]);
      hi[i] = __float_as_uint(xh);
      xl[i] = v[i] - xh;
    }
#pragma unroll
    for (int g = 0; g < BK / 8; ++g)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        lo[8 * g + i] = bf16x2(v[8 * g + 2 * i], v[8 * g + 2 * i + 1]);
        lo[8 * g + 4 + i] = bf16x2(xl[8 * g + 2 * i], xl[8 * g + 2 * i + 1]);
      }
  } else {
#pragma unroll
    for (int i = 0; i < BK; ++i) {
      hi[i] = __float_as_uint(v[i]);
      lo[i] = __float_as_uint(tf32_lo(v[i]));
    }
  }
  const uint32_t ta = tmem + ((uint32_t)(32 * wq) << 16) + col;
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
      "r"(hi[0]), "r"(hi[1]), "r"(hi[2]), "r"(hi[3]), "r"(hi[4]), "r"(hi[5]), "r"(hi[6]), "r"(hi[7]),
      "r"(hi[8]), "r"(hi[9]), "r"(hi[10]), "r"(hi[11]), "r"(hi[12]), "r"(hi[13]), "r"(hi[14]), "r"(hi[15])
      : "memory");
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta + BK),
      "r"(lo[0]), "r"(lo[1]), "r"(lo[2]), "r"(lo[3]), "r"(lo[4]), "r"(lo[5]), "r"(lo[6]), "r"(lo[7]),
      "r"(lo[8]), "r"(lo[9]), "r"(lo[10]), "r"(lo[11]), "r"(lo[12]), "r"(lo[13]), "r"(lo[14]), "r"(lo[15])
      : "memory");
}

// ---- TMA-fed operands (TmaParams, built by the host for affine views) ----

// SWIZZLE_32B K-major descriptor: SBO 256 B (8 rows x 32 B), LBO unused
__device__ __forceinline__ uint64_t sdesc_sw32(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(256 >> 4) << 32) |
         (1ull << 46) | (6ull << 61);
}

// TMA box coordinates of one operand for one producer lane: the tile's row
// coordinates (fixed per CTA) plus the lane's k digits, advanced by a k-block
// (16 k) per step with carries (k_ext[0] is a multiple of 8); no dynamic
// register indexing.
struct TmaCoord {
  int32_t r[5];        // row coordinates
  int32_t d0, d1, d2;  // k digits (inner first)
  int32_t e0, e1, nk, kp0, kp1, kp2;
  __device__ __forceinline__ void init(const TmaOperand& op, int row0, int k) {
#pragma unroll
    for (int i = 0; i < 5; ++i) r[i] = 0;
    int q = row0;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      if (i < op.nr) {
        const int v = q % op.r_ext[i];
        q /= op.r_ext[i];
#pragma unroll
        for (int j = 0; j < 5; ++j)
          if (op.r_pos[i] == j) r[j] = v;
      }
    }
    nk = op.nk;
    e0 = op.k_ext[0];
    e1 = nk > 1 ? op.k_ext[1] : 1;
    kp0 = op.k_pos[0];
    kp1 = nk > 1 ? op.k_pos[1] : -1;
    kp2 = nk > 2 ? op.k_pos[2] : -1;
    d0 = k % e0;
    q = k / e0;
    d1 = q % e1;
    d2 = q / e1;
  }
  __device__ __forceinline__ void step() {
    d0 += BK;
    while (d0 >= e0) {
      d0 -= e0;
      if (++d1 >= e1) {
        d1 = 0;
        ++d2;
      }
    }
  }
  __device__ __forceinline__ void coords(int32_t* c) const {
#pragma unroll
    for (int j = 0; j < 5; ++j)
      c[j] = r[j] + (kp0 == j ? d0 : 0) + (kp1 == j ? d1 : 0) + (kp2 == j ? d2 : 0);
  }
};

__device__ __forceinline__ void tma_load5(uint32_t dst, const CUtensorMap* map, const int32_t* c, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
      "l"(map), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(bar)
      : "memory");
}

template <bool AKF, bool BKF, bool AVEC, bool BVEC, bool TMA>
__global__ void __launch_bounds__(THREADS, 1)
    sgett_tc_kernel(const __grid_constant__ TiledParams<float> p, const __grid_constant__ TmaParams tp) {
  extern __shared__ __align__(1024) uint8_t smem[];
#ifdef GETT_TC_TRACE
  unsigned long long g_entry;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_entry));
  const long long c_entry = clock64();
#endif
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + BAR_OFF);  // gathers landed
  uint64_t* ready = full + STAGES;                               // split done
  uint64_t* empty = ready + STAGES;                              // MMAs done (stage reusable)
  uint64_t* done = empty + STAGES;
  uint64_t* lofree = done + 1;                                   // MMAs done (lo tile reusable)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  int64_t* ktabs = reinterpret_cast<int64_t*>(smem + BAR_OFF + BAR_BYTES);  // [2][TCAP]
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

  // this CTA's slice [q0, q1] of the K group's outer offset tables, staged in
  // shared memory when it fits (c5: 34 of 768 entries)
  // (in bytes)
  KDec kd{{p.gk.T[0], p.gk.T[1]}, {0u, 0u}, 0, {p.gk.s_in[0] * 4, p.gk.s_in[1] * 4}, p.gk.e_in};
  if (TMA) {
    // the boxes' descriptors, fetched while the barriers are set up
    if (tid == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tp.map[0]) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tp.map[1]) : "memory");
    }
  } else if (nkb > 0) {  // (the gathers' k tables; not used by the TMA path)
    const int q0 = kbeg / p.gk.e_in.d, q1 = (kend - 1) / p.gk.e_in.d;
    if (q1 - q0 + 1 <= TCAP) {
      for (int i = tid; i <= q1 - q0; i += THREADS) {
        ktabs[i] = __ldg(p.gk.T[0] + q0 + i) * 4;
        ktabs[TCAP + i] = __ldg(p.gk.T[1] + q0 + i) * 4;
      }
      kd.Ts[0] = smem_u32(ktabs);
      kd.Ts[1] = smem_u32(ktabs + TCAP);
      kd.q0 = q0;
    }
  }
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      // per producer thread: its cp.async group (zero fill included); TMA: the
      // expect_tx arrival of the one issuing thread
      mbar_init(smem_u32(full + s), TMA ? 1 : WG);
      mbar_init(smem_u32(ready + s), 4);  // the 4 warps of the split warpgroup of this k-block
      mbar_init(smem_u32(empty + s), 1);      // tcgen05.commit
    }
    mbar_init(smem_u32(done), 1);
    for (int l = 0; l < LO_BUFS; ++l) mbar_init(smem_u32(lofree + l), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
#ifdef GETT_TC_TRACE
  const long long c_setup = clock64() - c_entry;
#endif
  auto stage = [&](int s) { return smem + s * STAGE_BYTES; };

  if (TMA && warp < 4) {
    // ---------------- producer: lanes 0-3 of warp 0 each issue one TMA box
    // per k-block (A' k 0-7 / 8-15, B' k 0-7 / 8-15); lane 0 posts the bytes
    const int lane = tid & 31;
    if (warp == 0 && lane < 4) {
      const int t = lane >> 1, h = lane & 1;
      TmaCoord cc;
      if (t) cc.init(tp.op[1], n0, kbeg + 8 * h);
      else cc.init(tp.op[0], m0, kbeg + 8 * h);
      const CUtensorMap* map = t ? &tp.map[1] : &tp.map[0];
      const uint32_t dst0 = smem_u32(smem) + t * TILE_BYTES + 4096 * h;
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES, u = kb / STAGES;
        if (u > 0) mbar_wait(smem_u32(empty + s), (u - 1) & 1);
        const uint32_t fb = smem_u32(full + s);
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(2 * TILE_BYTES)
                       : "memory");
        int32_t c[5];
        cc.coords(c);
        tma_load5(dst0 + s * STAGE_BYTES, map, c, fb);
        cc.step();
      }
    }
  } else if (warp < 4) {
    // ---------------- producer warpgroup ----------------
    typename GatherSel<AKF, AVEC>::type ga;
    typename GatherSel<BKF, BVEC>::type gb;
    ga.setup(warp, tid & 31, p.gm, p.A, m0, p.M);
    gb.setup(warp, tid & 31, p.gn, p.B, n0, p.N);
    const uint32_t sbase = smem_u32(smem);
    TR_DECL(tp = 0, tw = 0, ti = 0)
    TR_T0()
    const int lane = tid & 31;
    // k offsets run one k-block ahead of the copies (two register sets, loop
    // unrolled by 2), so the k-table lookups never sit on the issue path
    auto run = [&](auto staged) {
      constexpr bool ST = decltype(staged)::value;
      auto prep = [&](auto par, int k0) {
        constexpr int P = decltype(par)::value;
        const int64_t kl = klane<ST>(kd, k0, kend, lane);
        ga.template prep<P>(kl, 0, k0, kend);
        gb.template prep<P>(kl, 1, k0, kend);
      };
      auto step = [&](auto par, int kb) {
        constexpr int P = decltype(par)::value;
        const int s = kb % STAGES, u = kb / STAGES;
        const int k0 = kbeg + kb * BK;
        if (u > 0) mbar_wait(smem_u32(empty + s), (u - 1) & 1);
        TR_ADD(tw)
        if (!(GETT_TC_ABLATE & 1)) {
          ga.template issue<P>(sbase + s * STAGE_BYTES);
          gb.template issue<P>(sbase + s * STAGE_BYTES + TILE_BYTES);
        }
        mbar_arrive_cpasync(smem_u32(full + s));
        TR_ADD(ti)
        prep(par, k0 + 2 * BK);
        TR_ADD(tp)
      };
      prep(std::integral_constant<int, 0>{}, kbeg);
      prep(std::integral_constant<int, 1>{}, kbeg + BK);
      for (int kb = 0; kb < nkb; kb += 2) {
        step(std::integral_constant<int, 0>{}, kb);
        if (kb + 1 < nkb) step(std::integral_constant<int, 1>{}, kb + 1);
      }
    };
    if (kd.Ts[0]) run(std::true_type{});
    else run(std::false_type{});
    cp_async_wait<0>();
    if (tid == 0) TR_PRINT("blk %d producer: prep %lld wait_empty %lld issue %lld (nkb %d)\n", blockIdx.x, tp, tw, ti, nkb);
  } else if (warp < MMA_WARP) {
    // ---------------- split warpgroup, then epilogue ----------------
    const int h = (warp - 4) >> 2, wq = warp & 3, tw = (tid - WG) & (WG - 1), lane = tid & 31;
    TR_DECL(tw_ = 0, tsp = 0, te = 0)
    TR_T0()
    constexpr int ALAY = TMA ? (AKF ? 2 : 1) : ((!AKF && AVEC) ? 1 : 0);
    constexpr bool BRV = TMA ? !BKF : (!BKF && BVEC);
    for (int kb = h; kb < nkb; kb += 2) {
      const int s = kb % STAGES, u = kb / STAGES;
      mbar_wait(smem_u32(full + s), u & 1);
      TR_ADD(tw_)
      uint8_t* st = stage(s);
      // the lo tile of k-block kb: free once the MMAs of kb - LO_BUFS are done
      const int lb = kb % LO_BUFS, lu = kb / LO_BUFS;
      if (lu > 0) mbar_wait(smem_u32(lofree + lb), (lu - 1) & 1);
      uint8_t* lo = smem + LO_OFF + lb * TILE_BYTES;
      if (!(GETT_TC_ABLATE & 2)) {
        split_a_tmem<ALAY>(st, tmem, ACC_COLS + s * A_COLS, wq, lane);
        if (BRV) split_tile_rv(st + TILE_BYTES, lo, tw, h);
        else if (!(GETT_TC_ABLATE & 8)) split_tile(st + TILE_BYTES, lo, tw);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(ready + s));
      TR_ADD(tsp)
    }
    if (nkb > 0) mbar_wait(smem_u32(done), 0);
    // the split-K reduce (a programmatic dependent launch) may be scheduled now
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    TR_DECL(twd = 0)
    TR_ADD(twd)
    // warp w may only read TMEM lanes 32(w%4)..32(w%4)+31: thread owns accumulator
    // row 32(w%4) + lane, and split warpgroup h = (w-4)/4 takes columns 64h..64h+63
    const int lane_row = 32 * (warp & 3) + (tid & 31);
    const int cbeg = 64 * ((warp - 4) >> 2);
    const int m = m0 + lane_row;
    const bool mok = m < p.M;
    // split-K partials, transposed [split][N][M]: a warp's 32 rows are 32
    // consecutive floats per column (coalesced); the reduce reads it m-fastest
    float* wcol = p.splits > 1 ? p.ws + (int64_t)split * p.M * p.N + (mok ? m : 0) : nullptr;
    // all 64 of this thread's columns leave TMEM before one wait (the loads
    // pipeline instead of paying the TMEM latency per 16 columns)
    uint32_t rr[64];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(cbeg + 16 * q);
      uint32_t* r = rr + 16 * q;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
            "=r"(r[14]), "=r"(r[15])
          : "r"(taddr));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (p.splits == 1) {
      // C += acc through shared memory: the planner puts C's smallest stride in
      // N, so a thread-per-row store would touch 32 lines per warp instruction.
      // Each warpgroup stages its 128 x 64 block (pitch 65: conflict-free both
      // ways) in the idle stage ring; then lane l of a warp owns columns l and
      // 32 + l of every 4th row, so each warp load / store covers 32
      // consecutive n.
      float* tb = reinterpret_cast<float*>(smem) + h * (BM * EPI_PITCH);
#pragma unroll
      for (int i = 0; i < 64; ++i) tb[lane_row * EPI_PITCH + i] = __uint_as_float(r_or_zero(rr[i], nkb));
      asm volatile("bar.sync %0, %1;" ::"r"(1 + h), "r"(WG) : "memory");
      int64_t con[2];
      bool nok[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int n = n0 + cbeg + 32 * j + lane;
        nok[j] = n < p.N;
        con[j] = nok[j] ? p.gn.off(1, n) : 0;
      }
      for (int r0 = wq; r0 < BM; r0 += 4 * EPI_ROWS) {
        float cv[EPI_ROWS][2];
        int64_t co[EPI_ROWS][2];
#pragma unroll
        for (int t = 0; t < EPI_ROWS; ++t) {
          const int r = r0 + 4 * t, mm = m0 + r;
          const bool rok = mm < p.M;
          const int64_t rof = rok ? p.gm.off(1, mm) : 0;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            co[t][j] = rof + con[j];
            cv[t][j] = (rok && nok[j]) ? p.C[co[t][j]] : 0.f;
          }
        }
#pragma unroll
        for (int t = 0; t < EPI_ROWS; ++t) {
          const int r = r0 + 4 * t;
          if (m0 + r >= p.M) continue;
#pragma unroll
          for (int j = 0; j < 2; ++j)
            if (nok[j]) p.C[co[t][j]] = epi(cv[t][j], tb[r * EPI_PITCH + 32 * j + lane], p.neg);
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c0 = cbeg + 16 * q;
        const uint32_t* r = rr + 16 * q;
        if (!mok) continue;
        // split-K partials, m-fastest: a warp's 32 rows are 32 consecutive floats
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int n = n0 + c0 + i;
          if (n < p.N) wcol[(int64_t)n * p.M] = nkb > 0 ? __uint_as_float(r[i]) : -0.0f;
        }
      }
    }
    TR_ADD(te)
    if (tid == WG) TR_PRINT("blk %d split: wait_full %lld split %lld wait_done %lld epilogue %lld\n", blockIdx.x, tw_, tsp, twd, te);
  } else {
    // ---------------- MMA warp ----------------
    if ((tid & 31) == 0) {
      const uint32_t smem_base = smem_u32(smem);
      TR_DECL(tw = 0, tm = 0)
      TR_T0()
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES, u = kb / STAGES;
        mbar_wait(smem_u32(ready + s), u & 1);
        TR_ADD(tw)
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t sb = smem_base + s * STAGE_BYTES;
        const uint32_t lob = smem_base + LO_OFF + (kb % LO_BUFS) * TILE_BYTES;
#pragma unroll
        for (int j = 0; j < BK / 8; ++j) {
          // k-step j: B' K-major tiles advance 256 B (2 k-chunks), A' 8 TMEM columns
          const uint32_t ah = tmem + ACC_COLS + s * A_COLS + 8 * j, al = ah + BK;
          // B' K-major tiles: no-swizzle core matrices (k-step = 256 B), or the
          // TMA SW32 boxes (k-step = one 4 KB box)
          constexpr bool SW = TMA && BKF;
          const uint64_t bh = SW ? sdesc_sw32(sb + TILE_BYTES + 4096 * j) : sdesc(sb + TILE_BYTES + 256 * j);
          const uint64_t bl = SW ? sdesc_sw32(lob + 4096 * j) : sdesc(lob + 256 * j);
          if (GETT_TC_ABLATE & 4) continue;
          mma_tf32_ta(tmem, ah, bh, (kb | j) != 0);  // first MMA of the tile overwrites D
          mma_tf32_ta(tmem, al, bh, 1);
          if (!(GETT_TC_ABLATE & 8)) mma_tf32_ta(tmem, ah, bl, 1);
        }
        commit(smem_u32(empty + s));
        commit(smem_u32(lofree + kb % LO_BUFS));
        TR_ADD(tm)
      }
      commit(smem_u32(done));
      TR_PRINT("blk %d mma: wait_ready %lld issue %lld\n", blockIdx.x, tw, tm);
    }
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == MMA_WARP)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
#ifdef GETT_TC_TRACE
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1)) {
    unsigned long long g_exit;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_exit));
    printf("blk %d entry_ns %llu setup %lld life %lld clk %llu ns\n", blockIdx.x, g_entry, c_setup,
           clock64() - c_entry, g_exit - g_entry);
  }
#endif
}


// ---------------------------------------------------------------------------
// CTA-pair variant (tcgen05.mma.cta_group::2, M = 256 per pair): for a
// K-major A' (TMA SW32 boxes, split into each CTA's TMEM: rows 128r..128r+127
// of the pair's 256) and a rows-major B' of at most 128 rows (one n-tile),
// split across the pair N-wise — CTA r holds rows NBH*r..NBH*r+NBH-1 of B' in
// its own shared memory (tools/umma_2cta_test.cu: B is split N-wise, A comes
// from each CTA's TMEM).  Halves B' traffic per SM and removes the M padding
// of a narrow N (c5: M' = 768 orig-A rows, N' = 96 orig-B rows).  Both CTAs
// load and split their own parts; their split warps arrive on the leader's
// ready barrier (cluster scope); the leader's MMA thread issues the pair MMAs
// and multicasts each commit to both CTAs' barriers.
namespace pair {
#ifndef GETT_PAIR_STAGES
#define GETT_PAIR_STAGES 12
#endif
constexpr int STAGES2 = GETT_PAIR_STAGES;
constexpr int NBH_MAX = 64;                        // B' rows per CTA
constexpr int A_BYTES = 128 * BK * 4;              // 8 KB: two SW32 boxes
constexpr int BRAW_BYTES = NBH_MAX * BK * 4;       // 4 KB: [16 k][NBH rows]
constexpr int STAGE2_BYTES = A_BYTES + BRAW_BYTES;
constexpr int BT_BYTES = NBH_MAX * BK * 4;         // one K-major B' hi or lo tile
constexpr int BHI_OFF = STAGES2 * STAGE2_BYTES;
constexpr int BLO_OFF = BHI_OFF + LO_BUFS * BT_BYTES;
constexpr int BAR2_OFF = BLO_OFF + LO_BUFS * BT_BYTES;
constexpr int SMEM2_BYTES = BAR2_OFF + 512;
static_assert(ACC_COLS + STAGES2 * A_COLS <= TMEM_COLS, "TMEM budget");
static_assert(3 * STAGES2 + 1 + LO_BUFS <= 512 / 8, "barrier area");
constexpr int SBO64 = CH * 128;                    // 8-row groups, K-major no-swizzle

__device__ __forceinline__ void arrive_leader(uint32_t local_bar) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(local_bar));
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t"
      "}" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mma_pair(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                         uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_pair_bf16(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                              uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc)
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

// raw [16 k][nbh rows] (TMA) -> K-major hi (raw) and lo tiles, 64-row capacity
__device__ __forceinline__ void split_b_pair(const uint8_t* raw, uint8_t* hi, uint8_t* lo, int nbh, int tw) {
  for (int u = tw; u < nbh * CH; u += WG) {
    const int c = u / nbh, row = u - c * nbh;
    float4 x;
    x.x = *reinterpret_cast<const float*>(raw + (4 * c + 0) * nbh * 4 + row * 4);
    x.y = *reinterpret_cast<const float*>(raw + (4 * c + 1) * nbh * 4 + row * 4);
    x.z = *reinterpret_cast<const float*>(raw + (4 * c + 2) * nbh * 4 + row * 4);
    x.w = *reinterpret_cast<const float*>(raw + (4 * c + 3) * nbh * 4 + row * 4);
    const uint32_t o = (uint32_t)((row >> 3) * SBO64 + c * LBO + (row & 7) * 16);
    *reinterpret_cast<float4*>(hi + o) = x;
    *reinterpret_cast<float4*>(lo + o) = make_float4(tf32_lo(x.x), tf32_lo(x.y), tf32_lo(x.z), tf32_lo(x.w));
  }
}

// grid: 2 x pairs x splits (clusters of 2); p.M = A' rows, p.N = 2 * nbh
__global__ void __launch_bounds__(THREADS, 1)
    sgett_tc_pair_kernel(const __grid_constant__ TiledParams<float> p, const __grid_constant__ TmaParams tp) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + BAR2_OFF);
  uint64_t* ready = full + STAGES2;   // leader: 8 warp arrivals (4 per CTA)
  uint64_t* empty = ready + STAGES2;  // pair commit
  uint64_t* done = empty + STAGES2;
  uint64_t* lofree = done + 1;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int npairs = (p.M + 255) / 256;
  const int cl = blockIdx.x >> 1;
  const int pr = cl % npairs, split = cl / npairs;
  const int m0 = pr * 256 + 128 * (int)rank;  // this CTA's A' rows
  const int nbh = p.N / 2;
  const int kbeg = split * p.k_chunk;
  const int kend = min(p.K, kbeg + p.k_chunk);
  const int nkb = kend > kbeg ? (kend - kbeg) / BK : 0;
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tp.map[0]) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tp.map[1]) : "memory");
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(smem_u32(full + s), 1);
      mbar_init(smem_u32(ready + s), 8);
      mbar_init(smem_u32(empty + s), 1);
    }
    mbar_init(smem_u32(done), 1);
    for (int l = 0; l < LO_BUFS; ++l) mbar_init(smem_u32(lofree + l), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync2();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    // producer lanes 0-1: A' boxes (k 0-7, 8-15); lanes 2-3: B' boxes
    if (lane < 4) {
      const int t = lane >> 1, h = lane & 1;
      TmaCoord cc;
      if (t) cc.init(tp.op[1], nbh * (int)rank, kbeg + 8 * h);
      else cc.init(tp.op[0], m0, kbeg + 8 * h);
      const CUtensorMap* map = t ? &tp.map[1] : &tp.map[0];
      const uint32_t dst0 = smem_u32(smem) + (t ? A_BYTES + h * 8 * nbh * 4 : 4096 * h);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES2, u = kb / STAGES2;
        if (u > 0) mbar_wait(smem_u32(empty + s), (u - 1) & 1);
        const uint32_t fb = smem_u32(full + s);
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(A_BYTES + 16 * nbh * 4)
                       : "memory");
        int32_t c[5];
        cc.coords(c);
        tma_load5(dst0 + s * STAGE2_BYTES, map, c, fb);
        cc.step();
      }
    }
  } else if (warp >= 4 && warp < MMA_WARP) {
    // ---------------- split warpgroups (alternate k-blocks), then epilogue ----------------
    const int h = (warp - 4) >> 2, wq = warp & 3, tw = (tid - WG) & (WG - 1);
    for (int kb = h; kb < nkb; kb += 2) {
      const int s = kb % STAGES2, u = kb / STAGES2;
      mbar_wait(smem_u32(full + s), u & 1);
      const int lb = kb % LO_BUFS, lu = kb / LO_BUFS;
      if (lu > 0) mbar_wait(smem_u32(lofree + lb), (lu - 1) & 1);
      const uint8_t* st = smem + s * STAGE2_BYTES;
      if (!(GETT_TC_ABLATE & 2)) {
        split_a_tmem<2>(st, tmem, ACC_COLS + s * A_COLS, wq, lane);
        split_b_pair(st + A_BYTES, smem + BHI_OFF + lb * BT_BYTES, smem + BLO_OFF + lb * BT_BYTES, nbh, tw);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) arrive_leader(smem_u32(ready + s));
    }
    if (nkb > 0) mbar_wait(smem_u32(done), 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // accumulator rows = this CTA's 128 A' rows (lane quarter wq), columns
    // 64h..64h+63 of the 2*nbh
    const int lane_row = 32 * wq + lane;
    const int m = m0 + lane_row;
    const bool mok = m < p.M;
    const int cbeg = 64 * h, cend = min(cbeg + 64, p.N);
    float* wcol = p.ws + (int64_t)split * p.M * p.N + (mok ? m : 0);
    for (int c0 = cbeg; c0 < cend; c0 += 16) {
      uint32_t r[16];
      const uint32_t taddr = tmem + ((uint32_t)(32 * wq) << 16) + (uint32_t)c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (!mok) continue;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int n = c0 + i;
        if (n < p.N) wcol[(int64_t)n * p.M] = nkb > 0 ? __uint_as_float(r[i]) : -0.0f;
      }
    }
  } else if (warp == MMA_WARP && rank == 0) {
    // ---------------- MMA issue (leader CTA) ----------------
    if (lane == 0) {
      const uint32_t base = smem_u32(smem);
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(p.N >> 3) << 17) | ((256u >> 4) << 24);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES2, u = kb / STAGES2;
        mbar_wait_cluster(smem_u32(ready + s), u & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const int lb = kb % LO_BUFS;
        const uint32_t bh0 = base + BHI_OFF + lb * BT_BYTES, bl0 = base + BLO_OFF + lb * BT_BYTES;
#pragma unroll
        for (int j = 0; j < BK / 8; ++j) {
          const uint32_t ah = tmem + ACC_COLS + s * A_COLS + 8 * j, al = ah + BK;
          const uint64_t bh = sdesc(bh0 + 256 * j, LBO, SBO64), bl = sdesc(bl0 + 256 * j, LBO, SBO64);
          if (GETT_TC_ABLATE & 4) continue;
          mma_pair(tmem, ah, bh, idesc, (kb | j) != 0);
          mma_pair(tmem, al, bh, idesc, 1);
          mma_pair(tmem, ah, bl, idesc, 1);
        }
        commit_pair(smem_u32(empty + s));
        commit_pair(smem_u32(lofree + lb));
      }
      commit_pair(smem_u32(done));
    }
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync2();
  if (warp == MMA_WARP)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}
}  // namespace pair

cudaError_t launch_pair(const TiledParams<float>& p, const TmaParams& tp, cudaStream_t s) {
  auto k = pair::sgett_tc_pair_kernel;
  static unsigned long long configured = 0;
  cudaError_t e = ensure_dyn_smem(k, pair::SMEM2_BYTES, configured);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * ((p.M + 255) / 256) * p.splits));
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = pair::SMEM2_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, p, tp);
}

template <bool AKF, bool BKF, bool AV, bool BV, bool TMA>
cudaError_t launch4(const TiledParams<float>& p, const TmaParams& tp, cudaStream_t s) {
  auto k = sgett_tc_kernel<AKF, BKF, AV, BV, TMA>;
  static unsigned long long configured = 0;
  cudaError_t e = ensure_dyn_smem(k, SMEM_BYTES, configured);
  if (e != cudaSuccess) return e;
  k<<<(unsigned)(p.tiles_m * p.tiles_n * p.splits), THREADS, SMEM_BYTES, s>>>(p, tp);
  return cudaGetLastError();
}

template <bool AKF, bool BKF>
cudaError_t launch2(const TiledParams<float>& p, const TmaParams* tp, bool av, bool bv, cudaStream_t s) {
  if (tp) return launch4<AKF, BKF, false, false, true>(p, *tp, s);
  static const TmaParams none{};
  if (av && bv) return launch4<AKF, BKF, true, true, false>(p, none, s);
  if (av) return launch4<AKF, BKF, true, false, false>(p, none, s);
  if (bv) return launch4<AKF, BKF, false, true, false>(p, none, s);
  return launch4<AKF, BKF, false, false, false>(p, none, s);
}


// ---------------------------------------------------------------------------
// Wide CTA-pair variant for large tilings (tcgen05.mma.cta_group::2, a
// 256 x 256 output tile per pair): CTA r of the cluster holds rows
// 128r..128r+127 of the pair's 256 A' rows in its TMEM and rows 128r..128r+127
// of the pair's 256 B' rows in its shared memory; the pair MMA (M = 256, N =
// 256) reads A from each CTA's TMEM and B split N-wise across the two CTAs
// (tools/umma_2cta_test.cu), so every B' byte staged, split and read by the
// tensor core feeds twice the MACs of the single-CTA kernel: per k-block a CTA
// moves the same 16 KB loaded + 16-24 KB split + 24 KB MMA reads as a
// 128 x 128 tile but for 128 x 256 of output, which takes the kernel from the
// shared-memory bound (sgett_tc_kernel at 2048^3: ~500 cycles of smem traffic
// against 384 of MMA per k-block) back under the MMA time.  Loads, split and
// lo ring are those of the single-CTA TMA kernel (same boxes: 128 rows per
// operand per CTA); the split warps of both CTAs arrive on the leader's ready
// barrier, the leader issues the pair MMAs and multicasts each commit.  TMEM:
// a 256-column accumulator + 8 stages x (A hi, A lo).  A CTA whose A' or B'
// rows lie wholly past the view skips that box (a fully out-of-bounds box
// faults) and expects fewer bytes; those accumulator rows / columns are never
// stored.
namespace wide {
constexpr int STAGESW = 8;
constexpr int ACCW = 256;                               // fp32 accumulator columns
constexpr int LO_OFFW = STAGESW * STAGE_BYTES;
constexpr int BAR_OFFW = LO_OFFW + LO_BUFS * TILE_BYTES;
constexpr int SMEMW_BYTES = BAR_OFFW + BAR_BYTES;
static_assert(ACCW + STAGESW * A_COLS <= TMEM_COLS, "TMEM budget");
static_assert(2 * BM * EPI_PITCH * 4 <= STAGESW * STAGE_BYTES, "epilogue staging fits the stage ring");
static_assert(SMEMW_BYTES <= 227 * 1024, "shared memory budget");
// D f32, A/B tf32, K-major, N = 256, M = 256 (the pair)
constexpr uint32_t IDESCW = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(256 >> 3) << 17) |
                            ((uint32_t)(256 >> 4) << 24);
// the same shape for kind::f16 with bf16 operands (format 1)
constexpr uint32_t IDESCW_BF = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) |
                               ((uint32_t)(256 >> 4) << 24);

// grid: 2 x (pair tiles x splits), clusters of 2; p.tiles_m / tiles_n count 256-row pair tiles
// pair tile -> (tm, tn): groups of GROUP_M tile rows, column by column
__device__ __forceinline__ void wide_tile(const TiledParams<float>& p, int tile, int& tm, int& tn) {
  const int per_group = GROUP_M * p.tiles_n;
  const int group = tile / per_group, first_m = group * GROUP_M;
  const int gsize = min(p.tiles_m - first_m, GROUP_M);
  const int in_group = tile % per_group;
  tm = first_m + in_group % gsize;
  tn = in_group / gsize;
}

// MIX: the mixed split (above) — 4 instead of 6 pair MMAs per k-block
// W64: K-major operands arrive as one SWIZZLE_64B box [16 k][128 rows] per
// k-block (half the TMA lines of two SW32 boxes)
template <bool AKF, bool BKF, bool MIX, bool W64>
__global__ void __launch_bounds__(THREADS, 1)
    sgett_tc_wide_kernel(const __grid_constant__ TiledParams<float> p, const __grid_constant__ TmaParams tp) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + BAR_OFFW);  // this CTA's boxes landed
  uint64_t* ready = full + STAGESW;    // leader: 8 split-warp arrivals (4 per CTA)
  uint64_t* empty = ready + STAGESW;   // pair commit (multicast)
  uint64_t* done = empty + STAGESW;
  uint64_t* lofree = done + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(lofree + LO_BUFS);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int ntiles = p.tiles_m * p.tiles_n;
  const int cl = blockIdx.x >> 1;
  // tail split: clusters [0, tail_tile0) run one whole tile each; the rest are
  // the two K halves of the tail tiles (blocks are dispatched in index order,
  // so the halves share the last wave)
  int tile, split;
  bool tail = false;
  if (p.tail_tiles > 0) {
    tail = cl >= p.tail_tile0;
    const int t = cl - p.tail_tile0;
    tile = tail ? p.tail_tile0 + t % p.tail_tiles : cl;
    split = tail ? t / p.tail_tiles : 0;
  } else {
    tile = cl % ntiles;
    split = cl / ntiles;
  }
  int tm, tn;
  wide_tile(p, tile, tm, tn);
  const int m0 = tm * 256 + 128 * (int)rank;  // this CTA's A' rows (accumulator rows)
  const int nb0 = tn * 256;                    // the pair's B' rows (accumulator columns)
  const int n0 = nb0 + 128 * (int)rank;        // this CTA's B' rows
  const bool a_live = m0 < p.M, b_live = n0 < p.N;
  const bool whole = p.tail_tiles > 0 && !tail;  // (a whole-K tile of a tail-split launch)
  const int kbeg = whole ? 0 : split * p.k_chunk;
  const int kend = whole ? p.K : min(p.K, kbeg + p.k_chunk);
  const int nkb = kend > kbeg ? (kend - kbeg) / BK : 0;  // K % 16 == 0 on the TMA path
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tp.map[0]) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tp.map[1]) : "memory");
    for (int s = 0; s < STAGESW; ++s) {
      mbar_init(smem_u32(full + s), 1);
      mbar_init(smem_u32(ready + s), 8);
      mbar_init(smem_u32(empty + s), 1);
    }
    mbar_init(smem_u32(done), 1);
    for (int l = 0; l < LO_BUFS; ++l) mbar_init(smem_u32(lofree + l), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  pair::cluster_sync2();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // producer: lanes 0-1 A' boxes (k 0-7 / 8-15), lanes 2-3 B' boxes
    if (warp == 0 && lane < 4) {
      const int t = lane >> 1, h = lane & 1;
      // (a K-major operand's single 16-k box is issued by the h = 0 lane)
      const bool live = (t ? b_live : a_live) && !(W64 && h == 1 && (t ? BKF : AKF));
      TmaCoord cc;
      if (t) cc.init(tp.op[1], live ? n0 : 0, kbeg + 8 * h);
      else cc.init(tp.op[0], live ? m0 : 0, kbeg + 8 * h);
      const CUtensorMap* map = t ? &tp.map[1] : &tp.map[0];
      const uint32_t dst0 = smem_u32(smem) + t * TILE_BYTES + 4096 * h;
      const uint32_t bytes = (a_live ? TILE_BYTES : 0) + (b_live ? TILE_BYTES : 0);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGESW, u = kb / STAGESW;
        if (u > 0) mbar_wait(smem_u32(empty + s), (u - 1) & 1);
        const uint32_t fb = smem_u32(full + s);
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(bytes) : "memory");
        int32_t c[5];
        cc.coords(c);
        if (live) tma_load5(dst0 + s * STAGE_BYTES, map, c, fb);
        cc.step();
      }
    }
  } else if (warp < MMA_WARP) {
    // ---------------- split warpgroups (alternate k-blocks), then epilogue ----------------
    const int h = (warp - 4) >> 2, wq = warp & 3, tw = (tid - WG) & (WG - 1);
    constexpr int ALAY = AKF ? (W64 ? 3 : 2) : 1;
    for (int kb = h; kb < nkb; kb += 2) {
      const int s = kb % STAGESW, u = kb / STAGESW;
      mbar_wait(smem_u32(full + s), u & 1);
      const int lb = kb % LO_BUFS, lu = kb / LO_BUFS;
      if (lu > 0) mbar_wait(smem_u32(lofree + lb), (lu - 1) & 1);
      uint8_t* st = smem + s * STAGE_BYTES;
      uint8_t* lo = smem + LO_OFFW + lb * TILE_BYTES;
      split_a_tmem<ALAY, MIX>(st, tmem, ACCW + s * A_COLS, wq, lane);
      if (MIX) {
        if (!BKF) split_tile_rv_mix(st + TILE_BYTES, lo, tw, h);
        else if (W64) split_tile_mix64(st + TILE_BYTES, lo, tw);
        else split_tile_mix(st + TILE_BYTES, lo, tw);
      } else {
        if (!BKF) split_tile_rv(st + TILE_BYTES, lo, tw, h);
        else split_tile(st + TILE_BYTES, lo, tw);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) pair::arrive_leader(smem_u32(ready + s));
    }
    if (nkb > 0) mbar_wait(smem_u32(done), 0);
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // thread = accumulator row 32 wq + lane of this CTA; warpgroup h takes
    // columns 128h..128h+127 of the pair's 256, in two halves of 64
    const int lane_row = 32 * wq + lane;
    const int m = m0 + lane_row;
    const bool mok = m < p.M;
    float* tb = reinterpret_cast<float*>(smem) + h * (BM * EPI_PITCH);
    for (int half = 0; half < 2; ++half) {
      const int cbeg = 128 * h + 64 * half;
      uint32_t rr[64];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t taddr = tmem + ((uint32_t)(wq * 32) << 16) + (uint32_t)(cbeg + 16 * q);
        uint32_t* r = rr + 16 * q;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (tail) {
        // compact partials [half][tail tile][256 n][256 m] (m fastest)
        float* wcol = p.ws + ((int64_t)(split * p.tail_tiles + (tile - p.tail_tile0)) << 16) + 128 * (int)rank +
                      lane_row;
#pragma unroll
        for (int i = 0; i < 64; ++i) wcol[(cbeg + i) << 8] = __uint_as_float(r_or_zero(rr[i], nkb));
        continue;
      }
      if (p.splits > 1) {
        // partials [split][N][M] (m fastest: a warp's 32 rows are 32 consecutive floats)
        if (!mok) continue;
        float* wcol = p.ws + (int64_t)split * p.M * p.N + m;
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          const int n = nb0 + cbeg + i;
          if (n < p.N) wcol[(int64_t)n * p.M] = __uint_as_float(r_or_zero(rr[i], nkb));
        }
        continue;
      }
      // C += acc staged through the (idle) stage ring, [128 rows][65], so each
      // warp's C loads and stores cover 32 consecutive n
      if (half) asm volatile("bar.sync %0, %1;" ::"r"(1 + h), "r"(WG) : "memory");  // previous half read
#pragma unroll
      for (int i = 0; i < 64; ++i) tb[lane_row * EPI_PITCH + i] = __uint_as_float(r_or_zero(rr[i], nkb));
      asm volatile("bar.sync %0, %1;" ::"r"(1 + h), "r"(WG) : "memory");
      int64_t con[2];
      bool nok[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int n = nb0 + cbeg + 32 * j + lane;
        nok[j] = n < p.N;
        con[j] = nok[j] ? p.gn.off(1, n) : 0;
      }
      for (int r0 = wq; r0 < BM; r0 += 4 * EPI_ROWS) {
        float cv[EPI_ROWS][2];
        int64_t co[EPI_ROWS][2];
#pragma unroll
        for (int t = 0; t < EPI_ROWS; ++t) {
          const int mm = m0 + r0 + 4 * t;
          const bool rok = mm < p.M;
          const int64_t rof = rok ? p.gm.off(1, mm) : 0;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            co[t][j] = rof + con[j];
            cv[t][j] = (rok && nok[j]) ? p.C[co[t][j]] : 0.f;
          }
        }
#pragma unroll
        for (int t = 0; t < EPI_ROWS; ++t) {
          const int r = r0 + 4 * t;
          if (m0 + r >= p.M) continue;
#pragma unroll
          for (int j = 0; j < 2; ++j)
            if (nok[j]) p.C[co[t][j]] = epi(cv[t][j], tb[r * EPI_PITCH + 32 * j + lane], p.neg);
        }
      }
    }
  } else if (rank == 0) {
    // ---------------- MMA issue (leader CTA) ----------------
    if (lane == 0) {
      const uint32_t base = smem_u32(smem);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGESW, u = kb / STAGESW;
        pair::mbar_wait_cluster(smem_u32(ready + s), u & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t sb = base + s * STAGE_BYTES;
        const uint32_t lob = base + LO_OFFW + (kb % LO_BUFS) * TILE_BYTES;
#pragma unroll
        for (int j = 0; j < BK / 8; ++j) {
          const uint32_t ah = tmem + ACCW + s * A_COLS + 8 * j, al = ah + BK;
          const uint64_t bh = !BKF ? sdesc(sb + TILE_BYTES + 256 * j)
                              : W64 ? sdesc_sw64(sb + TILE_BYTES + 32 * j)
                                    : sdesc_sw32(sb + TILE_BYTES + 4096 * j);
          // (the 3xTF32 lo tile mirrors the hi layout; the bf16 tile is SW32 boxes)
          const uint64_t bl = !BKF ? sdesc(lob + 256 * j)
                              : (W64 && !MIX) ? sdesc_sw64(lob + 32 * j)
                                              : sdesc_sw32(lob + 4096 * j);
          pair::mma_pair(tmem, ah, bh, IDESCW, (kb | j) != 0);
          if (MIX) {
            pair::mma_pair_bf16(tmem, al, bl, IDESCW_BF, 1);
          } else {
            pair::mma_pair(tmem, al, bh, IDESCW, 1);
            pair::mma_pair(tmem, ah, bl, IDESCW, 1);
          }
        }
        pair::commit_pair(smem_u32(empty + s));
        pair::commit_pair(smem_u32(lofree + kb % LO_BUFS));
      }
      pair::commit_pair(smem_u32(done));
    }
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  pair::cluster_sync2();
  if (warp == MMA_WARP)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}
// C += half 0 + half 1 of the tail tiles' compact partials: block (tail tile,
// 32 m x 8 n sub-block), partials read m-fastest, staged through shared
// memory, C read and written n-fastest (as gett_splitk_reduce_t_kernel); sums
// from -0.0 in half order.
__global__ void __launch_bounds__(256) wide_tail_reduce_kernel(const __grid_constant__ TiledParams<float> p) {
  __shared__ float tl[8][33];
  const int t = threadIdx.x;
  const int ti = blockIdx.x >> 8, sub = blockIdx.x & 255;
  int tm, tn;
  wide_tile(p, p.tail_tile0 + ti, tm, tn);
  const int ml0 = (sub & 7) * 32, nl0 = (sub >> 3) * 8;  // within the 256 x 256 tile
  const int mw = tm * 256 + ml0 + t / 8, nw = tn * 256 + nl0 + t % 8;
  const bool okw = mw < p.M && nw < p.N;
  float* c = okw ? p.C + p.gm.off(1, mw) + p.gn.off(1, nw) : nullptr;
  const float c0 = okw ? *c : 0.f;  // (before the wait: the wide kernel never writes these tiles' C)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int mr = ml0 + t % 32, nr = nl0 + t / 32;
  const float* w = p.ws + ((int64_t)ti << 16) + (nr << 8) + mr;
  const float v0 = __ldcg(w), v1 = __ldcg(w + ((int64_t)p.tail_tiles << 16));
  tl[t / 32][t % 32] = (-0.0f + v0) + v1;
  __syncthreads();
  if (okw) *c = epi(c0, tl[t % 8][t / 8], p.neg);
}
}  // namespace wide

template <bool AKF, bool BKF, bool MIX, bool W64>
cudaError_t launch_wide_t(const TiledParams<float>& p, const TmaParams& tp, cudaStream_t s) {
  auto k = wide::sgett_tc_wide_kernel<AKF, BKF, MIX, W64>;
  static unsigned long long configured = 0;
  cudaError_t e = ensure_dyn_smem(k, wide::SMEMW_BYTES, configured);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = p.tail_tiles > 0 ? dim3((unsigned)(2 * (p.tail_tile0 + 2 * p.tail_tiles)))
                                 : dim3((unsigned)(2 * p.tiles_m * p.tiles_n * p.splits));
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = wide::SMEMW_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, p, tp);
}

}  // namespace tc

cudaError_t launch_sgett_tc(const TiledParams<float>& p, const TmaParams* tp, bool a_kf, bool b_kf,
                            bool a_vec, bool b_vec, cudaStream_t s) {
  cudaError_t e;
  if (a_kf && b_kf) e = tc::launch2<true, true>(p, tp, a_vec, b_vec, s);
  else if (a_kf) e = tc::launch2<true, false>(p, tp, a_vec, b_vec, s);
  else if (b_kf) e = tc::launch2<false, true>(p, tp, a_vec, b_vec, s);
  else e = tc::launch2<false, false>(p, tp, a_vec, b_vec, s);
  if (e != cudaSuccess || p.splits == 1) return e;
  return launch_splitk_reduce<float>(p, s);
}

cudaError_t launch_sgett_tc_pair(const TiledParams<float>& p, const TmaParams& tp, cudaStream_t s) {
  cudaError_t e = tc::launch_pair(p, tp, s);
  if (e != cudaSuccess) return e;
  return launch_splitk_reduce<float>(p, s);
}

// wide CTA-pair SGETT: p.tiles_m / tiles_n in 256-row pair tiles
template <bool MIX, bool W64>
cudaError_t launch_wide_m(const TiledParams<float>& p, const TmaParams& tp, bool a_kf, bool b_kf, cudaStream_t s) {
  if (a_kf && b_kf) return tc::launch_wide_t<true, true, MIX, W64>(p, tp, s);
  if (a_kf) return tc::launch_wide_t<true, false, MIX, W64>(p, tp, s);
  if (b_kf) return tc::launch_wide_t<false, true, MIX, W64>(p, tp, s);
  return tc::launch_wide_t<false, false, MIX, false>(p, tp, s);
}

cudaError_t launch_sgett_tc_wide(const TiledParams<float>& p, const TmaParams& tp, bool a_kf, bool b_kf,
                                 bool mix, bool k16, cudaStream_t s) {
  cudaError_t e;
  if (mix) e = k16 ? launch_wide_m<true, true>(p, tp, a_kf, b_kf, s) : launch_wide_m<true, false>(p, tp, a_kf, b_kf, s);
  else e = k16 ? launch_wide_m<false, true>(p, tp, a_kf, b_kf, s) : launch_wide_m<false, false>(p, tp, a_kf, b_kf, s);
  if (e != cudaSuccess) return e;
  if (p.tail_tiles > 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)p.tail_tiles * 256u);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = g_launch_pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, tc::wide::wide_tail_reduce_kernel, p);
  }
  if (p.splits == 1) return e;
  return launch_splitk_reduce<float>(p, s);
}

int tc_bm() { return tc::BM; }
int tc_bn() { return tc::BN; }
int tc_bk() { return tc::BK; }

}  // namespace gett
