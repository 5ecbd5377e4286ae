// SGETT on the 5th-generation tensor cores: 3xTF32 with tcgen05.mma + TMEM,
// warp-specialised.
//
// Replaces the fp32 hot loop (kernel.py:48-78 for sgett) for contractions big
// enough to tile.  Per 128x128 output tile, k-blocks of 16, STAGES-deep ring:
//   * producer warpgroup (warps 0-3): gathers the A' (M x K) and B' (N x K)
//     k-block straight from the strided views with cp.async (row offsets
//     decoded once per tile, k offsets stepped through the K group's outer
//     table staged in smem; 16-byte copies where the planner proved 4-k
//     contiguity) into the UMMA K-major no-swizzle layout (8-row x 16-byte
//     core matrices, LBO 128 B between k-chunks, SBO 512 B between 8-row
//     groups); completion is tracked per stage by cp.async.mbarrier.arrive,
//     so up to STAGES k-blocks are in flight without blocking anyone;
//   * split warpgroup (warps 4-7): when a stage lands, splits every value in
//     place into hi = rna_tf32(x) and lo = x - hi (exact in fp32) into the
//     stage's lo tile, fence.proxy.async, arrive;
//   * MMA warp (warp 8): one elected thread issues, per UMMA_K = 8 step,
//     tcgen05.mma.cta_group::1.kind::tf32 for hi*hi, lo*hi, hi*lo into one fp32
//     accumulator in TMEM (128 lanes x 128 columns) and tcgen05.commit frees
//     the stage for the producers;
//   * epilogue (split warpgroup, one TMEM lane quarter per warp):
//     tcgen05.ld 32x32b -> C += acc through the C offset tables, or the
//     split-K partial into the workspace.
// Accuracy: 3xTF32 products are within ~2^-22 relative, fp32 accumulation in
// TMEM; checked against the fp64 oracle and the reference (tests/).
#include <cstdint>

#include "device.cuh"
#include "kernels.hpp"

#ifndef GETT_TC_STAGES
#define GETT_TC_STAGES 6
#endif

namespace gett {
namespace tc {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int BK = 16;
constexpr int CH = BK / 4;                     // 16-byte k-chunks per row
constexpr int STAGES = GETT_TC_STAGES;
constexpr int WG = 128;                        // threads per warpgroup
constexpr int THREADS = 2 * WG + 32;           // producer WG, split/epilogue WG, MMA warp
constexpr int GROUP_M = 8;
constexpr int LBO = 128;                       // bytes between k-chunks
constexpr int SBO = CH * 128;                  // bytes between 8-row groups
constexpr int TILE_BYTES = 128 * BK * 4;       // one operand part (hi or lo): 8 KB
constexpr int STAGE_BYTES = 4 * TILE_BYTES;    // A hi, A lo, B hi, B lo
constexpr int TCAP = 256;                      // outer k-table entries staged in smem
constexpr int BAR_BYTES = 256;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + BAR_BYTES + 2 * TCAP * 8;
constexpr uint32_t TMEM_COLS = 128;
static_assert(3 * STAGES + 2 <= BAR_BYTES / 8, "barrier area");

// instruction descriptor: D f32, A/B tf32, both K-major, N = 128, M = 128
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);
// ... with A / B MN-major (bits 15 / 16) for operands gathered along their rows
__host__ __device__ constexpr uint32_t idesc(bool a_mn, bool b_mn) {
  return IDESC | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16);
}
// MN-major no-swizzle layout (rows contiguous): 16-byte chunk of 4 rows at k,
// core matrix 8 k x 16 B; SBO 128 B between row chunks, LBO 4 KB between k-groups
constexpr int MN_SBO = 128, MN_LBO = 32 * 128;
__device__ __forceinline__ uint32_t toff_mn(int mc, int k) {
  return (uint32_t)(mc * MN_SBO + (k & 7) * 16 + (k >> 3) * MN_LBO);
}

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

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t acc,
                                         uint32_t id = IDESC) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(tmem),
      "l"(a), "l"(b), "r"(id), "r"(acc)
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

// One operand's 128-row x BK gather with cp.async by the producer warpgroup.
// Warp w owns row groups 4w..4w+3 (8 rows each).  One warp instruction covers
// 8 consecutive rows x 4 k: lane l -> row 8g + l%8 and, for 16-byte copies
// (VEC: 4 contiguous k per row), chunk l/8 (8 rows x 64 B of gmem, four
// conflict-free 128 B smem wavefronts); for 4-byte copies, k = 4c + l/8 of
// chunk c (32 distinct smem banks; 8 rows x 4 k of gmem).
template <bool VEC>
struct Gather {
  int64_t roff[4];
  bool rok[4];
  int lr, le, w;
  int64_t ko[VEC ? 1 : CH];

  __device__ __forceinline__ void setup(int warp, int lane, const GroupDev& g, int base_row,
                                        int nrows) {
    w = warp;
    lr = lane & 7;
    le = lane >> 3;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int r = base_row + 8 * (4 * w + i) + lr;
      rok[i] = r < nrows;
      roff[i] = rok[i] ? g.off(0, r) : 0;
    }
  }

  __device__ __forceinline__ static int64_t koff(const KDec& kd, int k) {
    int q, r;
    kd.div.divmod(k, q, r);
    return kd.T[q] + (int64_t)r * kd.s;
  }

  __device__ __forceinline__ void prep(const KDec& kd, int k0, int kend) {
    if (VEC) {
      const int k = k0 + 4 * le;
      ko[0] = k < kend ? koff(kd, k) : 0;
    } else {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const int k = k0 + 4 * c + le;
        ko[c] = k < kend ? koff(kd, k) : 0;
      }
    }
  }

  __device__ __forceinline__ void issue(uint8_t* s, const float* base, int k0, int kend) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = 8 * (4 * w + i) + lr;
      if (VEC) {
        uint8_t* dst = s + toff(r, le);
        if (rok[i] && k0 + 4 * le < kend) cp_async_16(dst, base + roff[i] + ko[0]);
        else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          uint8_t* dst = s + toff(r, c) + 4 * le;
          if (rok[i] && k0 + 4 * c + le < kend) cp_async_4(dst, base + roff[i] + ko[c]);
          else *reinterpret_cast<float*>(dst) = 0.f;
        }
      }
    }
  }
};

// Rows-contiguous operand with 16-byte row chunks (unit-stride inner row mode,
// extent and all offsets divisible by 4): staged MN-major, [k][128 rows] fp32
// (512 B per k), and transposed into the K-major hi/lo tiles by the split
// warpgroup (split_tile_rv) — the tf32 UMMA reads K-major only.  Warp w,
// instruction i copies k = 4w + i: lane l -> rows 4l..4l+3, so one warp
// instruction moves 512 contiguous bytes of gmem into 512 contiguous bytes of
// smem (the 4-byte path needs 16 instructions for the same k-block).
struct GatherRV {
  int64_t roff;
  bool rok;
  int lane, w;
  int64_t ko[4];

  __device__ __forceinline__ void setup(int warp, int ln, const GroupDev& g, int base_row,
                                        int nrows) {
    w = warp;
    lane = ln;
    const int r = base_row + 4 * lane;
    rok = r < nrows;
    roff = rok ? g.off(0, r) : 0;
  }

  __device__ __forceinline__ void prep(const KDec& kd, int k0, int kend) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = k0 + 4 * w + i;
      ko[i] = k < kend ? Gather<true>::koff(kd, k) : 0;
    }
  }

  __device__ __forceinline__ void issue(uint8_t* s, const float* base, int k0, int kend) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int k = 4 * w + i;
      uint8_t* dst = s + k * 512 + lane * 16;
      if (rok && k0 + k < kend) cp_async_16(dst, base + roff + ko[i]);
      else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
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

// split + transpose one MN-major staged tile ([k][row] fp32, GatherRV) into the
// K-major hi tile (same 8 KB, in place) and lo tile.  Split thread t = 32ws + l
// reads units (k = 4ws + l/8, rows 4rc..4rc+3 with rc = 8i + l%8), i = 0..3
// (each 8-lane phase reads 128 contiguous bytes); after a warpgroup barrier
// (the writes land on other threads' inputs) it stores the 4 values of a unit
// rotated by s = (l/2)%4, so at each store the 32 lanes cover all 8 (row % 8)
// x 4 (k % 4) positions = 32 distinct banks.
__device__ __forceinline__ void split_tile_rv(uint8_t* hi_s, uint8_t* lo_s, int t) {
  const int ws = t >> 5, l = t & 31;
  const int k = 4 * ws + (l >> 3);
  float4 x[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int rc = 8 * i + (l & 7);
    x[i] = *reinterpret_cast<const float4*>(hi_s + k * 512 + rc * 16);
  }
  asm volatile("bar.sync 1, 128;" ::: "memory");
  const int rot = (l >> 1) & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int rc = 8 * i + (l & 7);
    float4 h, lo;
    split4(x[i], h, lo);
    float hv[4] = {h.x, h.y, h.z, h.w}, lv[4] = {lo.x, lo.y, lo.z, lo.w};
    // rotate left by rot with selects (no dynamic register indexing)
    if (rot & 1) {
      float th = hv[0], tl = lv[0];
      hv[0] = hv[1]; hv[1] = hv[2]; hv[2] = hv[3]; hv[3] = th;
      lv[0] = lv[1]; lv[1] = lv[2]; lv[2] = lv[3]; lv[3] = tl;
    }
    if (rot & 2) {
      float th0 = hv[0], th1 = hv[1], tl0 = lv[0], tl1 = lv[1];
      hv[0] = hv[2]; hv[1] = hv[3]; hv[2] = th0; hv[3] = th1;
      lv[0] = lv[2]; lv[1] = lv[3]; lv[2] = tl0; lv[3] = tl1;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int row = 4 * rc + ((j + rot) & 3);
      const uint32_t o = toff(row, k >> 2) + (k & 3) * 4;
      *reinterpret_cast<float*>(hi_s + o) = hv[j];
      *reinterpret_cast<float*>(lo_s + o) = lv[j];
    }
  }
}

// split one landed tile (8 KB, either layout): 512 dense 16-byte units, thread t
// handles units t, t+128, t+256, t+384 (consecutive threads -> consecutive
// 16 B: conflict-free)
__device__ __forceinline__ void split_tile(uint8_t* hi_s, uint8_t* lo_s, int t) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t o = (uint32_t)(t + WG * i) * 16;
    float4 x = *reinterpret_cast<const float4*>(hi_s + o);
    float4 h, l;
    split4(x, h, l);
    *reinterpret_cast<float4*>(hi_s + o) = h;
    *reinterpret_cast<float4*>(lo_s + o) = l;
  }
}

template <bool AKF, bool BKF, bool AVEC, bool BVEC>
__global__ void __launch_bounds__(THREADS, 1)
    sgett_tc_kernel(const __grid_constant__ TiledParams<float> p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr bool AMN = false, BMN = false;  // K-major smem layouts for both operands
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);  // gathers landed
  uint64_t* ready = full + STAGES;                                            // split done
  uint64_t* empty = ready + STAGES;                                           // MMAs done
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
  int64_t* ktabs = reinterpret_cast<int64_t*>(smem + STAGES * STAGE_BYTES + BAR_BYTES);  // [2][TCAP]
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

  // the K group's outer offset tables, staged in shared memory when small
  const int n_outer = (p.gk.G + p.gk.e_in.d - 1) / p.gk.e_in.d;
  KDec kda{p.gk.T[0], p.gk.s_in[0], p.gk.e_in}, kdb{p.gk.T[1], p.gk.s_in[1], p.gk.e_in};
  if (n_outer <= TCAP) {
    for (int i = tid; i < n_outer; i += THREADS) {
      ktabs[i] = __ldg(p.gk.T[0] + i);
      ktabs[TCAP + i] = __ldg(p.gk.T[1] + i);
    }
    kda.T = ktabs;
    kdb.T = ktabs + TCAP;
  }
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(full + s), 2 * WG);  // per producer thread: cp.async + plain arrival
      mbar_init(smem_u32(ready + s), WG);
      mbar_init(smem_u32(empty + s), 1);      // tcgen05.commit
    }
    mbar_init(smem_u32(done), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  auto stage = [&](int s) { return smem + s * STAGE_BYTES; };

  if (warp < 4) {
    // ---------------- producer warpgroup ----------------
    typename GatherSel<AKF, AVEC>::type ga;
    typename GatherSel<BKF, BVEC>::type gb;
    ga.setup(warp, tid & 31, p.gm, m0, p.M);
    gb.setup(warp, tid & 31, p.gn, n0, p.N);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES, u = kb / STAGES;
      const int k0 = kbeg + kb * BK;
      ga.prep(kda, k0, kend);
      gb.prep(kdb, k0, kend);
      if (u > 0) mbar_wait(smem_u32(empty + s), (u - 1) & 1);
      ga.issue(stage(s), p.A, k0, kend);
      gb.issue(stage(s) + 2 * TILE_BYTES, p.B, k0, kend);
      mbar_arrive_cpasync(smem_u32(full + s));
      mbar_arrive(smem_u32(full + s));
    }
    cp_async_wait<0>();
  } else if (warp < 8) {
    // ---------------- split warpgroup, then epilogue ----------------
    const int t = tid - WG;
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES, u = kb / STAGES;
      mbar_wait(smem_u32(full + s), u & 1);
      uint8_t* st = stage(s);
      if (!AKF && AVEC) split_tile_rv(st, st + TILE_BYTES, t);
      else split_tile(st, st + TILE_BYTES, t);
      if (!BKF && BVEC) split_tile_rv(st + 2 * TILE_BYTES, st + 3 * TILE_BYTES, t);
      else split_tile(st + 2 * TILE_BYTES, st + 3 * TILE_BYTES, t);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(smem_u32(ready + s));
    }
    if (nkb > 0) mbar_wait(smem_u32(done), 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // thread t owns accumulator row t (TMEM lane t; warp w%4 reads lanes 32(w%4)..)
    const int m = m0 + t;
    const bool mok = m < p.M;
    const int64_t ro = (mok && p.splits == 1) ? p.gm.off(1, m) : 0;
    float* wrow = p.splits > 1 ? p.ws + ((int64_t)split * p.M + (mok ? m : 0)) * p.N : nullptr;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      uint32_t r[16];
      const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
            "=r"(r[14]), "=r"(r[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (!mok) continue;
      if (p.splits == 1) {
        float cv[16];
        int64_t co[16];
        const int nvalid = p.N - (n0 + c0);  // offsets may be negative: validity by index
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          co[i] = i < nvalid ? ro + p.gn.off(1, n0 + c0 + i) : 0;
          cv[i] = i < nvalid ? p.C[co[i]] : 0.f;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float acc = nkb > 0 ? __uint_as_float(r[i]) : -0.0f;
          if (i < nvalid) p.C[co[i]] = epi(cv[i], acc, p.neg);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int n = n0 + c0 + i;
          if (n < p.N) wrow[n] = nkb > 0 ? __uint_as_float(r[i]) : -0.0f;
        }
      }
    }
  } else {
    // ---------------- MMA warp ----------------
    if ((tid & 31) == 0) {
      const uint32_t smem_base = smem_u32(smem);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES, u = kb / STAGES;
        mbar_wait(smem_u32(ready + s), u & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t sb = smem_base + s * STAGE_BYTES;
#pragma unroll
        for (int j = 0; j < BK / 8; ++j) {
          // per k-step j: K-major advances 256 B (2 k-chunks), MN-major one k-group
          const uint32_t ja = AMN ? j * MN_LBO : 256 * j, jb = BMN ? j * MN_LBO : 256 * j;
          const uint32_t alb = AMN ? MN_LBO : LBO, asb = AMN ? MN_SBO : SBO;
          const uint32_t blb = BMN ? MN_LBO : LBO, bsb = BMN ? MN_SBO : SBO;
          const uint64_t ah = sdesc(sb + ja, alb, asb);
          const uint64_t al = sdesc(sb + TILE_BYTES + ja, alb, asb);
          const uint64_t bh = sdesc(sb + 2 * TILE_BYTES + jb, blb, bsb);
          const uint64_t bl = sdesc(sb + 3 * TILE_BYTES + jb, blb, bsb);
          constexpr uint32_t ID = idesc(AMN, BMN);
          mma_tf32(tmem, ah, bh, (kb | j) != 0, ID);  // first MMA of the tile overwrites D
          mma_tf32(tmem, al, bh, 1, ID);
          mma_tf32(tmem, ah, bl, 1, ID);
        }
        commit(smem_u32(empty + s));
      }
      commit(smem_u32(done));
    }
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 8)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

template <bool AKF, bool BKF, bool AV, bool BV>
cudaError_t launch4(const TiledParams<float>& p, cudaStream_t s) {
  auto k = sgett_tc_kernel<AKF, BKF, AV, BV>;
  static unsigned long long configured = 0;
  cudaError_t e = ensure_dyn_smem(k, SMEM_BYTES, configured);
  if (e != cudaSuccess) return e;
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
