// Streaming-load ceiling of the SGETT producer's copy engines: 148 CTAs each
// stream a contiguous share of a 1 GiB buffer through a STAGES-deep ring of
// 16 KB shared-memory stages (a consumer warp only waits + releases).
//   mode 0: cp.async 16 B per thread, 8-row x 64 B warp footprint (the K-major
//           gather pattern: rows 160 B apart, as c5's orig-A rows)
//   mode 1: cp.async 16 B per thread, 512 contiguous bytes per warp instruction
//   mode 2: cp.async.bulk (one thread, 4 x 4 KB bulk copies per stage,
//           mbarrier complete_tx)
// Prints GB/s per (mode, stages, producer warps).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stream_bw tools/stream_bw.cu
#include <cstdint>
#include <cstdio>
#include <cuda.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint32_t a, uint32_t ph) {
  asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(a), "r"(ph) : "memory");
}
__device__ __forceinline__ void arrive(uint32_t a) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(a) : "memory");
}

constexpr int SB = 16384;

template <int MODE>
__global__ void stream(const char* src, size_t per_cta, int stages, int pwarps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = (uint64_t*)(sm + stages * SB);
  uint64_t* empty = full + stages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int PT = pwarps * 32;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(full + s)), "r"(MODE == 2 ? 1 : PT));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(empty + s)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const char* base = src + blockIdx.x * per_cta;
  const int nst = (int)(per_cta / SB);
  if (warp < pwarps) {
    for (int i = 0; i < nst; ++i) {
      const int s = i % stages, u = i / stages;
      if (u > 0) wait(su32(empty + s), (u - 1) & 1);
      const char* g = base + (size_t)i * SB;
      const uint32_t d = su32(sm + s * SB);
      if (MODE == 2) {
        if (tid == 0) {
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + s)), "r"(SB) : "memory");
          for (int c = 0; c < 4; ++c)
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];"
                         ::"r"(d + c * 4096), "l"(g + c * 4096), "r"(su32(full + s)) : "memory");
        }
      } else {
        // 1024 16-byte units per stage
        for (int j = tid; j < SB / 16; j += PT) {
          uint32_t o;
          if (MODE == 0) {
            // unit j: row r = j / 4 (of 256 rows, 160 B apart in gmem... within
            // the stage's 16 KB window: rows of 64 B), chunk j % 4
            const int w8 = j / 32, l = j % 32;
            o = (uint32_t)((w8 * 8 + l % 8) * 64 + (l / 8) * 16);
          } else {
            o = (uint32_t)j * 16;
          }
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + o), "l"(g + o));
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(full + s)) : "memory");
      }
    }
    asm volatile("cp.async.wait_all;");
  } else if (warp == pwarps && lane == 0) {
    for (int i = 0; i < nst; ++i) {
      const int s = i % stages, u = i / stages;
      wait(su32(full + s), u & 1);
      arrive(su32(empty + s));
    }
  }
}

template <int MODE>
void run(const char* buf, size_t bytes, int stages, int pwarps, int grid = 148) {
  auto k = stream<MODE>;
  const int smem = stages * SB + 2 * stages * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const size_t per = (bytes / 148) / SB * SB / (grid < 148 ? 4 : 1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<<<grid, (pwarps + 1) * 32, smem>>>(buf, per, stages, pwarps);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<<<grid, (pwarps + 1) * 32, smem>>>(buf, per, stages, pwarps);
  cudaEventRecord(e1);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"mode\": %d, \"grid\": %d, \"stages\": %d, \"producer_warps\": %d, \"GBps\": %.0f, \"GBps_per_sm\": %.1f, \"err\": \"%s\"}\n", MODE,
         grid, stages, pwarps, 5.0 * per * grid / (ms * 1e6), 5.0 * per / (ms * 1e6), cudaGetErrorString(e ? e : cudaGetLastError()));
}


// mode 3/4: TMA tiled loads of 128 rows x BOXK floats from a [rows][40]-float
// tensor (rows 160 B apart: c5's orig-A rows), boxes of 8 floats (SWIZZLE_32B,
// mode 3) or 32 floats (SWIZZLE_128B, mode 4); 16 KB per stage
template <int BOXK>
__global__ void stream_tma(const __grid_constant__ CUtensorMap tm, int rows_per_cta, int stages) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = (uint64_t*)(sm + stages * SB);
  uint64_t* empty = full + stages;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(empty + s)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  constexpr int BOXES = SB / (128 * BOXK * 4);  // boxes per stage
  const int r0 = blockIdx.x * rows_per_cta;
  // walk: 128-row groups x k offsets (0, 8, .., 32 for BOXK 8: 5 boxes per row group)
  constexpr int KB = 40 / BOXK > 0 ? (BOXK == 8 ? 5 : 1) : 1;
  const int nbox = rows_per_cta / 128 * KB;
  const int nst = nbox / BOXES;
  if (tid == 0) {
    int b = 0;
    for (int i = 0; i < nst; ++i) {
      const int s = i % stages, u = i / stages;
      if (u > 0) wait(su32(empty + s), (u - 1) & 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + s)), "r"(SB) : "memory");
      for (int c = 0; c < BOXES; ++c, ++b) {
        const int kx = (b % KB) * BOXK, ry = r0 + (b / KB) * 128;
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(su32(sm + s * SB + c * 128 * BOXK * 4)), "l"(&tm), "r"(kx), "r"(ry), "r"(su32(full + s)) : "memory");
      }
    }
  } else if (tid == 32) {
    for (int i = 0; i < nst; ++i) {
      const int s = i % stages, u = i / stages;
      wait(su32(full + s), u & 1);
      arrive(su32(empty + s));
    }
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int BOXK>
void run_tma(char* buf, size_t bytes, int stages, int grid) {
  static EncodeFn enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  }
  const cuuint64_t rows = bytes / 160;
  cuuint64_t dims[2] = {40, rows}, strides[1] = {160};
  cuuint32_t box[2] = {BOXK, 128}, es[2] = {1, 1};
  CUtensorMap tm;
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE,
                   BOXK == 8 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  auto k = stream_tma<BOXK>;
  const int smem = stages * SB + 2 * stages * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int rpc = (int)((rows / 148) / 1280 * 1280 / (grid < 148 ? 4 : 1));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<<<grid, 64, smem>>>(tm, rpc, stages);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) k<<<grid, 64, smem>>>(tm, rpc, stages);
  cudaEventRecord(e1);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  // bytes moved: BOXK 8 reads all 40 floats of each row; BOXK 32 reads 32 of 40
  const double per = (double)rpc * (BOXK == 8 ? 160 : 128);
  printf("{\"mode\": %d, \"grid\": %d, \"stages\": %d, \"box_k\": %d, \"GBps\": %.0f, \"GBps_per_sm\": %.1f, \"enc\": %d, \"err\": \"%s\"}\n",
         BOXK == 8 ? 3 : 4, grid, stages, BOXK, 5.0 * per * grid / (ms * 1e6), 5.0 * per / (ms * 1e6), (int)r,
         cudaGetErrorString(e ? e : cudaGetLastError()));
}


// mode 5: c5's orig-A operand exactly as the SGETT kernel loads it — rank-4
// tensor (k4 40 x 1, m3 16 x 40, m0 48 x 983040, k12 768 x 1280 floats),
// SWIZZLE_32B boxes (8, 16, 8, 1); 144 CTAs = 6 row tiles x 24 K slices, each
// walks its 1280 k in 80 k-blocks of two boxes (8 KB) per stage; optional
// second operand (c5's orig B: rows 96 x 1, k4 40 x 73728, k2 32 x 2304, k1
// 24 x 96) as [8 k][128 rows] boxes (OOB rows zero), 8 KB per stage
template <bool WITH_B>
__global__ void stream_c5(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, int stages) {
  extern __shared__ __align__(1024) uint8_t sm[];
  constexpr int STB = WITH_B ? 16384 : 8192;
  uint64_t* full = (uint64_t*)(sm + stages * STB);
  uint64_t* empty = full + stages;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(empty + s)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int tile = blockIdx.x % 6, split = blockIdx.x / 6;
  const int kbeg = split * 1280;
  if (tid == 0) {
    for (int kb = 0; kb < 80; ++kb) {
      const int s = kb % stages, u = kb / stages;
      if (u > 0) wait(su32(empty + s), (u - 1) & 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + s)), "r"(STB) : "memory");
      for (int h = 0; h < 2; ++h) {
        const int k = kbeg + kb * 16 + 8 * h;
        const int k4 = k % 40, k12 = k / 40;
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                     ::"r"(su32(sm + s * STB + 4096 * h)), "l"(&ta), "r"(k4), "r"(0), "r"(8 * tile), "r"(k12), "r"(su32(full + s)) : "memory");
        if (WITH_B) {
          const int k2 = k12 % 32, k1 = k12 / 32;
          asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                       ::"r"(su32(sm + s * STB + 8192 + 4096 * h)), "l"(&tb), "r"(0), "r"(k4), "r"(k2), "r"(k1), "r"(su32(full + s)) : "memory");
        }
      }
    }
  } else if (tid == 32) {
    for (int kb = 0; kb < 80; ++kb) {
      const int s = kb % stages, u = kb / stages;
      wait(su32(full + s), u & 1);
      arrive(su32(empty + s));
    }
  }
}

template <bool WITH_B>
void run_c5(int stages) {
  static EncodeFn enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  }
  float *A, *B;
  cudaMalloc(&A, 47185920ull * 4);
  cudaMalloc(&B, 2949120ull * 4);
  cudaMemset(A, 0, 47185920ull * 4);
  cudaMemset(B, 0, 2949120ull * 4);
  CUtensorMap ta, tb;
  cuuint64_t da[4] = {40, 16, 48, 768}, sa[3] = {160, 3932160, 5120};
  cuuint32_t ba[4] = {8, 16, 8, 1}, es[4] = {1, 1, 1, 1};
  enc(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, A, da, sa, ba, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t db[4] = {96, 40, 32, 24}, sb[3] = {294912, 9216, 384};
  cuuint32_t bb[4] = {128, 8, 1, 1};
  enc(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, B, db, sb, bb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  auto k = stream_c5<WITH_B>;
  const int smem = stages * (WITH_B ? 16384 : 8192) + 2 * stages * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<<<144, 64, smem>>>(ta, tb, stages);
  cudaEventRecord(e0);
  for (int i = 0; i < 10; ++i) k<<<144, 64, smem>>>(ta, tb, stages);
  cudaEventRecord(e1);
  cudaError_t e = cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"mode\": \"c5_%s\", \"stages\": %d, \"us_per_pass\": %.1f, \"err\": \"%s\"}\n", WITH_B ? "A+B" : "A", stages,
         ms * 100.0, cudaGetErrorString(e ? e : cudaGetLastError()));
  cudaFree(A);
  cudaFree(B);
}

int main() {
  const size_t bytes = 1ull << 30;
  char* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  for (int st : {8, 16}) {
    run_c5<false>(st);
    run_c5<true>(st);
  }
  for (int g : {148, 48, 16}) {
    run_tma<8>(buf, bytes, 8, g);
    run_tma<32>(buf, bytes, 8, g);
  }
  for (int g : {16, 48}) {
    run<0>(buf, bytes, 8, 4, g);
    run<1>(buf, bytes, 8, 4, g);
    run<2>(buf, bytes, 8, 1, g);
    run<0>(buf, bytes, 8, 8, g);
  }
  return 0;
}
