// Checks the TMA-fed operand layouts of the SGETT kernel: A and B (128 rows x
// 16 k, fp32) loaded by cp.async.bulk.tensor with 8-float boxes and
// SWIZZLE_32B (one 4 KB box per 8 k), consumed by tcgen05.mma.kind::tf32 with
// SWIZZLE_32B K-major smem descriptors (mode 0), or A read back by threads
// through the swizzle formula of sgett_tc.cu, written to TMEM and used as the
// TMEM A operand (mode 1).  D (128 x 128) compared with a CPU product of
// truncated tf32 inputs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_tma_test tools/umma_tma_test.cu
#include <cuda.h>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc_sw32(uint32_t a) {
  // start, LBO 16 (unused for swizzled K-major), SBO 256 (8 rows x 32 B), version 1, SWIZZLE_32B
  return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)(16 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         (1ull << 46) | (6ull << 61);
}
// byte offset of (row r, k) in one SWIZZLE_32B box of 128 rows x 8 floats
__host__ __device__ __forceinline__ uint32_t sw32_off(int r, int k) {
  return (uint32_t)(r * 32 + ((((k >> 2) ^ (r >> 2)) & 1) << 4) + (k & 3) * 4);
}

__global__ void kern(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, float* D,
                     int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sa = sm;           // 2 boxes x 4 KB
  uint8_t* sb = sm + 8192;    // 2 boxes x 4 KB
  uint64_t* bar = (uint64_t*)(sm + 16384);
  uint32_t* slot = (uint32_t*)(bar + 2);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + 1)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(16384) : "memory");
    for (int j = 0; j < 2; ++j) {
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su32(sa + 4096 * j)), "l"(&ta), "r"(8 * j), "r"(0), "r"(su32(bar)) : "memory");
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(su32(sb + 4096 * j)), "l"(&tb), "r"(8 * j), "r"(0), "r"(su32(bar)) : "memory");
    }
  }
  asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W_%=;\n\t}" ::"r"(su32(bar)));
  const int w = threadIdx.x / 32, m = threadIdx.x;
  if (mode == 1) {
    // thread = row: read its 16 k through the swizzle formula -> TMEM columns 128..143
    uint32_t r[16];
    for (int kk = 0; kk < 16; ++kk) r[kk] = *(const uint32_t*)(sa + 4096 * (kk >> 3) + sw32_off(m, kk & 7));
    const uint32_t t = tmem + ((uint32_t)(w * 32) << 16) + 128;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(t), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                 "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    for (int j = 0; j < 2; ++j) {
      const uint64_t db = sdesc_sw32(su32(sb + 4096 * j));
      if (mode == 0) {
        const uint64_t da = sdesc_sw32(su32(sa + 4096 * j));
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(j));
      } else {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                     ::"r"(tmem), "r"(tmem + 128 + 8 * j), "l"(db), "r"(idesc), "r"(j));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar + 1)));
  }
  asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W_%=;\n\t}" ::"r"(su32(bar + 1)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < 128; c0 += 16) {
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(tmem + ((uint32_t)(w * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 16; ++i) D[m * 128 + c0 + i] = __uint_as_float(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static float trunc_tf32(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xffffe000u; memcpy(&x, &u, 4); return x; }

int main() {
  static float hA[128 * 16], hB[128 * 16], hD[128 * 128];
  uint64_t s = 7;
  auto rnd = [&]() { s = s * 6364136223846793005ull + 1442695040888963407ull; return (float)((double)(s >> 11) / 9007199254740992.0 * 2.0 - 1.0); };
  for (int i = 0; i < 128 * 16; ++i) { hA[i] = rnd(); hB[i] = rnd(); }
  float *A, *B, *D;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap ta, tb;
  cuuint64_t dims[2] = {16, 128}, strides[1] = {64};
  cuuint32_t box[2] = {8, 128}, es[2] = {1, 1};
  int r1 = enc(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, A, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int r2 = enc(&tb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, B, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 64);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(D, 0, sizeof hD);
    kern<<<1, 128, 16384 + 64>>>(ta, tb, D, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 128; ++n) {
        double ref = 0;
        for (int kk = 0; kk < 16; ++kk) ref += (double)trunc_tf32(hA[m * 16 + kk]) * trunc_tf32(hB[n * 16 + kk]);
        maxerr = fmax(maxerr, fabs(ref - hD[m * 128 + n]));
      }
    printf("{\"mode\": \"%s\", \"encode\": [%d, %d], \"max_abs_err\": %g, \"err\": \"%s\"}\n",
           mode == 0 ? "A,B smem SW32" : "A via swizzle formula -> TMEM, B smem SW32", r1, r2, maxerr,
           cudaGetErrorString(e));
  }
  return 0;
}
