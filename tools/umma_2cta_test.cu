// Probe of the CTA-pair MMA (tcgen05.mma.cta_group::2.kind::tf32) the SGETT
// kernel would use for M = 256 tiles: a cluster of 2 CTAs; CTA r holds rows
// 128r..128r+127 of A (256 x 8) in its TMEM (tcgen05.st, lane = row) and rows
// 64r..64r+63 of B (128 x 8) in its shared memory (K-major no-swizzle core
// matrices); the leader (rank 0) issues one M=256 N=128 MMA with A from TMEM;
// the commit is multicast to both CTAs' barriers; each CTA reads its 128 x 128
// accumulator back.  Small-integer data (exact in tf32), compared with a CPU
// product.  Mode 1 loads all 128 B rows into both CTAs instead (tells whether
// B is split N-wise across the pair).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_2cta_test tools/umma_2cta_test.cu
#include <cmath>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
         (1ull << 46);
}

__global__ void __cluster_dims__(2, 1, 1) k2(const float* A, const float* B, float* D, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bar = (uint64_t*)(sm + 8192);
  uint32_t* slot = (uint32_t*)(bar + 1);
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tid = threadIdx.x, w = tid / 32;
  // B rows for this CTA: mode 0 -> rows 64*rank .. +63 (64-row tile), mode 1 -> all 128
  const int nb = mode == 0 ? 64 : 128, b0 = mode == 0 ? 64 * (int)rank : 0;
  for (int i = tid; i < nb * 8; i += blockDim.x) {
    const int n = i / 8, kk = i % 8;
    const uint32_t o = (n / 8) * 256 + (kk / 4) * 128 + (n % 8) * 16 + (kk % 4) * 4;
    *(float*)(sm + o) = B[(b0 + n) * 8 + kk];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *slot;
  // A rows 128*rank + tid -> this CTA's TMEM lanes, columns 128..135
  {
    uint32_t r[8];
    for (int i = 0; i < 8; ++i) r[i] = __float_as_uint(A[(128 * rank + tid) * 8 + i]);
    const uint32_t ta = tmem + ((uint32_t)(w * 32) << 16) + 128;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (rank == 0 && tid == 0) {
    // D f32, A/B tf32, K-major, N = 128, M = 256
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((256u >> 4) << 24);
    const uint64_t db = sdesc(su32(sm), 128, 256);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                 "r"(tmem + 128), "l"(db), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                     su32(bar)),
                 "h"((uint16_t)3));
  }
  asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W_%=;\n\t}" ::"r"(su32(bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < 128; c0 += 16) {
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(tmem + ((uint32_t)(w * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 16; ++i) D[(128 * rank + tid) * 128 + c0 + i] = __uint_as_float(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
  static float hA[256 * 8], hB[128 * 8], hD[256 * 128];
  for (int i = 0; i < 256 * 8; ++i) hA[i] = (float)((i * 7) % 13 - 6);
  for (int i = 0; i < 128 * 8; ++i) hB[i] = (float)((i * 5) % 11 - 5);
  float *A, *B, *D;
  cudaMalloc(&A, sizeof hA);
  cudaMalloc(&B, sizeof hB);
  cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 + 64);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(D, 0, sizeof hD);
    k2<<<2, 128, 8192 + 64>>>(A, B, D, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
    double err = 0, err_lo = 0, err_hi = 0;
    for (int m = 0; m < 256; ++m)
      for (int n = 0; n < 128; ++n) {
        double ref = 0;
        for (int kk = 0; kk < 8; ++kk) ref += (double)hA[m * 8 + kk] * hB[n * 8 + kk];
        const double d = fabs(ref - hD[m * 128 + n]);
        err = fmax(err, d);
        if (n < 64) err_lo = fmax(err_lo, d); else err_hi = fmax(err_hi, d);
      }
    printf("{\"mode\": \"%s\", \"max_abs_err\": %g, \"err_cols_0_63\": %g, \"err_cols_64_127\": %g, \"err\": \"%s\"}\n",
           mode == 0 ? "B split N-wise (64 rows per CTA)" : "B whole in both CTAs", err, err_lo, err_hi,
           cudaGetErrorString(e));
  }
  return 0;
}
