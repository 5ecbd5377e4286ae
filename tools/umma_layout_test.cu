// Checks the UMMA no-swizzle smem layouts used by sgett_tc.cu: one
// tcgen05.mma.kind::tf32 (M=N=128, K=8) with A K-major or MN-major (two
// LBO/SBO assignments), B K-major; D compared with a CPU product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_layout_test tools/umma_layout_test.cu
#include <cstdint>
#include <cstdio>
#include <cmath>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) | (1ull << 46);
}

// mode 0: A K-major (LBO 128 between k-chunks, SBO 256 between 8-row groups; K = 8 -> 2 chunks)
// mode 1: A MN-major, element (m,k) at (m/4)*128 + k*16 + (m%4)*4, desc lbo=4096 sbo=128
// mode 2: same layout, desc lbo=128 sbo=4096
__global__ void k(const float* A, const float* B, float* D, int mode, int layout, uint32_t lbo, uint32_t sbo) {
  extern __shared__ __align__(1024) uint8_t sm[];
  float* sa = (float*)sm;             // 4 KB
  float* sb = (float*)(sm + 8192);    // 4 KB
  uint64_t* bar = (uint64_t*)(sm + 16384);
  uint32_t* slot = (uint32_t*)(bar + 1);
  for (int i = threadIdx.x; i < 128 * 8; i += blockDim.x) {
    int m = i / 8, kk = i % 8;
    float a = A[m * 8 + kk], b = B[m * 8 + kk];
    // K-major: row m chunk c=kk/4 at (m/8)*256 + c*128 + (m%8)*16 + (kk%4)*4
    uint32_t ok = (m / 8) * 256 + (kk / 4) * 128 + (m % 8) * 16 + (kk % 4) * 4;
    uint32_t om = layout == 1 ? (m / 4) * 128 + kk * 16 + (m % 4) * 4
                : layout == 2 ? (m / 32) * 1024 + kk * 128 + (m % 32) * 4
                : layout == 4 ? ([&] { uint32_t lg = (m / 32) * 1024 + kk * 128 + (m % 32) * 4;
                                       return lg ^ (((lg >> 7) & 7u) << 4); })()
                : layout == 5 ? ok
                : kk * 512 + m * 4;
    *(float*)((uint8_t*)sa + (mode == 0 ? ok : om)) = a;
    *(float*)((uint8_t*)sb + ok) = b;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24) |
                     ((mode != 0 ? 1u : 0u) << 15);
    uint64_t da = mode == 0 ? sdesc(su32(sa), 128, 256) : sdesc(su32(sa), lbo, sbo);
    if (layout == 4) da |= (2ull << 61);  // SWIZZLE_128B
    uint64_t db = sdesc(su32(sb), 128, 256);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)));
  }
  asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W_%=;\n\t}" ::"r"(su32(bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  int w = threadIdx.x / 32, m = threadIdx.x;
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
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main() {
  float hA[128 * 8], hB[128 * 8], hD[128 * 128];
  for (int i = 0; i < 128 * 8; ++i) { hA[i] = (float)((i * 7) % 13 - 6); hB[i] = (float)((i * 5) % 11 - 5); }
  float *A, *B, *D;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 64);
  struct { int mode, layout; uint32_t lbo, sbo; } cfg[] = {
      {0, 0, 128, 256}, {1, 1, 4096, 128}, {1, 1, 128, 4096}, {1, 1, 128, 128}, {1, 1, 16, 128},
      {1, 1, 128, 16}, {1, 1, 512, 128}, {1, 2, 1024, 128}, {1, 2, 128, 1024}, {1, 2, 512, 1024},
      {1, 2, 1024, 512}, {1, 3, 512, 128}, {1, 3, 128, 512}, {1, 3, 4096, 512}, {1, 3, 512, 4096},
      {1, 2, 4096, 1024}, {1, 2, 1024, 4096}, {1, 4, 1024, 8192}, {1, 4, 8192, 1024},
      {1, 4, 1024, 1024}, {1, 5, 128, 256}};
  for (auto c : cfg) {
    int mode = c.mode;
    cudaMemset(D, 0, sizeof hD);
    k<<<1, 128, 16384 + 64>>>(A, B, D, mode, c.layout, c.lbo, c.sbo);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 128; ++n) {
        double ref = 0;
        for (int kk = 0; kk < 8; ++kk) ref += (double)hA[m * 8 + kk] * hB[n * 8 + kk];
        maxerr = fmax(maxerr, fabs(ref - hD[m * 128 + n]));
      }
    printf("{\"mode\": %d, \"layout\": %d, \"lbo\": %u, \"sbo\": %u, \"max_abs_err\": %g, \"err\": \"%s\"}\n", mode, c.layout, c.lbo, c.sbo, maxerr, cudaGetErrorString(e));
  }
  return 0;
}
