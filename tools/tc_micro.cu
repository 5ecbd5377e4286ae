// tcgen05 kind::tf32 micro-benchmark: latency of (6 MMAs + commit + mbarrier
// wait) per iteration and back-to-back MMA throughput, one CTA, clock64.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_micro tools/tc_micro.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
__device__ __forceinline__ uint64_t sdesc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(512u >> 4) << 32) | (1ull << 46);
}

__global__ void micro(long long* out, int iters, int wait_each) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bar = (uint64_t*)(sm + 65536);
  uint32_t* slot = (uint32_t*)(bar + 2);
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((float*)sm)[i] = 0.f;
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
    uint32_t base = su32(sm);
    long long t0 = clock64();
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
      for (int j = 0; j < 6; ++j) {
        uint64_t a = sdesc(base + 256 * (j & 1)), b = sdesc(base + 16384 + 256 * (j & 1));
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                     "l"(a), "l"(b), "r"(IDESC), "r"((it | j) != 0 ? 1 : 0));
      }
      if (wait_each) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)));
        asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(su32(bar)), "r"(phase));
        phase ^= 1;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)));
    asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(su32(bar)), "r"(phase));
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 148);
  cudaFuncSetAttribute(micro, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 64);
  for (int w = 0; w < 2; ++w) {
    int iters = 2000;
    micro<<<1, 128, 65536 + 64>>>(d, iters, w);
    long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("{\"wait_each\": %d, \"cycles_per_iter_6mma\": %.1f, \"err\": \"%s\"}\n", w, (double)h / iters,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
