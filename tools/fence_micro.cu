// cost of fence.proxy.async.shared::cta + bar.sync per iteration (128 threads)
#include <cstdio>
#include <cstdint>
__global__ void k(long long* out, int iters, int mode) {
  __shared__ float4 buf[4096];
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    buf[(threadIdx.x * 8 + it) & 4095] = make_float4(it, 1, 2, 3);
    if (mode == 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (mode == 2) asm volatile("fence.proxy.async;" ::: "memory");
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = clock64() - t0;
}
int main() {
  long long* d; cudaMalloc(&d, 8);
  for (int m = 0; m < 3; ++m) {
    k<<<1, 128>>>(d, 10000, m); long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("{\"mode\": %d, \"cycles_per_iter\": %.1f}\n", m, h / 10000.0);
  }
}
