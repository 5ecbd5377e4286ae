// DMMA (mma.sync.m8n8k4.f64) issue rate vs warps per SM: does one warp per
// sub-partition reach the FP64 tensor peak, or does it take two?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_rate tools/dmma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC>
__global__ void dmma_loop(double* out, int iters) {
  double acc[ACC][2];
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
#pragma unroll
  for (int i = 0; i < ACC; ++i) acc[i][0] = acc[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1234.5) out[0] = s;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 20000;
  for (int warps : {1, 2, 4, 8, 12, 16}) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dmma_loop<32><<<sms, warps * 32>>>(out, 100);
    cudaEventRecord(e0);
    dmma_loop<32><<<sms, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 32 * (double)iters * warps * 32 / 32 * sms;
    printf("{\"warps_per_sm\": %d, \"acc\": 32, \"tflops\": %.2f}\n", warps, flops / ms / 1e9);
  }
  return 0;
}
