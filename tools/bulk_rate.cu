// Throughput of shared->global bulk requests per SM: cp.reduce.async.bulk
// .add.f64 (the DGETT bulk-add epilogue) vs plain cp.async.bulk stores, by
// request size, 8 issuing warps per CTA, one CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bulk_rate tools/bulk_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <bool RED>
__global__ void __launch_bounds__(256, 1) bulk_kernel(double* out, int bytes, int reps) {
  extern __shared__ __align__(128) double sm[];
  for (int i = threadIdx.x; i < 65536 / 8; i += blockDim.x) sm[i] = 1.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // each CTA owns 8 MB of out, each warp 1 MB
  char* base = reinterpret_cast<char*>(out) + ((size_t)blockIdx.x * 8 + warp) * (1 << 20);
  const uint32_t src = (uint32_t)__cvta_generic_to_shared(sm) + warp * 8192;
  if (lane == 0) {
    int off = 0;
    for (int r = 0; r < reps; ++r) {
      char* dst = base + off;
      if (RED)
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(dst),
                     "r"(src), "r"(bytes) : "memory");
      else
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src),
                     "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      off += bytes;
      if (off + bytes > (1 << 20)) off = 0;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, (size_t)sms * 8 << 20);
  cudaMemset(out, 0, (size_t)sms * 8 << 20);
  cudaFuncSetAttribute(bulk_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(bulk_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  for (int grid : {1, 8, sms})
  for (int red = 1; red >= 0; --red)
    for (int bytes : {256, 1024, 4096}) {
      const int reps = 2048;  // per warp: 2048 requests (wrapping in the warp's 1 MB)
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      auto k = red ? bulk_kernel<true> : bulk_kernel<false>;
      k<<<grid, 256, 65536>>>(out, bytes, 16);
      cudaEventRecord(e0);
      k<<<grid, 256, 65536>>>(out, bytes, reps);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double tot = (double)grid * 8 * reps * bytes;
      const double per_sm_ns = ms * 1e6;
      printf("{\"ctas\": %d, \"op\": \"%s\", \"bytes\": %d, \"reqs_per_warp\": %d, \"GB_s\": %.1f, \"ns_per_req_per_sm\": %.2f, "
             "\"B_per_ns_per_sm\": %.1f, \"err\": \"%s\"}\n",
             grid, red ? "reduce_add_f64" : "store", bytes, reps, tot / ms / 1e6, per_sm_ns / (8.0 * reps),
             tot / grid / per_sm_ns, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
