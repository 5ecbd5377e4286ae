// Peak-throughput microbenchmarks for the pipes the GETT kernels can use on
// B200 (sm_100a): FP64 DFMA (SIMT), FP64 DMMA (mma.sync f64 shapes), FP32
// FFMA, and an HBM copy.  Prints one JSON object per measurement.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks tools/peaks.cu
// These numbers are the FP64/FP32 roofline denominators (MEASURED_PEAKS.json
// carries only HBM and bf16), see DESIGN.md.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double s) {
  double acc[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc[i] = fma(acc[i], s, 1e-9);
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) r += acc[i];
  if (r == 12345.678) out[0] = r;
}

template <int CHAINS>
__global__ void ffma_loop(float* out, int iters, float s) {
  float acc[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc[i] = fmaf(acc[i], s, 1e-9f);
  }
  float r = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) r += acc[i];
  if (r == 12345.678f) out[0] = r;
}

// m8n8k4: A 1 f64, B 1 f64, C/D 2 f64 per lane; 256 MAC per warp-op
template <int CHAINS>
__global__ void dmma884_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-6;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) r += c[i][0] + c[i][1];
  if (r == 12345.678) out[0] = r;
}

// m16n8k4: A 2, B 1, C 4 per lane; 512 MAC per warp-op
template <int CHAINS>
__global__ void dmma1684_loop(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-6, a1 = a0 * 0.5, b = 1.0 - threadIdx.x * 1e-6;
  double c[CHAINS][4];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) r += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (r == 12345.678) out[0] = r;
}

// m16n8k16: A 8, B 4, C 4 per lane; 2048 MAC per warp-op
template <int CHAINS>
__global__ void dmma16816_loop(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-6;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-6;
  double c[CHAINS][4];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                   "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double r = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) r += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (r == 12345.678) out[0] = r;
}

__global__ void copy_kernel(const float4* __restrict__ in, float4* __restrict__ out, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = in[i];
}

template <typename F>
static float time_ms(F launch, int reps) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  launch();  // warm
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  printf("{\"device\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\"}\n", p.name, sms, p.major, p.minor);
  double* dout; float* fout; CK(cudaMalloc(&dout, 64)); CK(cudaMalloc(&fout, 64));
  const int iters = 4096;
  for (int bpsm : {1, 2, 4, 8}) {
    for (int threads : {128, 256}) {
      int blocks = sms * bpsm;
      double macs = (double)blocks * threads * iters * 8;
      float ms = time_ms([&] { dfma_loop<8><<<blocks, threads>>>(dout, iters, 0.999999); }, 5);
      printf("{\"op\": \"dfma\", \"blocks_per_sm\": %d, \"threads\": %d, \"tflops\": %.3f}\n", bpsm, threads, 2 * macs / ms / 1e9);
      macs = (double)blocks * threads * iters * 8;
      ms = time_ms([&] { ffma_loop<8><<<blocks, threads>>>(fout, iters, 0.999999f); }, 5);
      printf("{\"op\": \"ffma\", \"blocks_per_sm\": %d, \"threads\": %d, \"tflops\": %.3f}\n", bpsm, threads, 2 * macs / ms / 1e9);
      double warps = (double)blocks * threads / 32;
      ms = time_ms([&] { dmma884_loop<4><<<blocks, threads>>>(dout, iters); }, 5);
      printf("{\"op\": \"dmma_m8n8k4\", \"blocks_per_sm\": %d, \"threads\": %d, \"tflops\": %.3f}\n", bpsm, threads, 2 * warps * iters * 4 * 256 / ms / 1e9);
      ms = time_ms([&] { dmma1684_loop<4><<<blocks, threads>>>(dout, iters); }, 5);
      printf("{\"op\": \"dmma_m16n8k4\", \"blocks_per_sm\": %d, \"threads\": %d, \"tflops\": %.3f}\n", bpsm, threads, 2 * warps * iters * 4 * 512 / ms / 1e9);
      ms = time_ms([&] { dmma16816_loop<2><<<blocks, threads>>>(dout, iters / 4); }, 5);
      printf("{\"op\": \"dmma_m16n8k16\", \"blocks_per_sm\": %d, \"threads\": %d, \"tflops\": %.3f}\n", bpsm, threads, 2 * warps * (iters / 4) * 2 * 2048 / ms / 1e9);
    }
  }
  size_t n = (size_t)1 << 28;  // 4 GiB of float4? no: 2^28 float4 = 4 GiB; use 2^26 -> 1 GiB each
  n >>= 2;
  float4 *x, *y; CK(cudaMalloc(&x, n * 16)); CK(cudaMalloc(&y, n * 16));
  CK(cudaMemset(x, 0, n * 16));
  float ms = time_ms([&] { copy_kernel<<<sms * 8, 512>>>(x, y, n); }, 10);
  printf("{\"op\": \"hbm_copy\", \"gbs\": %.1f}\n", 2.0 * n * 16 / ms / 1e6);
  return 0;
}
