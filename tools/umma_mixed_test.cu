// Mixed-precision split check for the k-run SGETT: per 8 k one
// tcgen05.mma.kind::tf32 (hi*hi, hi = fp32 rounded to tf32) plus ONE
// tcgen05.mma.kind::f16 (bf16, K = 16) whose 16 k are [bf16(x) | bf16(x_lo)]
// against [bf16(y_lo) ; bf16(y)] — both cross terms of the 3xTF32 split in one
// instruction at the bf16 rate.  A operands in TMEM (tf32: one column per k;
// bf16: two k per 32-bit column, low half = even k), B K-major no-swizzle in
// shared memory.  Reports the error against an fp64 product next to the plain
// 3xTF32 (truncation split) result on the same data.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_mixed_test tools/umma_mixed_test.cu
#include <cuda_bf16.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ float rn_tf32(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}
__device__ __forceinline__ float tr_tf32(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi, int swap) {
  __nv_bfloat162 v = swap ? __floats2bfloat162_rn(hi, lo) : __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

constexpr int N = 96;

// mode 0: 3xTF32 truncation split; mode 1: tf32 + one bf16 MMA per 8 k
__global__ void k(const float* A, const float* B, float* D, int ksteps, int mode, int swap) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int KT = 8 * ksteps, CHN = KT / 4;
  uint8_t* sh = sm;                 // Y hi  (fp32 K-major)
  uint8_t* sl = sm + 32768;         // Y lo  (fp32 K-major) or the bf16 tile [ylo_b | y_b] per 8 k
  uint64_t* bar = (uint64_t*)(sm + 65536);
  uint32_t* slot = (uint32_t*)(bar + 1);
  for (int i = threadIdx.x; i < N * KT; i += blockDim.x) {
    const int n = i / KT, kk = i % KT;
    const float y = B[n * KT + kk];
    const uint32_t o = (n / 8) * (CHN * 128) + (kk / 4) * 128 + (n % 8) * 16 + (kk % 4) * 4;
    if (mode == 0) {
      *(float*)(sh + o) = y;
      *(float*)(sl + o) = y - tr_tf32(y);
    } else {
      const float yh = rn_tf32(y);
      *(float*)(sh + o) = yh;
      // bf16 tile: 8-k step j = kk / 8 has chunks 2j (y_lo) and 2j + 1 (y), 8 k x 2 B per row
      const uint32_t ob = (n / 8) * (CHN * 128) + (kk / 8) * 256 + (n % 8) * 16 + (kk % 8) * 2;
      *(__nv_bfloat16*)(sl + ob) = __float2bfloat16_rn(y - yh);
      *(__nv_bfloat16*)(sl + ob + 128) = __float2bfloat16_rn(y);
    }
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *slot;
  const int w = threadIdx.x / 32, m = threadIdx.x;
  const uint32_t ah0 = 128, al0 = 128 + KT;  // hi columns, lo / bf16 columns
  for (int j = 0; j < ksteps; ++j) {
    uint32_t h[8], l[8];
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = A[m * KT + 8 * j + i];
    if (mode == 0) {
      for (int i = 0; i < 8; ++i) {
        h[i] = __float_as_uint(x[i]);
        l[i] = __float_as_uint(x[i] - tr_tf32(x[i]));
      }
    } else {
      float xl[8];
      for (int i = 0; i < 8; ++i) {
        const float xh = rn_tf32(x[i]);
        h[i] = __float_as_uint(xh);
        xl[i] = x[i] - xh;
      }
      for (int i = 0; i < 4; ++i) {
        l[i] = pack_bf16(x[2 * i], x[2 * i + 1], swap);
        l[4 + i] = pack_bf16(xl[2 * i], xl[2 * i + 1], swap);
      }
    }
    const uint32_t base = tmem + ((uint32_t)(w * 32) << 16);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(base + ah0 + 8 * j),
                 "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3]), "r"(h[4]), "r"(h[5]), "r"(h[6]), "r"(h[7]));
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(base + al0 + 8 * j),
                 "r"(l[0]), "r"(l[1]), "r"(l[2]), "r"(l[3]), "r"(l[4]), "r"(l[5]), "r"(l[6]), "r"(l[7]));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    const uint32_t id_tf32 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    const uint32_t id_bf16 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    for (int j = 0; j < ksteps; ++j) {
      const uint64_t bh = sdesc(su32(sh) + 256 * j, 128, CHN * 128);
      const uint64_t bl = sdesc(su32(sl) + 256 * j, 128, CHN * 128);
#define MMA(KIND, AT, BD, ID, ACC)                                                                               \
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::" KIND            \
               " [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),                                                        \
               "r"(AT), "l"(BD), "r"(ID), "r"(ACC))
      MMA("tf32", tmem + ah0 + 8 * j, bh, id_tf32, j);
      if (mode == 0) {
        MMA("tf32", tmem + ah0 + 8 * j, bl, id_tf32, 1);
        MMA("tf32", tmem + al0 + 8 * j, bh, id_tf32, 1);
      } else {
        MMA("f16", tmem + al0 + 8 * j, bl, id_bf16, 1);
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)));
  }
  asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W_%=;\n\t}" ::"r"(su32(bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(tmem + ((uint32_t)(w * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 16; ++i) D[m * N + c0 + i] = __uint_as_float(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  const int KS = 10, KT = 8 * KS;
  static float hA[128 * KT], hB[N * KT], hD[128 * N];
  srand(7);
  for (int i = 0; i < 128 * KT; ++i) hA[i] = (float)(2.0 * rand() / RAND_MAX - 1.0);
  for (int i = 0; i < N * KT; ++i) hB[i] = (float)(2.0 * rand() / RAND_MAX - 1.0);
  float *A, *B, *D;
  cudaMalloc(&A, sizeof hA);
  cudaMalloc(&B, sizeof hB);
  cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 64);
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(D, 0, sizeof hD);
    k<<<1, 128, 65536 + 64>>>(A, B, D, KS, mode ? 1 : 0, mode == 2);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
    double maxerr = 0, bias = 0, rms = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int kk = 0; kk < KT; ++kk) ref += (double)hA[m * KT + kk] * hB[n * KT + kk];
        const double d = hD[m * N + n] - ref;
        maxerr = fmax(maxerr, fabs(d));
        bias += d;
        rms += d * d;
      }
    printf("{\"scheme\": \"%s\", \"K\": %d, \"max_abs_err\": %g, \"rms_err\": %g, \"mean_err\": %g, \"err\": \"%s\"}\n",
           mode == 0 ? "3xtf32_trunc" : (mode == 1 ? "tf32+bf16 (low half = even k)" : "tf32+bf16 (low half = odd k)"), KT,
           maxerr, sqrt(rms / (128 * N)), bias / (128 * N), cudaGetErrorString(e));
  }
  return 0;
}
