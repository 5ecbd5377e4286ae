// How does tcgen05.mma.kind::tf32 read a raw fp32 operand (low 13 mantissa
// bits set)?  Same harness as umma_tmem_a_test.cu (A in TMEM, B K-major in
// smem), fed full-precision fp32 values; the GPU product is compared with CPU
// products of (a) truncated and (b) round-to-nearest tf32 inputs.  If the
// tensor core truncates, a raw fp32 tile IS the hi part of a 3xTF32 split
// (hi = x & 0xffffe000) and only lo = x - hi needs computing.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tf32_trunc_test tools/tf32_trunc_test.cu
#include <cstdint>
#include <cstdio>
#include <cmath>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) | (1ull << 46);
}

__global__ void k(const float* A, const float* B, float* D, int ksteps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  float* sb = (float*)sm;  // B: 128 rows x (8*ksteps) k, K-major core matrices
  uint64_t* bar = (uint64_t*)(sm + 16384);
  uint32_t* slot = (uint32_t*)(bar + 1);
  const int KT = 8 * ksteps, CHN = KT / 4;
  for (int i = threadIdx.x; i < 128 * KT; i += blockDim.x) {
    int n = i / KT, kk = i % KT;
    uint32_t ok = (n / 8) * (CHN * 128) + (kk / 4) * 128 + (n % 8) * 16 + (kk % 4) * 4;
    *(float*)((uint8_t*)sb + ok) = B[n * KT + kk];
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = *slot;
  const int w = threadIdx.x / 32, m = threadIdx.x;
  // A row m -> TMEM lane m, columns 128 + k
  for (int j = 0; j < ksteps; ++j) {
    uint32_t r[8];
    for (int i = 0; i < 8; ++i) r[i] = __float_as_uint(A[m * KT + 8 * j + i]);
    uint32_t ta = tmem + ((uint32_t)(w * 32) << 16) + 128 + 8 * j;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                 ::"r"(ta), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    for (int j = 0; j < ksteps; ++j) {
      uint64_t db = sdesc(su32(sb) + 256 * j, 128, CHN * 128);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                   ::"r"(tmem), "r"(tmem + 128 + 8 * j), "l"(db), "r"(idesc), "r"(j));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)));
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
    for (int i = 0; i < 16; ++i) D[m * 128 + c0 + i] = __uint_as_float(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}


#include <cstring>
static float trunc_tf32(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xffffe000u; memcpy(&x, &u, 4); return x; }
static float rn_tf32(float x) { uint32_t u; memcpy(&u, &x, 4); u += 0x1000u; u &= 0xffffe000u; memcpy(&x, &u, 4); return x; }

int main() {
  const int KS = 2, KT = 8 * KS;
  static float hA[128 * KT], hB[128 * KT], hD[128 * 128];
  uint64_t s = 12345;
  auto rnd = [&]() { s = s * 6364136223846793005ull + 1442695040888963407ull; return (float)((double)(s >> 11) / 9007199254740992.0 * 2.0 - 1.0); };
  for (int i = 0; i < 128 * KT; ++i) { hA[i] = rnd(); hB[i] = rnd(); }
  float *A, *B, *D;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 64);
  k<<<1, 128, 16384 + 64>>>(A, B, D, KS);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
  double e_tr = 0, e_rn = 0, e_fp = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 128; ++n) {
      double rt = 0, rr = 0, rf = 0;
      for (int kk = 0; kk < KT; ++kk) {
        float a = hA[m * KT + kk], b = hB[n * KT + kk];
        rt += (double)trunc_tf32(a) * trunc_tf32(b);
        rr += (double)rn_tf32(a) * rn_tf32(b);
        rf += (double)a * b;
      }
      double d = hD[m * 128 + n];
      e_tr = fmax(e_tr, fabs(d - rt)); e_rn = fmax(e_rn, fabs(d - rr)); e_fp = fmax(e_fp, fabs(d - rf));
    }
  printf("{\"vs_truncated\": %g, \"vs_round_nearest\": %g, \"vs_fp32_exact\": %g, \"err\": \"%s\"}\n", e_tr, e_rn, e_fp, cudaGetErrorString(e));
  return 0;
}
