// tcgen05.mma issue-rate micro-benchmark: cycles per back-to-back MMA for
// kind::tf32 / kind::f16, M = 128, N in {64, 128, 256}, A from shared memory
// or from TMEM, B from shared memory (K-major, no swizzle).  One CTA per SM
// (grid 148), one elected thread issues; block 0's clock64 span is reported.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_rate tools/mma_rate.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
         (1ull << 46);
}

template <int N, bool ATM, bool F16>
__global__ void rate(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bar = (uint64_t*)(sm + 98304);
  uint32_t* slot = (uint32_t*)(bar + 2);
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) ((float*)sm)[i] = 0.f;
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
  constexpr uint32_t AF = F16 ? 0u : 2u;
  constexpr uint32_t IDESC =
      (1u << 4) | (AF << 7) | (AF << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
  if (threadIdx.x == 0) {
    const uint32_t base = su32(sm);
    // A: 128 rows x 32 B of K at base (SBO 256: two 16 B chunks per 8-row group)
    // B: N rows x 32 B at base + 32 KB
    const uint64_t ad = sdesc(base, 128, 256), bd = sdesc(base + 32768, 128, 256);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#define MMA_TM(K) asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t" \
                     "tcgen05.mma.cta_group::1.kind::" K " [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem), \
                     "r"(tmem + 256), "l"(bd), "r"(IDESC), "r"(it))
#define MMA_SS(K) asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t" \
                     "tcgen05.mma.cta_group::1.kind::" K " [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), \
                     "l"(ad), "l"(bd), "r"(IDESC), "r"(it))
      if (ATM) {
        if (F16) MMA_TM("f16"); else MMA_TM("tf32");
      } else {
        if (F16) MMA_SS("f16"); else MMA_SS("tf32");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar)));
    asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W_%=;\n\t}" ::"r"(su32(bar)));
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, bool ATM, bool F16>
void run(long long* d) {
  auto k = rate<N, ATM, F16>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304 + 64);
  const int iters = 4096;
  k<<<148, 128, 98304 + 64>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double cyc = (double)h[0] / iters;
  const double kk = F16 ? 16 : 8;
  printf("{\"kind\": \"%s\", \"N\": %d, \"a_from\": \"%s\", \"cycles_per_mma\": %.2f, "
         "\"max_block_cycles_per_mma\": %.2f, \"mac_per_clk\": %.0f, \"err\": \"%s\"}\n",
         F16 ? "f16" : "tf32", N, ATM ? "tmem" : "smem", cyc, (double)mx / iters,
         128.0 * N * kk / cyc, cudaGetErrorString(e));
}


// The SGETT kernel's MMA issue pattern without its producers: per k-block 2
// k-steps x (hi*hi, lo*hi, hi*lo), A hi/lo in TMEM at column abase + 32 s
// (+16 for lo) of stage s, B hi/lo K-major tiles per stage in smem (SBO 512),
// one tcgen05.commit per k-block onto the stage's mbarrier (never waited).
template <int ABASE, bool COMMIT>
__global__ void pattern(long long* out, int kblocks) {
  extern __shared__ __align__(1024) uint8_t sm[];
  constexpr int STG = 8, TB = 8192, SB = 3 * TB;
  uint64_t* bar = (uint64_t*)(sm + STG * SB);
  uint32_t* slot = (uint32_t*)(bar + STG + 1);
  for (int i = threadIdx.x; i < STG * SB / 4; i += blockDim.x) ((float*)sm)[i] = 0.f;
  if (threadIdx.x == 0) {
    for (int i = 0; i <= STG; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + i)));
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
  constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
  if (threadIdx.x == 0) {
    const uint32_t base = su32(sm);
    long long t0 = clock64();
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % STG;
      const uint32_t sb = base + s * SB;
      for (int j = 0; j < 2; ++j) {
        const uint32_t ah = tmem + ABASE + s * 32 + 8 * j, al = ah + 16;
        const uint64_t bh = sdesc(sb + TB + 256 * j, 128, 512), bl = sdesc(sb + 2 * TB + 256 * j, 128, 512);
#define MMA_P(A, B, ACC) asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t" \
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem), \
                     "r"(A), "l"(B), "r"(IDESC), "r"((int)(ACC)))
        MMA_P(ah, bh, (kb | j) != 0);
        MMA_P(al, bh, 1);
        MMA_P(ah, bl, 1);
      }
      if (COMMIT)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar + s)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar + STG)));
    asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W_%=;\n\t}" ::"r"(su32(bar + STG)));
    out[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int ABASE, bool COMMIT>
void runp(long long* d) {
  auto k = pattern<ABASE, COMMIT>;
  const int smem = 8 * 3 * 8192 + 128;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int kb = 2048;
  k<<<148, 128, smem>>>(d, kb);
  cudaError_t e = cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("{\"pattern\": \"sgett_tc k-block\", \"a_col_base\": %d, \"commit\": %d, \"cycles_per_kblock\": %.1f, "
         "\"ideal\": 384, \"err\": \"%s\"}\n", ABASE, (int)COMMIT, (double)h / kb, cudaGetErrorString(e));
}

// the k-run kernel's pattern (sgett_kr.cu): per k-block KR/8 k-steps x 3
// MMAs, M = 128, N = NT, A from TMEM, B K-major no-swizzle with SBO = KR/4 x 128
// COMMIT2: two commits per k-block (the kernel frees an operand slot and a
// TMEM slot); STW: the other three warps keep writing TMEM columns (the split
// warps' tcgen05.st traffic) while the MMAs run
template <int NT, int KR, bool RND, int FENCE = 0, bool COMMIT2 = false, bool STW = false>
__global__ void pattern_kr(long long* out, int kblocks) {
  extern __shared__ __align__(1024) uint8_t sm[];
  constexpr int STG = KR > 40 ? 2 : 4, TB = NT * KR * 4, SB = 2 * TB;
  uint64_t* bar = (uint64_t*)(sm + STG * SB);
  uint32_t* slot = (uint32_t*)(bar + STG + 1);
  for (int i = threadIdx.x; i < STG * SB / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u + 12345u;
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    ((float*)sm)[i] = RND ? ((float)(h & 0xffffff) / 16777216.0f - 0.5f) : 0.f;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i <= STG; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + i)));
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
  if (RND) {  // random A columns in TMEM (each warp its lane quarter)
    const int w = threadIdx.x >> 5;
    for (int c = 0; c < 384; c += 8) {
      uint32_t v[8];
      for (int j = 0; j < 8; ++j) {
        uint32_t h = (uint32_t)(threadIdx.x * 977 + c * 131 + j * 7919) * 2654435761u;
        h ^= h >> 15;
        v[j] = __float_as_uint((float)(h & 0xffffff) / 16777216.0f - 0.5f);
      }
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tmem + ((uint32_t)(32 * w) << 16) + 128 + c),
                   "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NT >> 3) << 17) | ((128u >> 4) << 24);
  volatile __shared__ int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (STW && threadIdx.x >= 32) {
    // warps 1-3: tcgen05.st 32x32b.x16 into columns 448.. (not read by the MMAs)
    const int w = threadIdx.x >> 5;
    uint32_t v[16];
    for (int j = 0; j < 16; ++j) v[j] = threadIdx.x * 16 + j;
    while (!stop) {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(tmem + ((uint32_t)(32 * w) << 16) + 448u),
                   "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                   "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) {
    const uint32_t base = su32(sm);
    long long t0 = clock64();
    for (int kb = 0; kb < kblocks; ++kb) {
      const int s = kb % STG;
      const uint32_t sb = base + s * SB;
      // FENCE n: every n-th k-block waits on an (already completed) mbarrier
      // phase and issues tcgen05.fence::after_thread_sync, as the kernels do
      // after their `ready` waits
      if (FENCE && kb % FENCE == 0) {
        asm volatile("{\n\t.reg .pred P1;\nWF_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 1;\n\t@!P1 bra WF_%=;\n\t}" ::"r"(su32(bar + STG)));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      for (int j = 0; j < KR / 8; ++j) {
        const uint32_t ah = tmem + 128 + s * 2 * KR + 8 * j, al = ah + KR;
        const uint64_t bh = sdesc(sb + 256 * j, 128, KR / 4 * 128), bl = sdesc(sb + TB + 256 * j, 128, KR / 4 * 128);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                     "r"(ah), "l"(bh), "r"(IDESC), "r"((int)((kb | j) != 0)));
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                     "r"(al), "l"(bh), "r"(IDESC), "r"(1));
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                     "r"(ah), "l"(bl), "r"(IDESC), "r"(1));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar + s)));
      if (COMMIT2)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar + (s + 1) % STG)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar + STG)));
    asm volatile("{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W_%=;\n\t}" ::"r"(su32(bar + STG)));
    out[blockIdx.x] = clock64() - t0;
    stop = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int NT, int KR, bool RND = false, int FENCE = 0, bool COMMIT2 = false, bool STW = false>
void runkr(long long* d) {
  auto k = pattern_kr<NT, KR, RND, FENCE, COMMIT2, STW>;
  const int smem = (KR > 40 ? 2 : 4) * 2 * NT * KR * 4 + 128;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int kb = 1024;
  k<<<148, 128, smem>>>(d, kb);
  cudaError_t e = cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("{\"pattern\": \"sgett_kr k-block\", \"NT\": %d, \"KR\": %d, \"random_data\": %d, \"fence_every\": %d, \"commit2\": %d, \"tmem_st_warps\": %d, \"cycles_per_kblock\": %.1f, "
         "\"ideal\": %.1f, \"err\": \"%s\"}\n", NT, KR, (int)RND, FENCE, (int)COMMIT2, STW ? 3 : 0, (double)h / kb, 3.0 * 128 * NT * KR / 2048.0,
         cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 148);
  runkr<96, 40>(d);
  runkr<96, 40, false, 1>(d);
  runkr<96, 40, false, 2>(d);
  runkr<96, 40, false, 4>(d);
  runkr<96, 40, false, 0, true>(d);
  runkr<96, 40, false, 0, false, true>(d);
  runkr<96, 40, false, 1, true, true>(d);
  runkr<96, 40, false, 1, false, true>(d);
  runkr<96, 80, false, 1, false, true>(d);
  runkr<96, 40, true>(d);
  runkr<128, 40, true>(d);
  runkr<128, 40>(d);
  runkr<96, 16>(d);
  runkr<128, 32>(d);
  run<96, true, false>(d);
  run<64, false, false>(d);
  run<128, false, false>(d);
  run<256, false, false>(d);
  run<64, true, false>(d);
  run<128, true, false>(d);
  run<256, true, false>(d);
  run<128, false, true>(d);
  run<256, false, true>(d);
  run<128, true, true>(d);
  run<256, true, true>(d);
  runp<128, true>(d);
  runp<128, false>(d);
  runp<256, true>(d);
  return 0;
}
