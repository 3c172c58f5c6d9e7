// peaks.cu — measured B200 compute peaks used as roofline denominators
// (bench.py reads profiles/r02_peaks.json).  MEASURED_PEAKS.json carries the
// driver's HBM and cuBLAS-bf16 figures only; the hot paths here run FP32
// SIMT (row programs: FFMA, and the packed FFMA2 of sm_100a) and the tf32
// tensor-core kind (3xTF32 GEMMs), so those peaks are measured the same way:
// one kernel per unit, every SM busy, CUDA events around a long run.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu
//   tools/peaks > profiles/r02_peaks.json
//
// * ffma:  8 independent FFMA chains per thread, 148 x 8 CTAs x 256 threads
// * ffma2: the same with fma.rn.f32x2 (one instruction = two lanes' FMAs)
// * tcgen05 kind::tf32 / kind::f16 (bf16): one CTA per SM, one elected
//   thread issuing M=128 x N=256 MMAs back to back on smem-resident operands
//   (128B-swizzled K-major descriptors, as sf_gemm_tc.cu), accumulator in TMEM.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));    \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3f + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 1234.5f) out[0] = s;
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long x, unsigned long long a,
                                                    unsigned long long b) {
  unsigned long long r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(x), "l"(a), "l"(b));
  return r;
}

__global__ void ffma2_kernel(float* out, int iters, float a, float b) {
  unsigned long long x[8];
  const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
  const unsigned long long av = *(const unsigned long long*)&a2;
  const unsigned long long bv = *(const unsigned long long*)&b2;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float2 v = make_float2(threadIdx.x * 1e-3f + j, j * 0.5f);
    x[j] = *(unsigned long long*)&v;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = ffma2(x[j], av, bv);
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float2 v = *(float2*)&x[j];
    s += v.x + v.y;
  }
  if (s == 1234.5f) out[0] = s;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(1024u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

template <bool TF32>
__global__ void __launch_bounds__(128, 1) mma_kernel(int iters, unsigned long long* cycles) {
  constexpr int BM = 128, BN = 256;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  // A: 128 rows x 128 B, B: 256 rows x 128 B (one k-block of 32 tf32 / 64 bf16)
  uint32_t* fill = (uint32_t*)smem;
  for (int i = threadIdx.x; i < (BM + BN) * 32; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u;
    fill[i] = 0x3F800000u | (h >> 9);  // floats in [1, 2) (bf16 pairs likewise finite)
  }
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(&tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_slot;
  if (threadIdx.x == 0) {
    // c = f32; a/b = tf32 (2) or bf16 (1); K-major; N >> 3, M >> 4
    const uint32_t fmt = TF32 ? 2u : 1u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + BM * 128);
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {  // 4 k-steps of 32 B: K = 8 (tf32) or 16 (bf16)
        const uint64_t da = sw128_desc(a + 32u * j), db = sw128_desc(b + 32u * j);
        const uint32_t acc = (i | j) != 0;
        if (TF32)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
              "l"(da), "l"(db), "r"(idesc), "r"(acc));
        else
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
              "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(&bar))
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred P;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t"
        "@!P bra W;\n}" ::"r"(smem_u32(&bar))
        : "memory");
    if (blockIdx.x == 0) cycles[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

template <class F>
static float time_ms(F launch, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();  // warm-up
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  int sms = 0, clk_khz = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  float* out;
  unsigned long long* cyc;
  CK(cudaMalloc(&out, 16));
  CK(cudaMalloc(&cyc, 16));
  const int iters = 1 << 16, blocks = sms * 8, threads = 256;
  const double ffma_flops = 2.0 * 8 * iters * (double)blocks * threads;
  float ms1 = time_ms([&] { ffma_kernel<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f); }, 5);
  float ms2 = time_ms([&] { ffma2_kernel<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f); }, 5);
  CK(cudaGetLastError());
  const int smem = (128 + 256) * 128 + 1024;
  CK(cudaFuncSetAttribute(mma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(mma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int mi = 1 << 15;
  // per MMA: 2 * 128 * 256 * K, K = 8 (tf32) / 16 (bf16); 4 MMAs per iteration
  float mt = time_ms([&] { mma_kernel<true><<<sms, 128, smem>>>(mi, cyc); }, 3);
  unsigned long long c_tf32 = 0;
  CK(cudaMemcpy(&c_tf32, cyc, 8, cudaMemcpyDeviceToHost));
  float mb = time_ms([&] { mma_kernel<false><<<sms, 128, smem>>>(mi, cyc); }, 3);
  unsigned long long c_bf16 = 0;
  CK(cudaMemcpy(&c_bf16, cyc, 8, cudaMemcpyDeviceToHost));
  CK(cudaGetLastError());
  const double tf32_flops = 2.0 * 128 * 256 * 8 * 4.0 * mi * sms;
  const double bf16_flops = 2.0 * 128 * 256 * 16 * 4.0 * mi * sms;
  printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f,\n", sms, clk_khz / 1e3);
  printf(" \"ffma_tflops\": %.2f, \"ffma2_tflops\": %.2f,\n", ffma_flops / ms1 / 1e9,
         ffma_flops * 2 / ms2 / 1e9);
  printf(" \"tcgen05_tf32_tflops\": %.1f, \"tcgen05_bf16_tflops\": %.1f,\n",
         tf32_flops / mt / 1e9, bf16_flops / mb / 1e9);
  printf(" \"tf32_cycles_per_mma_128x256x8\": %.2f, \"bf16_cycles_per_mma_128x256x16\": %.2f,\n",
         (double)c_tf32 / (4.0 * mi), (double)c_bf16 / (4.0 * mi));
  printf(" \"method\": \"CUDA events around %d-rep runs after one warm-up; ffma: %d CTAs x %d "
         "threads x 8 chains x %d iters; mma: %d CTAs, one thread issuing %d tcgen05.mma "
         "(M=128, N=256) on smem-resident 128B-swizzled operands\"}\n",
         5, blocks, threads, iters, sms, 4 * mi);
  return 0;
}
