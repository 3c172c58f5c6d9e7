// Dev test (GPU): one tcgen05.mma kind::tf32 (M=128, N=64, K=8) with A
// K-major and B MN-major (or K-major), operands TMA-loaded with SWIZZLE_128B.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o mnm mn_mma_test.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cmath>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t kdesc(uint32_t s) {
  return (uint64_t)((s >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint64_t mndesc(uint32_t s, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((s >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (1ull << 61);
}
__device__ void tma(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(su(dst)), "l"(m), "r"(x), "r"(y), "r"(su(bar)) : "memory");
}
__device__ void wait(uint64_t* bar, uint32_t ph) {
  asm volatile("{\n\t.reg .pred P;\nW%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W%=;\n}" ::"r"(su(bar)), "r"(ph) : "memory");
}

__global__ void one_mma(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                        float* out, int bmn, uint32_t lbo, uint32_t sbo) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* A = sm;            // 128 x 32 fp32 K-major: 16 KB
  uint8_t* B = sm + 16384;    // 64 x 32: 8 KB (K-major) or 2 boxes of 32x32 (MN-major)
  uint64_t* bar = (uint64_t*)(sm + 32768);
  uint64_t* done = bar + 1;
  uint32_t* tslot = (uint32_t*)(bar + 2);
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(done)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = *tslot;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar)), "r"(16384 + 8192) : "memory");
    tma(A, &ta, bar, 0, 0);
    if (bmn) { tma(B, &tb, bar, 0, 0); tma(B + 4096, &tb, bar, 32, 0); }
    else tma(B, &tb, bar, 0, 0);
    wait(bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((bmn ? 1u : 0u) << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
    uint64_t da = kdesc(su(A));
    uint64_t db = bmn ? mndesc(su(B), lbo, sbo) : kdesc(su(B));
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                 ::"r"(tmem), "l"(da), "l"(db), "r"(idesc));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(done)) : "memory");
  }
  __syncwarp();
  wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < 64; c0 += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 8; ++i) out[(warp * 32 + lane) * 64 + c0 + i] = __uint_as_float(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

static CUtensorMap mk(float* p, int rows, int cols, int box_rows, CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t st[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)box_rows}, es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, p, dims, st, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) printf("encode error %d\n", (int)r);
  return m;
}

int main(int argc, char** argv) {
  const int M = 128, N = 64, K = 32;
  std::vector<float> a(M * K), b(N * K), bt(K * N);
  srand(1);
  for (auto& v : a) v = (float)(rand() % 7 - 3);
  for (int n = 0; n < N; ++n) for (int k = 0; k < K; ++k) { b[n * K + k] = (float)(rand() % 5 - 2); bt[k * N + n] = b[n * K + k]; }
  float *da, *db, *dbt, *dout;
  cudaMalloc(&da, a.size() * 4); cudaMalloc(&db, b.size() * 4); cudaMalloc(&dbt, bt.size() * 4); cudaMalloc(&dout, M * N * 4);
  cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dbt, bt.data(), bt.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap ta = mk(da, M, K, 128), tbk = mk(db, N, K, 64), tbm = mk(dbt, K, N, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  cudaFuncSetAttribute(one_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  uint32_t cfg[][2] = {{4096, 512}, {512, 4096}, {4096, 1024}, {1024, 4096}, {4096, 256}};
  for (int t = -1; t < 5; ++t) {
    int bmn = t >= 0;
    cudaMemset(dout, 0, M * N * 4);
    one_mma<<<1, 128, 40000>>>(ta, bmn ? tbm : tbk, dout, bmn, bmn ? cfg[t][0] : 0, bmn ? cfg[t][1] : 0);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> o(M * N);
    cudaMemcpy(o.data(), dout, M * N * 4, cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
      double s = 0; for (int k = 0; k < 8; ++k) s += (double)a[m * K + k] * b[n * K + k];
      err = fmax(err, fabs(s - o[m * N + n])); mx = fmax(mx, fabs(o[m * N + n]));
    }
    printf("bmn=%d lbo=%u sbo=%u: %s maxabs %g err %g\n", bmn, bmn ? cfg[t][0] : 0, bmn ? cfg[t][1] : 0, cudaGetErrorString(e), mx, err);
  }
  return 0;
}
