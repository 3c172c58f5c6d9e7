// Dev test (GPU): TMA-load one MN-major 32x32 fp32 box with SWIZZLE_128B and
// one tcgen05 MMA (M=128, N=64, K=8) with an MN-major B operand; prints
// diagnostics.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/mnt mn_tma_test.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cmath>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void tma_box(const __grid_constant__ CUtensorMap map, float* out, int x, int y) {
  __shared__ __align__(1024) float buf[32 * 32];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(4096) : "memory");
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(smem_u32(buf)), "l"(&map), "r"(x), "r"(y), "r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred P;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n}" ::"r"(smem_u32(&bar)) : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int K = 64, M = 64;  // stored K x M (M contiguous)
  std::vector<float> h(K * M);
  for (int k = 0; k < K; ++k) for (int m = 0; m < M; ++m) h[k * M + m] = k * 1000 + m;
  float *d, *o;
  cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 4096);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)M, (cuuint64_t)K};
  cuuint64_t strides[1] = {(cuuint64_t)M * 4};
  cuuint32_t box[2] = {32, 32}, estr[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  tma_box<<<1, 128>>>(map, o, 32, 8);  // MN offset 32, K offset 8
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel %s\n", cudaGetErrorString(e));
  std::vector<float> out(1024);
  cudaMemcpy(out.data(), o, 4096, cudaMemcpyDeviceToHost);
  // row r of smem (128 B) should hold K index 8 + r, MN 32..63 (swizzled in 16B units)
  for (int r = 0; r < 3; ++r) {
    printf("row %d:", r);
    for (int c = 0; c < 32; c += 4) printf(" %g", out[r * 32 + c]);
    printf("\n");
  }
  return 0;
}
