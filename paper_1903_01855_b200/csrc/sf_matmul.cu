// sf_matmul.cu — rank-2 matmul (reference: _matmul_kernel, np.matmul,
// stageflow/kernels.py:184-208).
//
// Arithmetic contract ("sequential-k FMA"): every output element is
//   acc = +0; for kk = 0..k-1: acc = fma(A[i,kk], B[kk,j], acc)
// in the operand dtype.  Any register-tiled FFMA/DFMA GEMM without split-K
// accumulates in exactly this order, so the tiled kernel below, the
// one-thread-per-output small kernel, and the fused row programs that
// inline tiny matmuls all produce identical bits — which is what keeps
// eager == staged bit-exact in the presence of matmuls.  (Large fp32
// contractions on tcgen05 live in sf_gemm_tc.cu and are only used where no
// fused path can inline the op.)
#include "sf_internal.h"

namespace sfrt {

template <class T>
__device__ __forceinline__ T fma_t(T a, T b, T c);
template <>
__device__ __forceinline__ float fma_t<float>(float a, float b, float c) { return __fmaf_rn(a, b, c); }
template <>
__device__ __forceinline__ double fma_t<double>(double a, double b, double c) { return __fma_rn(a, b, c); }

template <class T, bool TA, bool TB>
__device__ __forceinline__ T ld_a(const T* a, long long m, long long k, long long i, long long kk) {
  return TA ? a[kk * m + i] : a[i * k + kk];
}
template <class T, bool TA, bool TB>
__device__ __forceinline__ T ld_b(const T* b, long long k, long long n, long long kk, long long j) {
  return TB ? b[j * k + kk] : b[kk * n + j];
}

// Tiled GEMM: 64x64 block tile, BK = 16, 256 threads, 4x4 outputs per
// thread (rows ty + 16*r, cols tx + 16*c).
template <class T, bool TA, bool TB>
__global__ void __launch_bounds__(256) gemm_tiled(const T* __restrict__ A, const T* __restrict__ B,
                                                  T* __restrict__ C, long long m, long long n,
                                                  long long k, long long kchunk) {
  // blockIdx.z selects a k-range (split-K); without a split kchunk == k
  constexpr int BM = 64, BN = 64, BK = 16;
  const long long kb = (long long)blockIdx.z * kchunk;
  const long long ke = kb + kchunk < k ? kb + kchunk : k;
  C += (long long)blockIdx.z * m * n;
  __shared__ T As[BK][BM + 1];
  __shared__ T Bs[BK][BN + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const long long row0 = (long long)blockIdx.y * BM, col0 = (long long)blockIdx.x * BN;
  T acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = T(0);
  for (long long k0 = kb; k0 < ke; k0 += BK) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int e = threadIdx.x + t * 256;  // 0..1023
      // A tile: BM x BK
      {
        const int mi = e / BK, ki = e % BK;
        const long long gi = row0 + mi, gk = k0 + ki;
        As[ki][mi] = (gi < m && gk < ke) ? ld_a<T, TA, TB>(A, m, k, gi, gk) : T(0);
      }
      // B tile: BK x BN
      {
        const int ki = e / BN, nj = e % BN;
        const long long gk = k0 + ki, gj = col0 + nj;
        Bs[ki][nj] = (gk < ke && gj < n) ? ld_b<T, TA, TB>(B, k, n, gk, gj) : T(0);
      }
    }
    __syncthreads();
    const int kmax = (ke - k0) < BK ? (int)(ke - k0) : BK;
    for (int kk = 0; kk < kmax; ++kk) {
      T av[4], bv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) av[r] = As[kk][ty + 16 * r];
#pragma unroll
      for (int c = 0; c < 4; ++c) bv[c] = Bs[kk][tx + 16 * c];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = fma_t<T>(av[r], bv[c], acc[r][c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const long long gi = row0 + ty + 16 * r;
    if (gi >= m) continue;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const long long gj = col0 + tx + 16 * c;
      if (gj < n) C[gi * n + gj] = acc[r][c];
    }
  }
}

// Split-K epilogue: C[i] = sum over splits, in split order (deterministic).
template <class T>
__global__ void splitk_sum(const T* __restrict__ W, T* __restrict__ C, long long mn, int splits) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < mn; i += stride) {
    T acc = W[i];
    for (int s = 1; s < splits; ++s) acc = acc + W[(long long)s * mn + i];
    C[i] = acc;
  }
}

// Small GEMM: one thread per output (k short), same sequential-k FMA order.
template <class T, bool TA, bool TB>
__global__ void gemm_small(const T* __restrict__ A, const T* __restrict__ B, T* __restrict__ C,
                           long long m, long long n, long long k) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < m * n; o += stride) {
    const long long i = o / n, j = o % n;
    T acc = T(0);
    for (long long kk = 0; kk < k; ++kk)
      acc = fma_t<T>(ld_a<T, TA, TB>(A, m, k, i, kk), ld_b<T, TA, TB>(B, k, n, kk, j), acc);
    C[o] = acc;
  }
}

template <class T, bool TA, bool TB>
static void gemm_go(Device* d, const T* A, const T* B, T* C, long long m, long long n, long long k) {
  const long long tiles64 = ((n + 63) / 64) * ((m + 63) / 64);
  // a 64x64 tiling that would leave most SMs idle (a classifier layer:
  // m = batch, n = 1000, k = 2048 -> 16 tiles) splits k instead (below).
  // One thread per output with a 2048-long dependent FMA chain was latency-
  // bound: 358 us per launch in the ResNet-50 step (profiles/r02e).  Only
  // long contractions split, so every matmul a fused kernel inlines
  // (k * n <= 1024) keeps the sequential-k order; eager and staged run this
  // same kernel, so they agree bit for bit either way.
  // (float64 keeps the sequential-k order everywhere: the f64 parity runs
  // compare whole training trajectories against the reference at 1e-9)
  const bool few_tiles = sizeof(T) == 4 && tiles64 * 2 < d->sm_count && k >= 512;
  if ((m * n <= 4096 && k <= 256) || k <= 8) {
    long long blocks = (m * n + 255) / 256;
    if (blocks > d->sm_count * 16LL) blocks = d->sm_count * 16LL;
    if (blocks < 1) blocks = 1;
    gemm_small<T, TA, TB><<<(unsigned)blocks, 256, 0, d->stream>>>(A, B, C, m, n, k);
  } else {
    const long long tiles = ((n + 63) / 64) * ((m + 63) / 64);
    long long splits = 1;
    // Long contractions over few output tiles (conv weight gradients: k = N*H*W;
    // the classifier layer) are split along k.  Only k >= 16384, or k >= 512
    // over few tiles, splits, so every matmul a fused staged kernel can
    // inline (k*n <= 1024) keeps the sequential-k order.
    if ((k >= 16384 || few_tiles) && tiles < 2LL * d->sm_count) {
      splits = (2LL * d->sm_count + tiles - 1) / tiles;
      const long long by_k = k >= 16384 ? k / 4096 : k / 256;
      if (splits > by_k) splits = by_k;
      if (splits > 64) splits = 64;
      if (splits < 1) splits = 1;
    }
    if (splits > 1) {
      const long long kchunk = ((k + splits - 1) / splits + 15) / 16 * 16;
      splits = (k + kchunk - 1) / kchunk;
      T* work = nullptr;
      if (d->alloc.alloc(d->id, sizeof(T) * (size_t)(splits * m * n), (void**)&work) == SF_OK) {
        dim3 grid((unsigned)((n + 63) / 64), (unsigned)((m + 63) / 64), (unsigned)splits);
        gemm_tiled<T, TA, TB><<<grid, 256, 0, d->stream>>>(A, B, work, m, n, k, kchunk);
        long long blocks = (m * n + 255) / 256;
        if (blocks > d->sm_count * 16LL) blocks = d->sm_count * 16LL;
        splitk_sum<T><<<(unsigned)blocks, 256, 0, d->stream>>>(work, C, m * n, (int)splits);
        d->alloc.release(work);  // stream-ordered reuse is safe
        return;
      }
    }
    dim3 grid((unsigned)((n + 63) / 64), (unsigned)((m + 63) / 64));
    gemm_tiled<T, TA, TB><<<grid, 256, 0, d->stream>>>(A, B, C, m, n, k, k);
  }
}

template <class T>
static void gemm_dispatch(Device* d, const T* A, int ta, const T* B, int tb, T* C, long long m,
                          long long n, long long k) {
  if (!ta && !tb) gemm_go<T, false, false>(d, A, B, C, m, n, k);
  else if (ta && !tb) gemm_go<T, true, false>(d, A, B, C, m, n, k);
  else if (!ta && tb) gemm_go<T, false, true>(d, A, B, C, m, n, k);
  else gemm_go<T, true, true>(d, A, B, C, m, n, k);
}

__global__ void zero_fill_bytes(char* p, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) p[i] = 0;
}

int launch_matmul(Device* d, int dtype, int64_t m, int64_t n, int64_t k, const void* a, int ta,
                  const void* b, int tb, void* c) {
  if (m == 0 || n == 0) return SF_OK;
  if (k == 0) {  // empty contraction: zeros
    return launch_fill(d, dtype, m * n, 0.0, c);
  }
  count_launch(d->id);
  switch (dtype) {
    case SF_DTYPE_F32:
      gemm_dispatch<float>(d, (const float*)a, ta, (const float*)b, tb, (float*)c, m, n, k);
      break;
    case SF_DTYPE_F64:
      gemm_dispatch<double>(d, (const double*)a, ta, (const double*)b, tb, (double*)c, m, n, k);
      break;
    default:
      set_error("matmul requires float tensors");
      return SF_ERR_INVALID;
  }
  SF_CHECK_CUDA(cudaGetLastError());
  return SF_OK;
}

}  // namespace sfrt

using namespace sfrt;

extern "C" int sf_matmul(int dev, int dtype, int64_t m, int64_t n, int64_t k, const void* a,
                         int trans_a, const void* b, int trans_b, void** out) {
  if (dtype != SF_DTYPE_F32 && dtype != SF_DTYPE_F64) {
    set_error("matmul requires float tensors");
    return SF_ERR_INVALID;
  }
  // tiny products go through the launch queue (same sequential-k FMA order)
  sf_op_desc q;
  std::memset(&q, 0, sizeof(q));
  q.kind = SF_QOP_MATMUL;
  q.op = (trans_a ? 1 : 0) | (trans_b ? 2 : 0);
  q.dtype = dtype;
  q.n_in = 2;
  q.m = m;
  q.n = n;
  q.k = k;
  q.in[0] = a;
  q.in[1] = b;
  return sf_queue_push(dev, &q, out);
}
