// sf_reduce.cu — reduce_sum / reduce_mean over arbitrary axes.
//
// Reference: _reduce_kernel (np.sum / np.mean), stageflow/kernels.py:323-364.
// Summation follows the canonical reduction order (CRO) defined in
// sf_ops.cuh, which depends only on the reduced length, so the eager kernel
// and any fused staged kernel that inlines a reduction agree bit-for-bit.
//
// dtype semantics mirrored from NumPy:
//   f32/f64 sum accumulates in the input dtype; mean = sum / count in dtype.
//   i32 sum wraps modulo 2^32 (numpy accumulates in int64, _wrap casts back).
//   i32 mean (eager only; staged inference rejects it, kernels.py:344-352)
//   accumulates in f64, divides, truncates to int32 like the astype in _wrap.
#include <atomic>
#include <type_traits>

#include "sf_internal.h"
#include "sf_ops.cuh"

namespace sfrt {

struct RedArgs {
  long long n_out;     // kept elements
  long long r;         // reduced elements per output
  long long chunk;     // elements per chunk (SF_CRO_CHUNK or r)
  long long n_chunks;  // chunks per output
  int kept_nd, red_nd;
  long long kept_shape[SF_MAX_DIMS], kept_stride[SF_MAX_DIMS];
  long long red_shape[SF_MAX_DIMS], red_stride[SF_MAX_DIMS];
};

template <class T>
struct Acc { typedef T type; };
template <>
struct Acc<int> { typedef unsigned type; };

template <class A>
__device__ __forceinline__ A cadd(A a, A b) { return a + b; }

__device__ __forceinline__ long long kept_offset(const RedArgs& a, long long o) {
  long long off = 0;
#pragma unroll
  for (int d = SF_MAX_DIMS - 1; d >= 0; --d) {
    if (d < a.kept_nd) {
      const long long e = a.kept_shape[d];
      off += (o % e) * a.kept_stride[d];
      o /= e;
    }
  }
  return off;
}

__device__ __forceinline__ long long red_offset(const RedArgs& a, long long j) {
  if (a.red_nd == 1) return j * a.red_stride[0];
  long long off = 0;
#pragma unroll
  for (int d = SF_MAX_DIMS - 1; d >= 0; --d) {
    if (d < a.red_nd) {
      const long long e = a.red_shape[d];
      off += (j % e) * a.red_stride[d];
      j /= e;
    }
  }
  return off;
}

// One warp per (output, chunk).  Lane l folds elements l, l+32, ... of the
// chunk left to right, then the xor butterfly combines the lanes (lanes with
// no element are absent).  Writes the chunk partial (A) to part.
template <class T, class A>
__global__ void reduce_chunks(const RedArgs a, const T* __restrict__ in, A* __restrict__ part) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long w = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5);
       w < a.n_out * a.n_chunks; w += warps) {
    const long long o = w / a.n_chunks, c = w % a.n_chunks;
    const long long base = kept_offset(a, o);
    const long long j0 = c * a.chunk;
    long long len = a.r - j0;
    if (len > a.chunk) len = a.chunk;
    A acc = A();
    bool present = false;
    if (len == 1024) {
      // full chunk: issue all 32 loads before folding (same fold order)
      A v[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) v[q] = (A)in[base + red_offset(a, j0 + lane + 32 * q)];
      acc = v[0];
#pragma unroll
      for (int q = 1; q < 32; ++q) acc = cadd(acc, v[q]);
      present = true;
    } else {
      for (long long j = lane; j < len; j += 32) {
        const A v = (A)in[base + red_offset(a, j0 + j)];
        acc = present ? cadd(acc, v) : v;
        present = true;
      }
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const A ov = __shfl_xor_sync(0xffffffffu, acc, off);
      const bool op = __shfl_xor_sync(0xffffffffu, present, off);
      if (present && op) acc = cadd(acc, ov);
      else if (op) acc = ov;
      present = present || op;
    }
    if (lane == 0) part[w] = acc;
  }
}

// Column reduction (x viewed as (R, C), reduce over R, C contiguous): the same
// CRO per column, but threadIdx.x walks columns so every load is coalesced.
// Block = 32 columns x 32 partial lanes; partial lane l of column c folds rows
// l, l+32, ... of the chunk left to right, then the 32 partials of a column
// are combined with the butterfly tree in shared memory.  Writes one value
// per (column, chunk) to part[c * n_chunks + chunk].
template <class T, class A>
__global__ void __launch_bounds__(1024) reduce_cols(const T* __restrict__ in, long long R,
                                                    long long C, long long chunk,
                                                    long long n_chunks, A* __restrict__ part) {
  __shared__ A acc_s[32][33];
  __shared__ bool pres_s[32][33];
  const int tc = threadIdx.x, tl = threadIdx.y;
  const long long c = (long long)blockIdx.x * 32 + tc;
  const long long j = blockIdx.y;
  const long long g0 = j * chunk;
  long long len = R - g0;
  if (len > chunk) len = chunk;
  A acc = A();
  bool present = false;
  if (c < C) {
    if (len == chunk && chunk == 1024) {
      // full chunk: this lane's 32 elements are all loaded before the fold,
      // so the loads overlap (one DRAM latency instead of 32 in a row);
      // the fold order is unchanged
      const T* p = in + (g0 + tl) * C + c;
      A v[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) v[q] = (A)p[(long long)q * 32 * C];
      acc = v[0];
#pragma unroll
      for (int q = 1; q < 32; ++q) acc = cadd(acc, v[q]);
      present = true;
    } else {
#pragma unroll 8
      for (long long g = tl; g < len; g += 32) {
        const A v = (A)in[(g0 + g) * C + c];
        acc = present ? cadd(acc, v) : v;
        present = true;
      }
    }
  }
  acc_s[tl][tc] = acc;
  pres_s[tl][tc] = present;
  __syncthreads();
  if (tl == 0 && c < C) {
    A a[32];
    bool p[32];
#pragma unroll
    for (int l = 0; l < 32; ++l) {
      a[l] = acc_s[l][tc];
      p[l] = pres_s[l][tc];
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
#pragma unroll
      for (int l = 0; l < off; ++l) {
        if (p[l] && p[l + off]) a[l] = cadd(a[l], a[l + off]);
        else if (p[l + off]) a[l] = a[l + off];
        p[l] = p[l] || p[l + off];
      }
    }
    part[c * n_chunks + j] = a[0];
  }
}

// float32 column reduction with 16-byte loads (C % 4 == 0, 16-byte aligned):
// thread (tx, l) folds partial lane l of 4 adjacent columns — rows l, l+32,
// ... of the chunk, left to right, exactly the fold of reduce_cols — and the
// 32 lane partials of each column are then combined by one warp with the xor
// butterfly (the same tree; lanes past the chunk's end are absent).
// XT column-quads per block; rows are staged in batches of 128 / XT.
static constexpr int kColsStageBytes = 128 * 32 * 16;  // NB * XT * 32 float4 = 64 KB

template <int XT>
__global__ void __launch_bounds__(XT * 32) reduce_cols_f32x4(const float* __restrict__ in,
                                                             long long R, long long C,
                                                             long long chunk, long long n_chunks,
                                                             float* __restrict__ part,
                                                             float* __restrict__ out, int mean,
                                                             float countf,
                                                             unsigned* __restrict__ counters,
                                                             int NB) {
  __shared__ float acc_s[32][XT * 4 + 1];
  // per-thread staging slots [NB][XT * 32] (dynamic, NB * XT * 512 bytes): a
  // batch of NB rows is copied with cp.async, so all NB loads are in flight
  // at once — with register loads ptxas interleaves load and add (the fold
  // order is strict) and keeps only 2-3 loads outstanding, which starves
  // HBM on the small grids of wide-channel layers
  constexpr int NT = XT * 32;
  extern __shared__ float4 stage[];
  const int tx = threadIdx.x, tl = threadIdx.y, tid = tl * XT + tx;
  const long long c0 = ((long long)blockIdx.x * XT + tx) * 4;
  const long long j = blockIdx.y;
  const long long g0 = j * chunk;
  long long len = R - g0;
  if (len > chunk) len = chunk;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c0 < C && tl < len) {
    const float* p = in + (g0 + tl) * C + c0;
    const long long step = 32 * C;
    const int n_rows = (int)((len - tl + 31) / 32);  // rows tl, tl+32, ... < len
    for (int q = 0; q < n_rows; q += NB) {
      const int cnt = n_rows - q < NB ? n_rows - q : NB;
      for (int u = 0; u < cnt; ++u) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&stage[u * NT + tid]);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                     "l"(p + (q + u) * step)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
      // the lane's first element starts the fold (not 0 + x: keeps -0.0)
      int u = 0;
      if (q == 0) {
        acc = stage[tid];
        u = 1;
      }
      for (; u < cnt; ++u) {
        const float4 v = stage[u * NT + tid];
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
    }
  }
  acc_s[tl][tx * 4 + 0] = acc.x;
  acc_s[tl][tx * 4 + 1] = acc.y;
  acc_s[tl][tx * 4 + 2] = acc.z;
  acc_s[tl][tx * 4 + 3] = acc.w;
  __syncthreads();
  // warp w combines the lane partials of columns 4w .. 4w+3 of this block
  const int lin = tl * XT + tx, warp = lin >> 5, lane = lin & 31;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int col = warp * 4 + k;
    const long long c = (long long)blockIdx.x * XT * 4 + col;
    float a = acc_s[lane][col];
    bool present = lane < len;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, a, off);
      const bool op = __shfl_xor_sync(0xffffffffu, present, off);
      if (present && op) a = a + ov;
      else if (op) a = ov;
      present = present || op;
    }
    if (lane == 0 && c < C) {
      if (n_chunks == 1) out[c] = mean ? a / countf : a;
      else part[c * n_chunks + j] = a;
    }
  }
  if (n_chunks == 1) return;
  // Several chunks: the last block to finish a column group folds that
  // group's chunk partials with the CRO (reduce_partials' order) and applies
  // the mean — one launch instead of three.
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (tx == 0 && tl == 0) {
    const unsigned prev = atomicAdd(&counters[blockIdx.x], 1u);
    last = prev == (unsigned)n_chunks - 1;
    if (last) counters[blockIdx.x] = 0;  // at rest again for the next launch
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const long long c = (long long)blockIdx.x * XT * 4 + warp * 4 + k;
    if (c >= C) continue;  // warp-uniform
    const float* pc = part + c * n_chunks;
    float a = 0.f;
    bool present = false;
    for (long long q = lane; q < n_chunks; q += 32) {
      const float v = __ldcg(pc + q);
      a = present ? a + v : v;
      present = true;
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, a, off);
      const bool op = __shfl_xor_sync(0xffffffffu, present, off);
      if (present && op) a = a + ov;
      else if (op) a = ov;
      present = present || op;
    }
    if (lane == 0) out[c] = mean ? a / countf : a;
  }
}

template <int XT>
static void launch_cols_x4(Device* d, const float* in, long long R, long long C, long long chunk,
                           long long n_chunks, float* part, float* out, int mean, float countf) {
  static std::atomic<unsigned long long> attr_set{0};  // one bit per device
  const unsigned long long bit = 1ull << (d->id & 63);
  if (!(attr_set.load() & bit)) {
    cudaFuncSetAttribute(reduce_cols_f32x4<XT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         2 * kColsStageBytes);
    attr_set.fetch_or(bit);
  }
  dim3 grid((unsigned)((C / 4 + XT - 1) / XT), (unsigned)n_chunks);
  // a grid of at most one block per SM (narrow late layers): stage a lane's
  // 32 rows in one batch — one memory round trip instead of two
  int nb = 128 / XT;
  if (XT == 8 && (long long)grid.x * grid.y <= d->sm_count) nb = 32;
  const size_t smem = (size_t)nb * XT * 32 * 16;
  reduce_cols_f32x4<XT><<<grid, dim3(XT, 32), smem, d->stream>>>(
      in, R, C, chunk, n_chunks, part, out, mean, countf, d->red_counters, nb);
}

// One launch: sum (or mean) over the rows of a row-major (R, C) float32
// matrix into out[C].  Requires C % 4 == 0, 16-byte aligned input and at most
// Device::kRedCounters column groups.
static bool cols_x4_ok(Device* d, const float* in, long long R, long long C) {
  return C % 4 == 0 && (uintptr_t)in % 16 == 0 && C / 4 <= Device::kRedCounters && R > 32 &&
         C >= 8 && (R + SF_CRO_CHUNK - 1) / SF_CRO_CHUNK < 65536;
}

static int cols_x4(Device* d, const float* in, long long R, long long C, float* out, int mean,
                   double count) {
  const long long chunk = R > SF_CRO_CHUNK ? SF_CRO_CHUNK : R;
  const long long n_chunks = (R + chunk - 1) / chunk;
  float* part = nullptr;
  if (n_chunks > 1) SF_TRY(d->alloc.alloc(d->id, sizeof(float) * C * n_chunks, (void**)&part));
  const float countf = (float)count;
  // widest block that still gives every SM several blocks; never narrower
  // than 8 column quads, so each row a warp touches is 128 contiguous bytes
  // (narrower blocks split sectors and measured 3-10x slower)
  const long long target = 4LL * d->sm_count;
#define SF_COLS(XT) launch_cols_x4<XT>(d, in, R, C, chunk, n_chunks, part, out, mean, countf)
  if ((C / 128) * n_chunks >= target) SF_COLS(32);
  else if ((C / 64) * n_chunks >= target) SF_COLS(16);
  else SF_COLS(8);
#undef SF_COLS
  count_launch(d->id);
  if (part) d->alloc.release(part);  // stream-ordered reuse is safe
  SF_CHECK_CUDA(cudaGetLastError());
  return SF_OK;
}

// Sequential CRO over <= 32 values per output, one thread per output; used
// for short reductions (r <= 32) and for the second level over chunk
// partials.  Identical tree to the warp butterfly above.
template <class A>
__device__ __forceinline__ A cro_small(A* acc, int p) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
#pragma unroll
    for (int l = 0; l < off; ++l)
      if (l + off < p) acc[l] = cadd(acc[l], acc[l + off]);
  }
  return acc[0];
}

template <class T, class A>
__global__ void reduce_short(const RedArgs a, const T* __restrict__ in, A* __restrict__ out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < a.n_out; o += stride) {
    const long long base = kept_offset(a, o);
    A acc[32];
    const int p = (int)a.r;
#pragma unroll
    for (int l = 0; l < 32; ++l)
      if (l < p) acc[l] = (A)in[base + red_offset(a, l)];
    out[o] = p > 0 ? cro_small(acc, p) : A();
  }
}

// Second level: CRO over the n_chunks partials of each output (any count).
template <class A>
__global__ void reduce_partials(const A* __restrict__ part, long long n_out, long long n_chunks,
                                A* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long o = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); o < n_out;
       o += warps) {
    A acc = A();
    bool present = false;
    for (long long j = lane; j < n_chunks; j += 32) {
      const A v = part[o * n_chunks + j];
      acc = present ? cadd(acc, v) : v;
      present = true;
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      const A ov = __shfl_xor_sync(0xffffffffu, acc, off);
      const bool op = __shfl_xor_sync(0xffffffffu, present, off);
      if (present && op) acc = cadd(acc, ov);
      else if (op) acc = ov;
      present = present || op;
    }
    if (lane == 0) out[o] = acc;
  }
}

// Finalise: out = cast(sum) or cast(sum / count).
template <class A, class T>
__global__ void reduce_finalize(const A* __restrict__ sums, long long n, int mean, double count,
                                T* __restrict__ out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    if (mean) out[i] = (T)(sums[i] / (A)count);
    else out[i] = (T)sums[i];
  }
}
// int32 mean: f64 accumulate, divide, truncate (numpy astype semantics).
__global__ void reduce_finalize_i32_mean(const double* __restrict__ sums, long long n,
                                         double count, int* __restrict__ out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride) {
    double q = sums[i] / count;
    if (q != q) q = 0.0;
    if (q >= 2147483648.0) q = -2147483648.0;  // x86 cvttsd2si overflow result
    if (q < -2147483648.0) q = -2147483648.0;
    out[i] = (int)q;
  }
}

static unsigned grid_cap(Device* d, long long threads) {
  long long b = (threads + 255) / 256;
  const long long cap = (long long)d->sm_count * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

template <class T, class A>
static int run_reduce(Device* d, const RedArgs& a, const T* in, A* sums) {
  const bool columns = a.kept_nd == 1 && a.kept_stride[0] == 1 && a.red_nd == 1 &&
                       a.red_stride[0] == a.kept_shape[0] && a.r > 32 && a.n_out >= 8;
  if (columns) {
    dim3 grid((unsigned)((a.n_out + 31) / 32), (unsigned)a.n_chunks);
    if (a.n_chunks == 1) {
      reduce_cols<T, A><<<grid, dim3(32, 32), 0, d->stream>>>(in, a.r, a.n_out, a.chunk, 1, sums);
      count_launch(d->id);
      return SF_OK;
    }
    A* part = nullptr;
    SF_TRY(d->alloc.alloc(d->id, sizeof(A) * a.n_out * a.n_chunks, (void**)&part));
    reduce_cols<T, A><<<grid, dim3(32, 32), 0, d->stream>>>(in, a.r, a.n_out, a.chunk,
                                                           a.n_chunks, part);
    reduce_partials<A><<<grid_cap(d, a.n_out * 32), 256, 0, d->stream>>>(part, a.n_out,
                                                                        a.n_chunks, sums);
    count_launch(d->id, 2);
    d->alloc.release(part);
    return SF_OK;
  }
  if (a.r <= 32) {
    reduce_short<T, A><<<grid_cap(d, a.n_out), 256, 0, d->stream>>>(a, in, sums);
    count_launch(d->id);
    return SF_OK;
  }
  if (a.n_chunks == 1) {
    reduce_chunks<T, A><<<grid_cap(d, a.n_out * 32), 256, 0, d->stream>>>(a, in, sums);
    count_launch(d->id);
    return SF_OK;
  }
  A* part = nullptr;
  SF_TRY(d->alloc.alloc(d->id, sizeof(A) * a.n_out * a.n_chunks, (void**)&part));
  reduce_chunks<T, A><<<grid_cap(d, a.n_out * a.n_chunks * 32), 256, 0, d->stream>>>(a, in, part);
  reduce_partials<A><<<grid_cap(d, a.n_out * 32), 256, 0, d->stream>>>(part, a.n_out, a.n_chunks, sums);
  count_launch(d->id, 2);
  d->alloc.release(part);  // stream-ordered reuse is safe
  return SF_OK;
}

void reduce_geometry(int ndim, const int64_t* shape, uint32_t axes_mask, RedGeom* g) {
  std::memset(g, 0, sizeof(*g));
  long long stride[SF_MAX_DIMS];
  long long s = 1;
  for (int i = ndim - 1; i >= 0; --i) {
    stride[i] = s;
    s *= shape[i];
  }
  g->n_out = 1;
  g->r = 1;
  for (int i = 0; i < ndim; ++i) {
    if (shape[i] == 1) continue;  // size-1 dims do not affect either side
    if (axes_mask & (1u << i)) {
      // merge with the previous reduced dim if contiguous
      if (g->red_nd > 0 && g->red_stride[g->red_nd - 1] == stride[i] * shape[i]) {
        g->red_shape[g->red_nd - 1] *= shape[i];
        g->red_stride[g->red_nd - 1] = stride[i];
      } else {
        g->red_shape[g->red_nd] = shape[i];
        g->red_stride[g->red_nd] = stride[i];
        ++g->red_nd;
      }
      g->r *= shape[i];
    } else {
      if (g->kept_nd > 0 && g->kept_stride[g->kept_nd - 1] == stride[i] * shape[i]) {
        g->kept_shape[g->kept_nd - 1] *= shape[i];
        g->kept_stride[g->kept_nd - 1] = stride[i];
      } else {
        g->kept_shape[g->kept_nd] = shape[i];
        g->kept_stride[g->kept_nd] = stride[i];
        ++g->kept_nd;
      }
      g->n_out *= shape[i];
    }
  }
}

int launch_reduce(Device* d, int op, int dtype, int ndim, const int64_t* shape,
                  uint32_t axes_mask, const void* in, void* out) {
  RedArgs a;
  std::memset(&a, 0, sizeof(a));
  RedGeom g;
  reduce_geometry(ndim, shape, axes_mask, &g);
  a.n_out = g.n_out;
  a.r = g.r;
  a.kept_nd = g.kept_nd;
  a.red_nd = g.red_nd;
  for (int i = 0; i < SF_MAX_DIMS; ++i) {
    a.kept_shape[i] = g.kept_shape[i];
    a.kept_stride[i] = g.kept_stride[i];
    a.red_shape[i] = g.red_shape[i];
    a.red_stride[i] = g.red_stride[i];
  }
  long long total = 1;
  for (int i = 0; i < ndim; ++i) total *= shape[i];
  if (total == 0) {
    // empty reduction: sum -> 0, mean -> nan (numpy), or empty output
    long long n_out = 1;
    for (int i = 0; i < ndim; ++i)
      if (!(axes_mask & (1u << i))) n_out *= shape[i];
    if (n_out == 0) return SF_OK;
    const double v = op == 1 ? (dtype == SF_DTYPE_I32 ? -2147483648.0 : __builtin_nan("")) : 0.0;
    return launch_fill(d, dtype, n_out, v, out);
  }
  if (a.red_nd == 0) a.red_shape[0] = 1, a.red_stride[0] = 1, a.red_nd = 1;
  a.chunk = a.r > SF_CRO_CHUNK ? SF_CRO_CHUNK : a.r;
  a.n_chunks = (a.r + a.chunk - 1) / a.chunk;
  const double count = (double)a.r;
  const unsigned gf = grid_cap(d, a.n_out);
  switch (dtype) {
    case SF_DTYPE_F32: {
      const bool columns = a.kept_nd == 1 && a.kept_stride[0] == 1 && a.red_nd == 1 &&
                           a.red_stride[0] == a.kept_shape[0];
      if (columns && cols_x4_ok(d, (const float*)in, a.r, a.n_out))
        return cols_x4(d, (const float*)in, a.r, a.n_out, (float*)out, op != 0, count);
      if (op == 0) {
        SF_TRY(run_reduce<float, float>(d, a, (const float*)in, (float*)out));
      } else {
        float* sums = nullptr;
        SF_TRY(d->alloc.alloc(d->id, sizeof(float) * a.n_out, (void**)&sums));
        SF_TRY(run_reduce<float, float>(d, a, (const float*)in, sums));
        reduce_finalize<float, float><<<gf, 256, 0, d->stream>>>(sums, a.n_out, 1, count, (float*)out);
        count_launch(d->id);
        d->alloc.release(sums);
      }
      break;
    }
    case SF_DTYPE_F64: {
      if (op == 0) {
        SF_TRY(run_reduce<double, double>(d, a, (const double*)in, (double*)out));
      } else {
        double* sums = nullptr;
        SF_TRY(d->alloc.alloc(d->id, sizeof(double) * a.n_out, (void**)&sums));
        SF_TRY(run_reduce<double, double>(d, a, (const double*)in, sums));
        reduce_finalize<double, double><<<gf, 256, 0, d->stream>>>(sums, a.n_out, 1, count, (double*)out);
        count_launch(d->id);
        d->alloc.release(sums);
      }
      break;
    }
    case SF_DTYPE_I32: {
      if (op == 0) {
        SF_TRY(run_reduce<int, unsigned>(d, a, (const int*)in, (unsigned*)out));
      } else {
        double* sums = nullptr;
        SF_TRY(d->alloc.alloc(d->id, sizeof(double) * a.n_out, (void**)&sums));
        SF_TRY(run_reduce<int, double>(d, a, (const int*)in, sums));
        reduce_finalize_i32_mean<<<gf, 256, 0, d->stream>>>(sums, a.n_out, count, (int*)out);
        count_launch(d->id);
        d->alloc.release(sums);
      }
      break;
    }
    default:
      set_error("reduce: not defined for this dtype");
      return SF_ERR_INVALID;
  }
  SF_CHECK_CUDA(cudaGetLastError());
  return SF_OK;
}

}  // namespace sfrt

using namespace sfrt;

extern "C" int sf_reduce(int dev, int op, int dtype, int ndim, const int64_t* shape,
                         uint32_t axes_mask, const void* in, void** out) {
  if (ndim < 0 || ndim > SF_MAX_DIMS) {
    set_error("sf_reduce: bad rank");
    return SF_ERR_INVALID;
  }
  // short float reductions (one CRO chunk per output) go through the launch
  // queue, which evaluates the same CRO tree (sf_queue.cu)
  if (dtype == SF_DTYPE_F32 || dtype == SF_DTYPE_F64) {
    sf_op_desc q;
    std::memset(&q, 0, sizeof(q));
    q.kind = SF_QOP_REDUCE;
    q.op = op;
    q.dtype = dtype;
    q.ndim = ndim;
    q.n_in = 1;
    q.m = axes_mask;
    q.in[0] = in;
    for (int i = 0; i < ndim; ++i) q.shape[i] = shape[i];
    return sf_queue_push(dev, &q, out);
  }
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  long long n_out = 1;
  for (int i = 0; i < ndim; ++i)
    if (!(axes_mask & (1u << i))) n_out *= shape[i];
  if (*out == nullptr) SF_TRY(d->alloc.alloc(dev, (size_t)n_out * dtype_size(dtype), out));
  return launch_reduce(d, op, dtype, ndim, shape, axes_mask, in, *out);
}
