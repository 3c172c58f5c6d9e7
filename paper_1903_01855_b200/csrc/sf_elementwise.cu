// sf_elementwise.cu — eager elementwise / broadcast primitives.
//
// One launch per primitive (reference: the numpy ufunc calls in
// stageflow/kernels.py:116-181, :222-232, :263-279).  NumPy broadcasting is
// expressed as per-operand element strides (0 on broadcast dims); the host
// side collapses contiguous dims so the common cases (same-shape operands,
// tensor-with-scalar) take a vectorised 128-bit path with no index math.
// Scalar operands that the front-end knows on the host travel as immediates
// in the launch parameters instead of through an H2D copy.
#include <type_traits>

#include "sf_internal.h"
#include "sf_ops.cuh"

namespace sfrt {

struct EwArgs {
  int op;
  int n_in;
  int ndim;
  int pad;
  long long n;
  const void* in[3];
  double imm[3];
  long long shape[SF_MAX_DIMS];
  long long strides[3][SF_MAX_DIMS];
};

template <class T>
__device__ __forceinline__ T fetch(const EwArgs& a, int j, long long off) {
  const T* p = (const T*)a.in[j];
  return p ? p[off] : (T)a.imm[j];
}

template <class T, class O>
__device__ __forceinline__ O apply(int op, T x, T y) {
  if (SF_OP_IS_BINARY(op)) {
    if (op == SF_OP_GREATER || op == SF_OP_LESS || op == SF_OP_EQUAL ||
        op == SF_OP_GREATER_EQUAL)
      return (O)sf::compare_f<T>(op, x, y);
    return (O)sf::binary_f<T>(op, x, y);
  }
  if (op == SF_OP_ISFINITE) return (O)sf::isfinite_(x);
  return (O)sf::unary_f<T>(op, x);
}

// Generic strided path (any broadcast pattern, ndim <= 8).
template <class T, class O>
__global__ void ew_strided(const EwArgs a, O* __restrict__ out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.n; i += stride) {
    long long rem = i, o0 = 0, o1 = 0;
#pragma unroll
    for (int d = SF_MAX_DIMS - 1; d >= 0; --d) {
      if (d < a.ndim) {
        const long long ext = a.shape[d];
        const long long idx = rem % ext;
        rem /= ext;
        o0 += idx * a.strides[0][d];
        o1 += idx * a.strides[1][d];
      }
    }
    const T x = fetch<T>(a, 0, o0);
    const T y = a.n_in > 1 ? fetch<T>(a, 1, o1) : x;
    out[i] = apply<T, O>(a.op, x, y);
  }
}

// Two collapsed dims, < 2^31 elements (row/column broadcasts, e.g. NHWC
// activations against per-channel vectors): 32-bit index math only.
template <class T, class O>
__global__ void ew_2d(const EwArgs a, O* __restrict__ out) {
  const unsigned n = (unsigned)a.n, cols = (unsigned)a.shape[1];
  const unsigned stride = gridDim.x * blockDim.x;
  const unsigned s00 = (unsigned)a.strides[0][0], s01 = (unsigned)a.strides[0][1];
  const unsigned s10 = (unsigned)a.strides[1][0], s11 = (unsigned)a.strides[1][1];
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const unsigned r = i / cols, c = i - r * cols;
    const T x = fetch<T>(a, 0, (long long)(r * s00 + c * s01));
    const T y = a.n_in > 1 ? fetch<T>(a, 1, (long long)(r * s10 + c * s11)) : x;
    out[i] = apply<T, O>(a.op, x, y);
  }
}

// Two collapsed dims, float32, cols % 4 == 0: each thread produces 4
// consecutive elements of one row.  An operand is a row-contiguous matrix
// (inner stride 1: one 16-byte load), a per-row value (inner stride 0: one
// scalar load shared by the 4 lanes), or an immediate.  The per-channel
// vectors of NHWC activations stay in L1/L2, so HBM sees one read per
// activation operand and one write.
__device__ __forceinline__ float4 fetch4(const EwArgs& a, int j, unsigned r, unsigned c) {
  const float* p = (const float*)a.in[j];
  if (!p) {
    const float v = (float)a.imm[j];
    return make_float4(v, v, v, v);
  }
  const unsigned s0 = (unsigned)a.strides[j][0];
  if (a.strides[j][1] == 0) {
    const float v = p[r * s0];
    return make_float4(v, v, v, v);
  }
  return *reinterpret_cast<const float4*>(p + r * s0 + c);
}

__device__ __forceinline__ float4 apply4(int op, float4 x, float4 y) {
  float4 o;
  o.x = apply<float, float>(op, x.x, y.x);
  o.y = apply<float, float>(op, x.y, y.y);
  o.z = apply<float, float>(op, x.z, y.z);
  o.w = apply<float, float>(op, x.w, y.w);
  return o;
}

// two independent vectors per thread and iteration (both loads in flight
// before either result is needed)
__global__ void __launch_bounds__(256) ew_2d_f32x4(const EwArgs a, float* __restrict__ out) {
  const unsigned n4 = (unsigned)(a.n >> 2), cols = (unsigned)a.shape[1];
  const unsigned stride = gridDim.x * blockDim.x;
  const bool two = a.n_in > 1;
  unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + stride < n4; i += 2 * stride) {
    const unsigned e0 = i << 2, r0 = e0 / cols, c0 = e0 - r0 * cols;
    const unsigned e1 = (i + stride) << 2, r1 = e1 / cols, c1 = e1 - r1 * cols;
    const float4 x0 = fetch4(a, 0, r0, c0), x1 = fetch4(a, 0, r1, c1);
    const float4 y0 = two ? fetch4(a, 1, r0, c0) : x0, y1 = two ? fetch4(a, 1, r1, c1) : x1;
    reinterpret_cast<float4*>(out)[i] = apply4(a.op, x0, y0);
    reinterpret_cast<float4*>(out)[i + stride] = apply4(a.op, x1, y1);
  }
  for (; i < n4; i += stride) {
    const unsigned e = i << 2, r = e / cols, c = e - r * cols;
    const float4 x = fetch4(a, 0, r, c);
    const float4 y = two ? fetch4(a, 1, r, c) : x;
    reinterpret_cast<float4*>(out)[i] = apply4(a.op, x, y);
  }
}

static bool ew_2d_x4_ok(const EwArgs& a, const void* out) {
  if (a.ndim != 2 || a.shape[1] % 4 != 0 || a.n >= (1LL << 32) || (uintptr_t)out % 16) return false;
  for (int j = 0; j < a.n_in; ++j) {
    if (!a.in[j]) continue;
    if (a.strides[j][1] == 1) {
      if (a.strides[j][0] % 4 || (uintptr_t)a.in[j] % 16) return false;
    } else if (a.strides[j][1] != 0) {
      return false;
    }
    if (a.shape[0] * (a.strides[j][0] + 1) >= (1LL << 32)) return false;
  }
  return true;
}

// Flat path: every operand is either full-size contiguous or a scalar.
template <class T, class O>
__global__ void ew_flat(const EwArgs a, O* __restrict__ out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const T* p0 = (const T*)a.in[0];
  const T* p1 = (const T*)a.in[1];
  const bool s0 = a.strides[0][0] == 0, s1 = a.strides[1][0] == 0;
  const T c0 = p0 ? (s0 ? p0[0] : T()) : (T)a.imm[0];
  const T c1 = a.n_in > 1 ? (p1 ? (s1 ? p1[0] : T()) : (T)a.imm[1]) : T();
  const bool v0 = p0 && !s0, v1 = a.n_in > 1 && p1 && !s1;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.n; i += stride) {
    const T x = v0 ? p0[i] : c0;
    const T y = a.n_in > 1 ? (v1 ? p1[i] : c1) : x;
    out[i] = apply<T, O>(a.op, x, y);
  }
}

// Flat float32 path with 128-bit accesses (n % 4 tail handled by thread 0..3).
template <int OP_KIND>
__global__ void ew_flat_f32x4(const EwArgs a, float* __restrict__ out) {
  const long long n4 = a.n >> 2;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const float* p0 = (const float*)a.in[0];
  const float* p1 = (const float*)a.in[1];
  const bool s0 = a.strides[0][0] == 0, s1 = a.strides[1][0] == 0;
  const float c0 = p0 ? (s0 ? p0[0] : 0.f) : (float)a.imm[0];
  const float c1 = a.n_in > 1 ? (p1 ? (s1 ? p1[0] : 0.f) : (float)a.imm[1]) : 0.f;
  const bool v0 = p0 && !s0, v1 = a.n_in > 1 && p1 && !s1;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 x = v0 ? reinterpret_cast<const float4*>(p0)[i] : make_float4(c0, c0, c0, c0);
    float4 y = v1 ? reinterpret_cast<const float4*>(p1)[i] : make_float4(c1, c1, c1, c1);
    if (a.n_in == 1) y = x;
    float4 r;
    r.x = apply<float, float>(a.op, x.x, y.x);
    r.y = apply<float, float>(a.op, x.y, y.y);
    r.z = apply<float, float>(a.op, x.z, y.z);
    r.w = apply<float, float>(a.op, x.w, y.w);
    reinterpret_cast<float4*>(out)[i] = r;
  }
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long j = (n4 << 2) + t;
  if (t < 4 && j < a.n) {
    const float x = v0 ? p0[j] : c0;
    const float y = a.n_in > 1 ? (v1 ? p1[j] : c1) : x;
    out[j] = apply<float, float>(a.op, x, y);
  }
}

// select(cond, a, b): cond is boolean, a/b of T (any broadcast pattern).
template <class T>
__global__ void ew_select(const EwArgs a, T* __restrict__ out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.n; i += stride) {
    long long rem = i, o[3] = {0, 0, 0};
#pragma unroll
    for (int d = SF_MAX_DIMS - 1; d >= 0; --d) {
      if (d < a.ndim) {
        const long long ext = a.shape[d];
        const long long idx = rem % ext;
        rem /= ext;
        o[0] += idx * a.strides[0][d];
        o[1] += idx * a.strides[1][d];
        o[2] += idx * a.strides[2][d];
      }
    }
    const bool* c = (const bool*)a.in[0];
    const bool cv = c ? c[o[0]] : (a.imm[0] != 0.0);
    out[i] = cv ? fetch<T>(a, 1, o[1]) : fetch<T>(a, 2, o[2]);
  }
}

static bool op_outputs_bool(int op) {
  return op == SF_OP_GREATER || op == SF_OP_LESS || op == SF_OP_EQUAL ||
         op == SF_OP_GREATER_EQUAL || op == SF_OP_ISFINITE || op == SF_OP_LOGICAL_NOT;
}

__global__ void ew_logical_not(const bool* __restrict__ in, bool* __restrict__ out, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = !in[i];
}

// Collapse size-1 dims and merge dims that are contiguous for every operand.
static void collapse(EwArgs& a) {
  int nd = 0;
  long long shape[SF_MAX_DIMS];
  long long st[3][SF_MAX_DIMS];
  for (int d = 0; d < a.ndim; ++d) {
    if (a.shape[d] == 1) continue;
    shape[nd] = a.shape[d];
    for (int j = 0; j < 3; ++j) st[j][nd] = a.strides[j][d];
    ++nd;
  }
  // merge from the innermost outward
  int out_nd = 0;
  long long s2[SF_MAX_DIMS];
  long long t2[3][SF_MAX_DIMS];
  for (int d = 0; d < nd; ++d) {
    if (out_nd > 0) {
      const int p = out_nd - 1;
      bool mergeable = true;
      for (int j = 0; j < a.n_in; ++j)
        if (t2[j][p] != st[j][d] * shape[d]) mergeable = false;
      if (mergeable) {
        s2[p] *= shape[d];
        for (int j = 0; j < 3; ++j) t2[j][p] = st[j][d];
        continue;
      }
    }
    s2[out_nd] = shape[d];
    for (int j = 0; j < 3; ++j) t2[j][out_nd] = st[j][d];
    ++out_nd;
  }
  a.ndim = out_nd;
  for (int d = 0; d < SF_MAX_DIMS; ++d) {
    a.shape[d] = d < out_nd ? s2[d] : 1;
    for (int j = 0; j < 3; ++j) a.strides[j][d] = d < out_nd ? t2[j][d] : 0;
  }
}

static unsigned grid_for(Device* d, long long work) {
  long long blocks = (work + 255) / 256;
  const long long cap = (long long)d->sm_count * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (unsigned)blocks;
}

template <class T, class O>
static void dispatch_ew(Device* d, const EwArgs& a, void* out, bool flat) {
  if (flat) {
    ew_flat<T, O><<<grid_for(d, a.n), 256, 0, d->stream>>>(a, (O*)out);
  } else if (std::is_same<T, float>::value && std::is_same<O, float>::value &&
             ew_2d_x4_ok(a, out)) {
    ew_2d_f32x4<<<grid_for(d, a.n / 4), 256, 0, d->stream>>>(a, (float*)out);
  } else if (a.ndim == 2 && a.n < (1LL << 31) &&
             a.shape[0] * (a.strides[0][0] + a.strides[1][0] + 1) < (1LL << 31)) {
    ew_2d<T, O><<<grid_for(d, a.n), 256, 0, d->stream>>>(a, (O*)out);
  } else {
    ew_strided<T, O><<<grid_for(d, a.n), 256, 0, d->stream>>>(a, (O*)out);
  }
}

int launch_elementwise(Device* d, int op, int dtype, int ndim, const int64_t* shape, void* out,
                       const void* const* ins, const int64_t* const* strides,
                       const double* imms, int n_in) {
  EwArgs a;
  std::memset(&a, 0, sizeof(a));
  a.op = op;
  a.n_in = n_in;
  a.ndim = ndim;
  long long n = 1;
  for (int i = 0; i < ndim; ++i) {
    a.shape[i] = shape[i];
    n *= shape[i];
  }
  a.n = n;
  if (n == 0) return SF_OK;
  for (int j = 0; j < n_in; ++j) {
    a.in[j] = ins[j];
    a.imm[j] = imms ? imms[j] : 0.0;
    for (int i = 0; i < ndim; ++i) a.strides[j][i] = ins[j] ? strides[j][i] : 0;
  }
  collapse(a);
  bool flat = a.ndim <= 1;
  if (flat && a.ndim == 1) {
    for (int j = 0; j < n_in; ++j)
      if (a.strides[j][0] != 0 && a.strides[j][0] != 1) flat = false;
  }
  if (a.ndim == 0) {
    for (int j = 0; j < 3; ++j) a.strides[j][0] = 0;
  }
  count_launch(d->id);
  if (op == SF_OP_SELECT) {
    switch (dtype) {
      case SF_DTYPE_F32: ew_select<float><<<grid_for(d, n), 256, 0, d->stream>>>(a, (float*)out); break;
      case SF_DTYPE_F64: ew_select<double><<<grid_for(d, n), 256, 0, d->stream>>>(a, (double*)out); break;
      case SF_DTYPE_I32: ew_select<int><<<grid_for(d, n), 256, 0, d->stream>>>(a, (int*)out); break;
      case SF_DTYPE_BOOL: ew_select<bool><<<grid_for(d, n), 256, 0, d->stream>>>(a, (bool*)out); break;
      default: set_error("select: bad dtype"); return SF_ERR_INVALID;
    }
    SF_CHECK_CUDA(cudaGetLastError());
    return SF_OK;
  }
  if (op == SF_OP_LOGICAL_NOT) {
    if (dtype != SF_DTYPE_BOOL || !flat || !a.in[0]) {
      set_error("logical_not: expects one contiguous boolean tensor");
      return SF_ERR_INVALID;
    }
    ew_logical_not<<<grid_for(d, n), 256, 0, d->stream>>>((const bool*)a.in[0], (bool*)out, n);
    SF_CHECK_CUDA(cudaGetLastError());
    return SF_OK;
  }
  const bool to_bool = op_outputs_bool(op);
  switch (dtype) {
    case SF_DTYPE_F32:
      if (to_bool) {
        dispatch_ew<float, bool>(d, a, out, flat);
      } else if (flat && n >= 1024) {
        ew_flat_f32x4<0><<<grid_for(d, (n + 3) / 4), 256, 0, d->stream>>>(a, (float*)out);
      } else {
        dispatch_ew<float, float>(d, a, out, flat);
      }
      break;
    case SF_DTYPE_F64:
      if (to_bool) dispatch_ew<double, bool>(d, a, out, flat);
      else dispatch_ew<double, double>(d, a, out, flat);
      break;
    case SF_DTYPE_I32:
      if (to_bool) dispatch_ew<int, bool>(d, a, out, flat);
      else dispatch_ew<int, int>(d, a, out, flat);
      break;
    case SF_DTYPE_BOOL:
      if (op == SF_OP_IDENTITY) {
        dispatch_ew<bool, bool>(d, a, out, flat);
        break;
      }
      if (op == SF_OP_EQUAL) {
        dispatch_ew<bool, bool>(d, a, out, flat);
        break;
      }
      set_error("elementwise op not defined for boolean tensors");
      return SF_ERR_INVALID;
    default:
      set_error("elementwise: bad dtype");
      return SF_ERR_INVALID;
  }
  SF_CHECK_CUDA(cudaGetLastError());
  return SF_OK;
}

// ------------------------------------------------------------- cast
template <class S, class D>
__global__ void cast_kernel(const S* __restrict__ in, D* __restrict__ out, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = (D)in[i];
}

template <class S>
static int cast_from(Device* d, int dst, long long n, const S* in, void* out) {
  const unsigned g = grid_for(d, n);
  switch (dst) {
    case SF_DTYPE_F32: cast_kernel<S, float><<<g, 256, 0, d->stream>>>(in, (float*)out, n); break;
    case SF_DTYPE_F64: cast_kernel<S, double><<<g, 256, 0, d->stream>>>(in, (double*)out, n); break;
    case SF_DTYPE_I32: cast_kernel<S, int><<<g, 256, 0, d->stream>>>(in, (int*)out, n); break;
    case SF_DTYPE_BOOL: cast_kernel<S, bool><<<g, 256, 0, d->stream>>>(in, (bool*)out, n); break;
    default: set_error("cast: bad dtype"); return SF_ERR_INVALID;
  }
  return SF_OK;
}

int launch_cast(Device* d, int src, int dst, int64_t n, const void* in, void* out) {
  if (n == 0) return SF_OK;
  count_launch(d->id);
  int st;
  switch (src) {
    case SF_DTYPE_F32: st = cast_from<float>(d, dst, n, (const float*)in, out); break;
    case SF_DTYPE_F64: st = cast_from<double>(d, dst, n, (const double*)in, out); break;
    case SF_DTYPE_I32: st = cast_from<int>(d, dst, n, (const int*)in, out); break;
    case SF_DTYPE_BOOL: st = cast_from<bool>(d, dst, n, (const bool*)in, out); break;
    default: set_error("cast: bad dtype"); return SF_ERR_INVALID;
  }
  if (st != SF_OK) return st;
  SF_CHECK_CUDA(cudaGetLastError());
  return SF_OK;
}

}  // namespace sfrt

using namespace sfrt;

static int out_dtype_for(int op, int dtype) {
  if (op == SF_OP_GREATER || op == SF_OP_LESS || op == SF_OP_EQUAL ||
      op == SF_OP_GREATER_EQUAL || op == SF_OP_ISFINITE || op == SF_OP_LOGICAL_NOT)
    return SF_DTYPE_BOOL;
  return dtype;
}

extern "C" int sf_elementwise(int dev, const sf_ew_desc* desc, void** out) {
  // small primitives go through the launch queue (sf_queue.cu); the rest
  // launch directly after the queue is flushed
  if (desc->ndim < 0 || desc->ndim > SF_MAX_DIMS || desc->n_in < 1 || desc->n_in > 3) {
    set_error("sf_elementwise: bad descriptor");
    return SF_ERR_INVALID;
  }
  sf_op_desc q;
  std::memset(&q, 0, sizeof(q));
  q.kind = SF_QOP_EW;
  q.op = desc->op;
  q.dtype = desc->dtype;
  q.ndim = desc->ndim;
  q.n_in = desc->n_in;
  for (int j = 0; j < 3; ++j) {
    q.in[j] = desc->in[j];
    q.imm[j] = desc->imm[j];
  }
  std::memcpy(q.shape, desc->shape, sizeof(q.shape));
  std::memcpy(q.strides, desc->strides, sizeof(q.strides));
  return sf_queue_push(dev, &q, out);
}

extern "C" int sf_cast(int dev, int src_dtype, int dst_dtype, int64_t n, const void* in, void** out) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  if (*out == nullptr) SF_TRY(d->alloc.alloc(dev, (size_t)n * dtype_size(dst_dtype), out));
  return launch_cast(d, src_dtype, dst_dtype, n, in, *out);
}
