// sf_queue.cu — the eager launch queue (north_star subsystem 1).
//
// Eager dispatch of a small primitive (reference: _dispatch_eager ->
// kernel -> one np.* call, stageflow/ops.py:318-347) costs the reference
// ~13 us of Python per op; a GPU build that launched one kernel per op
// would still pay one cudaLaunchKernel (~2 us of host time) plus a kernel
// boundary per op.  Small primitives therefore go into a per-device queue
// of compact op descriptors instead.  The queue is flushed as ONE launch of
// an interpreter kernel: a single CTA that executes the queued ops in push
// order with a __syncthreads() between consecutive ops (so op j may read
// what op i < j wrote), every op computed with the same per-element
// functions (sf_ops.cuh) and the same sequential-k FMA matmul contract as
// the one-op kernels — queued and direct results are bit-identical.
//
// Ordering: the queue is flushed before any other work is enqueued on the
// device's stream (ensure_device flushes; every C-ABI entry point that
// enqueues work goes through it), before a graph capture begins, and when it
// is full, so stream order is exactly push order.  Blocks freed by the host
// while a queued op still reads them are only reused by later allocations,
// whose writers are ordered after the queue; the allocator flushes before it
// returns memory to the driver.
#include "sf_internal.h"
#include "sf_ops.cuh"

namespace sfrt {

struct QOp {
  int kind;  // SF_QOP_EW / SF_QOP_MATMUL
  int op;    // EW: SF_OP_*; MATMUL: bit0 trans_a, bit1 trans_b
  int dtype;
  int ndim;  // EW: collapsed rank <= 4
  int n;     // EW: element count; MATMUL: m * n
  int n_in;
  int mm, mk;  // MATMUL: m, k (n = this->n / mm)
  int shape[kQueueDims];
  int st[3][kQueueDims];
  const void* in[3];
  void* out;
  double imm[3];
};

static_assert(sizeof(QOp) == sizeof(QOpSlot), "QOpSlot must hold one QOp");

template <int CAP>
struct QBatch {
  int count;
  int pad[3];
  QOp ops[CAP];
};

template <class T, class O>
__device__ __forceinline__ O q_apply(int op, T x, T y) {
  if (SF_OP_IS_BINARY(op)) {
    if (op == SF_OP_GREATER || op == SF_OP_LESS || op == SF_OP_EQUAL ||
        op == SF_OP_GREATER_EQUAL)
      return (O)sf::compare_f<T>(op, x, y);
    return (O)sf::binary_f<T>(op, x, y);
  }
  if (op == SF_OP_ISFINITE) return (O)sf::isfinite_(x);
  return (O)sf::unary_f<T>(op, x);
}

template <class T, class O>
__device__ void q_ew(const QOp& o) {
  const T* p0 = (const T*)o.in[0];
  const T* p1 = (const T*)o.in[1];
  const T c0 = (T)o.imm[0], c1 = (T)o.imm[1];
  O* out = (O*)o.out;
  for (int i = threadIdx.x; i < o.n; i += blockDim.x) {
    int rem = i, f0 = 0, f1 = 0;
#pragma unroll
    for (int d = kQueueDims - 1; d >= 0; --d) {
      if (d < o.ndim) {
        const int ext = o.shape[d];
        const int idx = rem % ext;
        rem /= ext;
        f0 += idx * o.st[0][d];
        f1 += idx * o.st[1][d];
      }
    }
    const T x = p0 ? p0[f0] : c0;
    const T y = o.n_in > 1 ? (p1 ? p1[f1] : c1) : x;
    out[i] = q_apply<T, O>(o.op, x, y);
  }
}

template <class T>
__device__ __forceinline__ T q_fma(T a, T b, T c);
template <>
__device__ __forceinline__ float q_fma<float>(float a, float b, float c) { return __fmaf_rn(a, b, c); }
template <>
__device__ __forceinline__ double q_fma<double>(double a, double b, double c) { return __fma_rn(a, b, c); }

// one thread per output, sequential-k FMA (the contract of sf_matmul.cu)
template <class T>
__device__ void q_mm(const QOp& o) {
  const T* A = (const T*)o.in[0];
  const T* B = (const T*)o.in[1];
  T* C = (T*)o.out;
  const int m = o.mm, k = o.mk, n = o.n / o.mm;
  const bool ta = o.op & 1, tb = o.op & 2;
  for (int idx = threadIdx.x; idx < o.n; idx += blockDim.x) {
    const int i = idx / n, j = idx - (idx / n) * n;
    T acc = T(0);
    for (int kk = 0; kk < k; ++kk) {
      const T a = ta ? A[kk * m + i] : A[i * k + kk];
      const T b = tb ? B[j * k + kk] : B[kk * n + j];
      acc = q_fma<T>(a, b, acc);
    }
    C[idx] = acc;
  }
}

// reduce_sum / reduce_mean with r <= SF_CRO_CHUNK per output: the
// canonical reduction order of sf_reduce.cu — lane l folds elements l,
// l+32, ... left to right, then the xor butterfly combines the lanes present
// — one warp per output; mean divides in the dtype (reduce_finalize).
// shape/st[0]: kept dims; st[1]/st[2]: reduced extents/strides.
template <class T>
__device__ void q_reduce(const QOp& o) {
  const T* in = (const T*)o.in[0];
  T* out = (T*)o.out;
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  const int r = o.mm;
  for (int w = threadIdx.x >> 5; w < o.n; w += warps) {
    int rem = w, base = 0;
#pragma unroll
    for (int d = kQueueDims - 1; d >= 0; --d) {
      if (d < o.ndim) {
        const int e = o.shape[d];
        base += (rem % e) * o.st[0][d];
        rem /= e;
      }
    }
    T acc = T(0);
    bool present = false;
    for (int j = lane; j < r; j += 32) {
      int jr = j, off = 0;
#pragma unroll
      for (int d = kQueueDims - 1; d >= 0; --d) {
        if (d < o.n_in) {
          const int e = o.st[1][d];
          off += (jr % e) * o.st[2][d];
          jr /= e;
        }
      }
      const T v = in[base + off];
      acc = present ? acc + v : v;
      present = true;
    }
#pragma unroll
    for (int sh = 16; sh >= 1; sh >>= 1) {
      const T ov = __shfl_xor_sync(0xffffffffu, acc, sh);
      const bool op = __shfl_xor_sync(0xffffffffu, present, sh);
      if (present && op) acc = acc + ov;
      else if (op) acc = ov;
      present = present || op;
    }
    if (lane == 0) out[w] = o.op ? acc / (T)r : acc;
  }
}

__device__ __forceinline__ bool q_to_bool(int op) {
  return op == SF_OP_GREATER || op == SF_OP_LESS || op == SF_OP_EQUAL ||
         op == SF_OP_GREATER_EQUAL || op == SF_OP_ISFINITE;
}

__device__ void q_run(const QOp& o) {
  if (o.kind == SF_QOP_MATMUL) {
    if (o.dtype == SF_DTYPE_F64) q_mm<double>(o);
    else q_mm<float>(o);
    return;
  }
  if (o.kind == SF_QOP_REDUCE) {
    if (o.dtype == SF_DTYPE_F64) q_reduce<double>(o);
    else q_reduce<float>(o);
    return;
  }
  const bool tb = q_to_bool(o.op);
  switch (o.dtype) {
    case SF_DTYPE_F32:
      if (tb) q_ew<float, bool>(o); else q_ew<float, float>(o);
      break;
    case SF_DTYPE_F64:
      if (tb) q_ew<double, bool>(o); else q_ew<double, double>(o);
      break;
    case SF_DTYPE_I32:
      if (tb) q_ew<int, bool>(o); else q_ew<int, int>(o);
      break;
    default:  // bool identity / equal
      q_ew<bool, bool>(o);
      break;
  }
}

template <int CAP>
__global__ void __launch_bounds__(kQueueThreads) queue_kernel(const __grid_constant__ QBatch<CAP> b) {
  for (int q = 0; q < b.count; ++q) {
    if (q) __syncthreads();
    q_run(b.ops[q]);
  }
}

// ------------------------------------------------------------- host side

static int flush_locked(Device* d) {
  const int n = (int)d->q_ops.size();
  if (n == 0) return SF_OK;
  count_launch(d->id);
  d->q_flushes++;
  // the smallest batch type that holds the queue (kernel parameter space
  // grows with it; a 64-op batch is ~9.5 KB of parameters)
  if (n <= 4) {
    QBatch<4> b;
    b.count = n;
    std::memcpy(b.ops, d->q_ops.data(), sizeof(QOp) * n);
    queue_kernel<4><<<1, kQueueThreads, 0, d->stream>>>(b);
  } else if (n <= 16) {
    QBatch<16> b;
    b.count = n;
    std::memcpy(b.ops, d->q_ops.data(), sizeof(QOp) * n);
    queue_kernel<16><<<1, kQueueThreads, 0, d->stream>>>(b);
  } else {
    QBatch<kQueueMaxOps> b;
    b.count = n;
    std::memcpy(b.ops, d->q_ops.data(), sizeof(QOp) * n);
    queue_kernel<kQueueMaxOps><<<1, kQueueThreads, 0, d->stream>>>(b);
  }
  d->q_ops.clear();
  d->q_pending.store(0, std::memory_order_release);
  SF_CHECK_CUDA(cudaGetLastError());
  return SF_OK;
}

int queue_flush(Device* d) {
  if (d->q_pending.load(std::memory_order_acquire) == 0) return SF_OK;
  std::lock_guard<std::mutex> lk(d->q_mu);
  return flush_locked(d);
}

int queue_flush_dev(int dev) {
  Device* d = device(dev);
  return d ? queue_flush(d) : SF_OK;
}

// Collapse an elementwise descriptor the way launch_elementwise does (drop
// size-1 dims, merge dims contiguous for every operand) into a QOp; false
// if it does not fit the queue's compact form.
static bool compact_ew(const Device* d, const sf_op_desc& s, QOp* o) {
  if (s.n_in < 1 || s.n_in > 2 || s.ndim < 0 || s.ndim > SF_MAX_DIMS) return false;
  if (s.op == SF_OP_SELECT || s.op == SF_OP_LOGICAL_NOT) return false;
  long long n = 1;
  for (int i = 0; i < s.ndim; ++i) n *= s.shape[i];
  if (n <= 0 || n > d->q_max_numel) return false;
  long long shape[SF_MAX_DIMS], st[2][SF_MAX_DIMS];
  int nd = 0;
  for (int i = 0; i < s.ndim; ++i) {
    if (s.shape[i] == 1) continue;
    shape[nd] = s.shape[i];
    for (int j = 0; j < 2; ++j) st[j][nd] = (j < s.n_in && s.in[j]) ? s.strides[j][i] : 0;
    ++nd;
  }
  int out_nd = 0;
  long long s2[SF_MAX_DIMS], t2[2][SF_MAX_DIMS];
  for (int i = 0; i < nd; ++i) {
    if (out_nd > 0) {
      const int p = out_nd - 1;
      bool ok = true;
      for (int j = 0; j < s.n_in; ++j)
        if (t2[j][p] != st[j][i] * shape[i]) ok = false;
      if (ok) {
        s2[p] *= shape[i];
        for (int j = 0; j < 2; ++j) t2[j][p] = st[j][i];
        continue;
      }
    }
    s2[out_nd] = shape[i];
    for (int j = 0; j < 2; ++j) t2[j][out_nd] = st[j][i];
    ++out_nd;
  }
  if (out_nd > kQueueDims) return false;
  std::memset(o, 0, sizeof(QOp));
  o->kind = SF_QOP_EW;
  o->op = s.op;
  o->dtype = s.dtype;
  o->ndim = out_nd;
  o->n = (int)n;
  o->n_in = s.n_in;
  for (int i = 0; i < out_nd; ++i) {
    o->shape[i] = (int)s2[i];
    for (int j = 0; j < 2; ++j) {
      if (t2[j][i] < 0 || t2[j][i] > (1LL << 30)) return false;
      o->st[j][i] = (int)t2[j][i];
    }
  }
  for (int j = 0; j < s.n_in; ++j) {
    o->in[j] = s.in[j];
    o->imm[j] = s.imm[j];
  }
  return true;
}

static bool out_is_bool(int op) {
  return op == SF_OP_GREATER || op == SF_OP_LESS || op == SF_OP_EQUAL ||
         op == SF_OP_GREATER_EQUAL || op == SF_OP_ISFINITE || op == SF_OP_LOGICAL_NOT;
}

static bool compact_reduce(const Device* d, const sf_op_desc& s, QOp* o) {
  if ((s.dtype != SF_DTYPE_F32 && s.dtype != SF_DTYPE_F64) || s.ndim < 0 || s.ndim > SF_MAX_DIMS)
    return false;
  long long total = 1;
  for (int i = 0; i < s.ndim; ++i) total *= s.shape[i];
  if (total <= 0 || total > d->q_max_numel) return false;
  RedGeom g;
  reduce_geometry(s.ndim, s.shape, (uint32_t)s.m, &g);
  if (g.r > SF_CRO_CHUNK || g.kept_nd > kQueueDims || g.red_nd > kQueueDims) return false;
  std::memset(o, 0, sizeof(QOp));
  o->kind = SF_QOP_REDUCE;
  o->op = s.op ? 1 : 0;
  o->dtype = s.dtype;
  o->ndim = g.kept_nd;
  o->n_in = g.red_nd;
  o->n = (int)g.n_out;
  o->mm = (int)g.r;
  for (int i = 0; i < g.kept_nd; ++i) {
    o->shape[i] = (int)g.kept_shape[i];
    o->st[0][i] = (int)g.kept_stride[i];
  }
  for (int i = 0; i < g.red_nd; ++i) {
    o->st[1][i] = (int)g.red_shape[i];
    o->st[2][i] = (int)g.red_stride[i];
  }
  o->in[0] = s.in[0];
  return true;
}

static int direct_launch(Device* d, const sf_op_desc& s, void* out) {
  if (s.kind == SF_QOP_REDUCE)
    return launch_reduce(d, s.op, s.dtype, s.ndim, s.shape, (uint32_t)s.m, s.in[0], out);
  if (s.kind == SF_QOP_MATMUL)
    return launch_matmul(d, s.dtype, s.m, s.n, s.k, s.in[0], s.op & 1, s.in[1], (s.op >> 1) & 1,
                         out);
  const int64_t* strides[3] = {s.strides[0], s.strides[1], s.strides[2]};
  return launch_elementwise(d, s.op, s.dtype, s.ndim, s.shape, out, s.in, strides, s.imm, s.n_in);
}

// Queue (or launch) one primitive whose output buffer is already known.
int queue_submit(Device* d, const sf_op_desc& s, void* out) {
  QOp o;
  bool fits = false;
  if (d->q_max_ops > 0 && !d->alloc.capturing()) {
    if (s.kind == SF_QOP_MATMUL) {
      const long long mn = s.m * s.n;
      if ((s.dtype == SF_DTYPE_F32 || s.dtype == SF_DTYPE_F64) && mn > 0 && s.k > 0 &&
          mn <= d->q_max_numel && s.k <= 256 && s.m * s.k < (1LL << 30) &&
          s.k * s.n < (1LL << 30)) {
        std::memset(&o, 0, sizeof(o));
        o.kind = SF_QOP_MATMUL;
        o.op = s.op & 3;
        o.dtype = s.dtype;
        o.n = (int)mn;
        o.mm = (int)s.m;
        o.mk = (int)s.k;
        o.n_in = 2;
        o.in[0] = s.in[0];
        o.in[1] = s.in[1];
        fits = true;
      }
    } else if (s.kind == SF_QOP_EW) {
      fits = compact_ew(d, s, &o);
    } else if (s.kind == SF_QOP_REDUCE) {
      fits = compact_reduce(d, s, &o);
    }
  }
  if (!fits) {
    SF_TRY(queue_flush(d));
    return direct_launch(d, s, out);
  }
  o.out = out;
  std::lock_guard<std::mutex> lk(d->q_mu);
  QOpSlot slot;
  std::memcpy(&slot, &o, sizeof(o));
  d->q_ops.push_back(slot);
  d->q_pushed++;
  d->q_pending.store(1, std::memory_order_release);
  if ((int)d->q_ops.size() >= d->q_max_ops) return flush_locked(d);
  return SF_OK;
}

}  // namespace sfrt

using namespace sfrt;

extern "C" {

int sf_queue_push(int dev, const sf_op_desc* desc, void** out) {
  Device* d;
  SF_TRY(ensure_device_noflush(dev, &d));
  const sf_op_desc& s = *desc;
  size_t bytes;
  if (s.kind == SF_QOP_MATMUL) {
    if (s.m < 0 || s.n < 0 || s.k < 0) {
      set_error("sf_queue_push: bad matmul extents");
      return SF_ERR_INVALID;
    }
    bytes = (size_t)(s.m * s.n) * dtype_size(s.dtype);
    if (s.m == 0 || s.n == 0 || s.k == 0) {  // empty output / empty contraction
      bool fresh = *out == nullptr;
      if (fresh) SF_TRY(d->alloc.alloc(dev, bytes, out));
      if (s.m == 0 || s.n == 0) return SF_OK;
      SF_TRY(queue_flush(d));
      return launch_fill(d, s.dtype, s.m * s.n, 0.0, *out);
    }
  } else if (s.kind == SF_QOP_EW) {
    if (s.ndim < 0 || s.ndim > SF_MAX_DIMS || s.n_in < 1 || s.n_in > 3) {
      set_error("sf_queue_push: bad elementwise descriptor");
      return SF_ERR_INVALID;
    }
    long long n = 1;
    for (int i = 0; i < s.ndim; ++i) n *= s.shape[i];
    const int odt = s.op == SF_OP_SELECT ? s.dtype : (out_is_bool(s.op) ? SF_DTYPE_BOOL : s.dtype);
    bytes = (size_t)n * dtype_size(odt);
  } else if (s.kind == SF_QOP_REDUCE) {
    if (s.ndim < 0 || s.ndim > SF_MAX_DIMS) {
      set_error("sf_queue_push: bad reduction rank");
      return SF_ERR_INVALID;
    }
    long long n_out = 1;
    for (int i = 0; i < s.ndim; ++i)
      if (!((uint32_t)s.m & (1u << i))) n_out *= s.shape[i];
    bytes = (size_t)n_out * dtype_size(s.dtype);
  } else {
    set_error("sf_queue_push: unknown op kind");
    return SF_ERR_INVALID;
  }
  bool fresh = false;
  if (*out == nullptr) {
    SF_TRY(d->alloc.alloc(dev, bytes, out));
    fresh = true;
  }
  int st = queue_submit(d, s, *out);
  if (st != SF_OK && fresh) {
    d->alloc.release(*out);
    *out = nullptr;
  }
  return st;
}

int sf_queue_flush(int dev) {
  Device* d;
  SF_TRY(ensure_device_noflush(dev, &d));
  return queue_flush(d);
}

int sf_queue_config(int dev, int max_ops, int64_t max_numel) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));  // flushes what is queued under the old limits
  std::lock_guard<std::mutex> lk(d->q_mu);
  d->q_max_ops = max_ops < 0 ? 0 : (max_ops > kQueueMaxOps ? kQueueMaxOps : max_ops);
  d->q_max_numel = max_numel < 0 ? 0 : max_numel;
  return SF_OK;
}

int sf_queue_stats(int dev, uint64_t* pushed, uint64_t* flushes) {
  Device* d;
  SF_TRY(ensure_device_noflush(dev, &d));
  std::lock_guard<std::mutex> lk(d->q_mu);
  if (pushed) *pushed = d->q_pushed;
  if (flushes) *flushes = d->q_flushes;
  return SF_OK;
}

}  // extern "C"
