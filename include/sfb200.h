/*
 * sfb200.h — C-ABI of libsfb200.so, the sm_100a execution backend behind the
 * stageflow-compatible front-end in paper_1903_01855_b200/.
 *
 * Every entry point is extern "C", takes plain pointers and sizes, returns an
 * int status (SF_OK == 0) and leaves a message for sf_last_error() on
 * failure.  All device work is stream-ordered on the device's single compute
 * stream; host-visible results (sf_memcpy_d2h) synchronise that stream.
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src):
 *   sf_alloc / sf_free / sf_memcpy_*  -> numpy buffer ownership in
 *        stageflow/tensor.py:38-70 (Tensor storage), :138-172 (host interchange)
 *        and the relabelling copies of stageflow/ops.py:245-286
 *   sf_elementwise  -> _binary_kernel / _unary_kernel / _greater_kernel /
 *        _broadcast_to_kernel / _identity_kernel, stageflow/kernels.py:116-181,
 *        :222-232, :263-279, :307-315
 *   sf_reduce       -> _reduce_kernel (np.sum / np.mean), stageflow/kernels.py:323-364
 *   sf_matmul       -> _matmul_kernel (np.matmul), stageflow/kernels.py:184-208
 *   sf_transpose2d  -> _transpose_kernel, stageflow/kernels.py:211-219
 *   sf_fill / sf_eye-> _eye_kernel / gradients.zeros_for/ones_for,
 *        stageflow/kernels.py:282-292, stageflow/gradients.py:65-76
 *   sf_rng          -> _random_normal_kernel (Runtime.draw), stageflow/kernels.py:372-384
 *   sf_dropout      -> _dropout_kernel, stageflow/kernels.py:387-404
 *   sf_jit_* / sf_plan_* -> execute_graph + _Plan, stageflow/executor.py:58-269
 *        (the traced graph is lowered once into fused kernels and replayed)
 */
#ifndef SFB200_H_
#define SFB200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define SF_OK 0
#define SF_ERR_INVALID 1
#define SF_ERR_CUDA 2
#define SF_ERR_OOM 3
#define SF_ERR_NVRTC 4
#define SF_ERR_UNSUPPORTED 5
#define SF_ERR_NO_DEVICE 6

/* dtype tags (same values as the reference wire tags, stageflow/dtypes.py:63-69) */
#define SF_DTYPE_F32 1
#define SF_DTYPE_F64 2
#define SF_DTYPE_I32 3
#define SF_DTYPE_BOOL 4

#define SF_MAX_DIMS 8

/* ---------------------------------------------------------------- runtime */
const char* sf_last_error(void);
int sf_version(void);
/* Enumerate CUDA devices; creates one non-blocking stream and one caching
 * allocator per device.  Idempotent. */
int sf_init(int* n_devices);
int sf_device_info(int dev, int* sm_count, int* cc_major, int* cc_minor, size_t* total_mem);
/* Route all work for `dev` onto an external stream (e.g. torch's current
 * stream, for NCCL interop); NULL restores the backend's own stream. */
int sf_set_stream(int dev, void* stream);
int sf_get_stream(int dev, void** stream);
int sf_device_sync(int dev);

int sf_alloc(int dev, size_t bytes, void** p);
int sf_free(int dev, void* p);
int sf_mem_stats(int dev, size_t* bytes_in_use, size_t* bytes_cached);
int sf_trim(int dev);
/* The device's arrival counters for single-launch multi-chunk column
 * reductions (zero at rest; every kernel using them leaves them zero).
 * Lowered (NVRTC) reduction kernels receive this address as a parameter.
 * Replaces: nothing in the reference (np.sum is one call). */
int sf_reduce_counters(int dev, void** counters);
/* Page-locked host memory (cudaHostAlloc, portable).  Transfers to/from it
 * skip the staging copies: sf_memcpy_d2h writes it directly, sf_memcpy_h2d
 * reads it directly when the stream is idle. */
int sf_host_alloc(size_t bytes, void** p);
int sf_host_free(void* p);

/* host <-> device copies.  h2d copies the host bytes before returning (the
 * caller may reuse `src` immediately); d2h blocks until the data is on the
 * host. */
int sf_memcpy_h2d(int dev, void* dst, const void* src, size_t bytes);
/* h2d from a source the caller guarantees immutable and alive until the
 * copy has executed (a read-only host array the new tensor keeps): a
 * page-locked source is DMA'd without waiting (*async = 1), others take the
 * sf_memcpy_h2d path.  Replaces: tensor_from_host's copy,
 * stageflow/tensor.py:138-162. */
int sf_memcpy_h2d_immutable(int dev, void* dst, const void* src, size_t bytes, int* async);
int sf_memcpy_d2h(int dev, void* dst, const void* src, size_t bytes);
/* d2h into page-locked memory, enqueued only: complete once any later
 * synchronising call on the device's stream returns (used to read a call's
 * small sibling outputs in the same round trip as the one asked for). */
int sf_memcpy_d2h_enqueue(int dev, void* dst, const void* src, size_t bytes);
int sf_memcpy_d2d(int dev, void* dst, const void* src, size_t bytes);
int sf_memcpy_p2p(int dst_dev, void* dst, int src_dev, const void* src, size_t bytes);

/* ------------------------------------------------------- eager primitives
 * Each launch allocates its output(s) from the caching allocator when the
 * passed *out is NULL, otherwise writes into *out. */

/* Packed elementwise descriptor (little-endian, natural alignment). */
typedef struct sf_ew_desc {
  int32_t op;          /* SF_OP_* from csrc/sf_ops.cuh */
  int32_t dtype;       /* input dtype; the output dtype follows the op */
  int32_t ndim;        /* <= SF_MAX_DIMS, 0 for scalars */
  int32_t n_in;        /* 1, 2 or 3 */
  const void* in[3];   /* NULL => operand is the immediate imm[i] */
  double imm[3];
  int64_t shape[SF_MAX_DIMS];       /* output shape */
  int64_t strides[3][SF_MAX_DIMS];  /* element strides per operand, 0 = broadcast */
} sf_ew_desc;

int sf_elementwise(int dev, const sf_ew_desc* desc, void** out);

/* ------------------------------------------------------- eager launch queue
 * Small primitives are queued as compact descriptors and executed in push
 * order by ONE launch of an interpreter kernel (a single CTA, one barrier
 * between consecutive ops, the same per-element functions and matmul
 * contract as the one-op kernels: queued and direct results are
 * bit-identical).  The queue is flushed when full, by sf_queue_flush, and
 * before any other call that enqueues work on the device's stream (copies,
 * syncs, plan runs, graph launches and captures), so stream order is push
 * order.  Ops too large for the queue (> max_numel elements, rank > 4 after
 * collapsing, k > 256 matmuls) flush it and launch directly.
 * sf_elementwise, sf_matmul, sf_transpose2d, sf_fill and the short float
 * reductions of sf_reduce (<= 1024 elements per output: one CRO chunk,
 * evaluated by one warp per output with the same fold and butterfly) go
 * through it.
 * Replaces: the per-op np.* call of _dispatch_eager -> kernel,
 * stageflow/ops.py:318-347 (kernels.py:116-219); the reference has no queue
 * (every op runs to completion inside dispatch). */
#define SF_QOP_EW 0
#define SF_QOP_MATMUL 1
#define SF_QOP_REDUCE 2 /* op: 0 sum, 1 mean; m = axes mask (float dtypes) */
typedef struct sf_op_desc {
  int32_t kind;   /* SF_QOP_* */
  int32_t op;     /* EW: SF_OP_*; MATMUL: bit0 = A transposed, bit1 = B transposed */
  int32_t dtype;  /* input dtype */
  int32_t ndim;   /* EW: output rank */
  int32_t n_in;   /* EW: 1..3 */
  int32_t pad;
  int64_t m, n, k;  /* MATMUL: C[m,n] = op(A)[m,k] @ op(B)[k,n] */
  const void* in[3];  /* NULL => immediate imm[i] (EW) */
  double imm[3];
  int64_t shape[SF_MAX_DIMS];
  int64_t strides[3][SF_MAX_DIMS];
} sf_op_desc;
/* Queue (or, when it does not fit, launch) one primitive; allocates *out
 * from the caching allocator when NULL. */
int sf_queue_push(int dev, const sf_op_desc* desc, void** out);
int sf_queue_flush(int dev);
/* max_ops (<= 64) per launch, 0 disables queueing; max_numel per op. */
int sf_queue_config(int dev, int max_ops, int64_t max_numel);
int sf_queue_stats(int dev, uint64_t* pushed, uint64_t* flushes);
/* op: 0 = sum, 1 = mean.  axes_mask bit i set => axis i reduced. */
int sf_reduce(int dev, int op, int dtype, int ndim, const int64_t* shape, uint32_t axes_mask,
              const void* in, void** out);
/* C[m,n] = op(A) @ op(B), row-major; trans_* = 1 reads the operand transposed. */
int sf_matmul(int dev, int dtype, int64_t m, int64_t n, int64_t k, const void* a, int trans_a,
              const void* b, int trans_b, void** out);
int sf_transpose2d(int dev, int dtype, int64_t rows, int64_t cols, const void* in, void** out);
int sf_fill(int dev, int dtype, int64_t n, double value, void** out);
int sf_eye(int dev, int dtype, int64_t n, void** out);
int sf_cast(int dev, int src_dtype, int dst_dtype, int64_t n, const void* in, void** out);
/* Device Philox RNG.  kind: 0 = standard normal, 1 = uniform [0,1).
 * offset == UINT64_MAX reserves the next n counters from the device stream. */
int sf_rng_seed(int dev, uint64_t seed);
int sf_rng_reserve(int dev, uint64_t n, uint64_t* offset);
int sf_rng(int dev, int kind, int dtype, int64_t n, uint64_t offset, void** out);
/* dropout: mask = (u >= rate) / (1 - rate) in dtype; out = x * mask.  u is a
 * buffer of uniforms of dtype u_dtype (host-drawn parity mode) or NULL to
 * draw from the device Philox stream. */
int sf_dropout(int dev, int dtype, int64_t n, const void* x, const void* u, int u_dtype,
               double rate, void** out, void** mask);

/* ------------------------------------------------------------ collectives
 * NCCL (libnccl.so.2, opened at first use) for the data-parallel gradient
 * all-reduce of config C5 — the build's only exchange step.  Each
 * communicator owns a comm stream; an all-reduce is forked from the
 * device's stream after the work enqueued so far and runs grouped and in
 * place.  Staged plans issue them per gradient bucket as the backward
 * produces the bucket (plan step 12) and join once at the end, so the
 * transfers overlap the remaining backward kernels.
 * Replaces: nothing in the reference (it has no distribution);
 * SURVEY.md §8(b) sf_nccl_init / sf_allreduce. */
/* 128-byte NCCL unique id (rank 0 creates it; every rank passes it to init) */
int sf_comm_unique_id(void* id_out);
int sf_comm_init(int dev, int nranks, int rank, const void* id, void** comm);
int sf_comm_destroy(void* comm);
/* Sum-all-reduce n buffers in place (counts in elements); scale != 1 sums
 * scale * x (NCCL premul sum).  Ordered after earlier work on the device's
 * stream; later work on it waits for the result. */
int sf_allreduce(void* comm, void* const* bufs, const size_t* counts, int n, int dtype,
                 double scale);
int sf_nccl_version(int* version);

/* ------------------------------------------------------- NN plugin kernels
 * (ResNet-50, configs C4/C5; no reference counterpart — the reference has no
 * convolution/pooling/xent).  NHWC; g8 = {N, H, W, C, KH, KW,
 * stride, pad}; output spatial size (H + 2 pad - KH) / stride + 1. */
int sf_im2col(int dev, int dtype, const int64_t* g8, const void* x, void** cols);
int sf_col2im(int dev, int dtype, const int64_t* g8, const void* dcols, void** dx);
/* f32 im2col written directly as 3xTF32 hi/lo parts with K padded to kp */
int sf_im2col_split(int dev, const int64_t* g8, int64_t kp, const void* x, void** hi, void** lo);
int sf_maxpool2d(int dev, int dtype, const int64_t* g8, const void* x, void** y);
int sf_maxpool2d_grad(int dev, int dtype, const int64_t* g8, const void* x, const void* dy,
                      void** dx);
/* per-row softmax cross-entropy with int32 labels, and its gradient scaled by g[row] */
int sf_softmax_xent(int dev, int dtype, int64_t rows, int64_t k, const void* logits,
                    const void* labels, void** loss);
int sf_softmax_xent_grad(int dev, int dtype, int64_t rows, int64_t k, const void* logits,
                         const void* labels, const void* g, void** out);

/* fp32-class GEMM on tcgen05 tensor cores (3xTF32):
 * C[m,n] = A[m,k] . B[n,k]^T, both operands K-major and pre-split into
 * hi (TF32-representable) + lo parts; k must be a multiple of 4. */
int sf_gemm_tf32x3(int dev, int64_t m, int64_t n, int64_t k, const void* a_hi, const void* a_lo,
                   const void* b_hi, const void* b_lo, void** c);
/* General form: a_mn / b_mn = 1 when the operand is stored MN-major
 * (A as k x m, B as k x n, the GEMM's m / n index contiguous) — e.g. the
 * activations of a weight-gradient GEMM — so no transposed copy is needed.
 * ak / bk: contraction rows each operand actually holds (<= k, zero beyond).
 * Leading dimensions (k-major: ak/bk; MN-major: m/n) must be multiples of 4. */
int sf_gemm_tf32x3_ex(int dev, int64_t m, int64_t n, int64_t k, int a_mn, int b_mn, int64_t ak,
                      int64_t bk, const void* a_hi, const void* a_lo, const void* b_hi,
                      const void* b_lo, void** c);
/* Implicit-GEMM convolution on tcgen05 (3xTF32), NHWC float32:
 * out[n*ho*wo, co] = im2col(x) . W with W (kh*kw*c, co) row-major and
 * g8 = {N, H, W, C, KH, KW, stride, pad}; the im2col rows are loaded into
 * shared memory by the GEMM itself (TMA im2col boxes, or cp.async gathers
 * where the driver has no im2col maps) and never materialised.  Requires
 * C % 32 == 0 and co % 4 == 0 (else SF_ERR_INVALID).  Bit-identical to
 * sf_im2col + sf_gemm_tf32x3_ex.  Replaces the im2col + GEMM of the
 * reference's conv2d plugin kernel (oracle/ref_plugins.py, the numpy
 * restatement of the C4 workload's convolution). */
int sf_conv2d_tc(int dev, const int64_t* g8, int64_t co, const void* x, const void* w,
                 void** out);
/* hi/lo split of an fp32 (rows x cols) matrix; transpose=1 writes the
 * (cols x ldo) transpose with rows zero-padded to ldo.  Without transpose,
 * hi may be NULL: the tensor cores ignore an fp32 operand's low 13 mantissa
 * bits, so the unsplit matrix can be passed as the hi operand. */
int sf_split_tf32(int dev, int64_t rows, int64_t cols, int64_t ldo, int transpose, const void* x,
                  void** hi, void** lo);

/* ------------------------------------------------------- staged graphs */
/* Compile CUDA C++ source (which may #include "sf_ops.cuh") for sm_100a with
 * NVRTC and load it; returns an opaque kernel handle. Cached by source. */
int sf_jit_compile(const char* kernel_name, const char* source, void** kernel);
const char* sf_jit_log(void);
/* Launch a jitted kernel with one by-value parameter blob. */
int sf_jit_launch(int dev, void* kernel, unsigned grid, unsigned block, unsigned smem,
                  const void* params, size_t params_bytes);

/* A plan is a lowered graph function: a list of steps over value slots
 * (inputs, plan-owned constants, per-call temporaries, outputs).  The binary
 * plan format is documented in csrc/sf_plan.cpp. */
int sf_plan_create(int dev, const void* desc, size_t desc_bytes, void** plan);
/* Runs the plan on its device's stream.  inputs: n_inputs device pointers;
 * outputs: receives n_outputs freshly allocated device pointers (ownership
 * passes to the caller, release with sf_free). */
int sf_plan_run(void* plan, const void* const* inputs, void** outputs);
int sf_plan_info(void* plan, int* n_inputs, int* n_outputs, int* n_steps, int* n_launches);
/* Per-step GPU timing: when enabled, every run brackets each step with CUDA
 * events on the device stream, synchronises, and accumulates the durations
 * (measurement aid for the roofline; adds a stream sync per run). */
int sf_plan_profile(void* plan, int enable);
int sf_plan_step_stats(void* plan, int step, int* kind, double* total_ms, uint64_t* runs);
int sf_plan_destroy(void* plan);

/* ------------------------------------------------------- device while_loop */
/* Replaces the host loop of _while_kernel (stageflow/kernels.py:513-538):
 * a CUDA graph  [cond -> set_cond] -> WHILE { body -> state copies -> cond
 * -> set_cond }  recorded by stream capture of the cond/body plans, so the
 * predicate never travels to the host.  Protocol: create; fixed buffers
 * (loop state, captures) with sf_while_buffer; capture part 0 (prologue:
 * cond plan + sf_while_set_cond), then part 1 (body plan, copies, cond plan,
 * sf_while_set_cond); then sf_while_launch per call.  Blocks allocated while
 * a capture is open belong to the graph until sf_while_destroy. */
int sf_while_create(int dev, void** w);
/* Device-side cond (replaces _cond_kernel's host read of the predicate,
 * stageflow/kernels.py:493-510): same object and protocol, an IF node with
 * an else branch; parts 0 = prologue (sf_while_set_cond on the predicate
 * buffer), 1 = then branch, 2 = else branch. */
int sf_cond_create(int dev, void** w);
/* Whole-program replay: the same object with a single part 0 and no
 * conditional node — a staged program recorded once by stream capture and
 * replayed with one graph launch per call (sf_while_launch). */
int sf_graph_create(int dev, void** w);
int sf_while_buffer(void* w, size_t bytes, void** p);
int sf_while_capture_begin(void* w, int part);
/* enqueue (inside a capture) the kernel that sets the loop handle from a
 * device boolean */
int sf_while_set_cond(void* w, const void* pred);
int sf_while_capture_end(void* w, int part);
int sf_while_launch(void* w);
int sf_while_destroy(void* w);

/* ------------------------------------------------------- counters */
/* number of kernels this library has launched on `dev` since sf_init */
int sf_launch_count(int dev, uint64_t* count);

#ifdef __cplusplus
}
#endif

#endif /* SFB200_H_ */
