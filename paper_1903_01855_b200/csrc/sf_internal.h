// sf_internal.h — shared internals of libsfb200.so (not part of the C-ABI).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <atomic>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/sfb200.h"

namespace sfrt {

// Thread-local last error, returned by sf_last_error().
void set_error(const std::string& msg);
const char* last_error();

#define SF_CHECK_CUDA(expr)                                                     \
  do {                                                                          \
    cudaError_t _e = (expr);                                                    \
    if (_e != cudaSuccess) {                                                    \
      ::sfrt::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));    \
      return SF_ERR_CUDA;                                                       \
    }                                                                           \
  } while (0)

// Driver-API entry points, resolved through cudart at sf_init time so the
// library has no link-time dependency on libcuda (it loads on GPU-less hosts,
// where every entry point then fails with SF_ERR_NO_DEVICE).
struct DriverApi {
  CUresult (*getErrorString)(CUresult, const char**) = nullptr;
  CUresult (*moduleLoadData)(CUmodule*, const void*) = nullptr;
  CUresult (*moduleGetFunction)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*moduleGetGlobal)(CUdeviceptr*, size_t*, CUmodule, const char*) = nullptr;
  CUresult (*funcSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*launchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned,
                           unsigned, unsigned, CUstream, void**, void**) = nullptr;
  // optional: TMA im2col maps (implicit-GEMM convolution A operand)
  CUresult (*tensorMapEncodeIm2col)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const int*, const int*,
                                    cuuint32_t, cuuint32_t, const cuuint32_t*,
                                    CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill) = nullptr;
  CUresult (*tensorMapEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill) = nullptr;
};
extern DriverApi drv;

#define SF_CHECK_CU(expr)                                                       \
  do {                                                                          \
    CUresult _r = (expr);                                                       \
    if (_r != CUDA_SUCCESS) {                                                   \
      const char* _s = nullptr;                                                 \
      if (::sfrt::drv.getErrorString) ::sfrt::drv.getErrorString(_r, &_s);      \
      ::sfrt::set_error(std::string(#expr) + ": " + (_s ? _s : "?"));           \
      return SF_ERR_CUDA;                                                       \
    }                                                                           \
  } while (0)

#define SF_TRY(...)                  \
  do {                               \
    int _st = (__VA_ARGS__);         \
    if (_st != SF_OK) return _st;    \
  } while (0)

// Size-class caching allocator: one per device, stream-ordered on the
// device's single compute stream (a block freed after a launch may be
// handed to the next launch without synchronisation, because both are
// ordered on the same stream).
class Allocator {
 public:
  int alloc(int dev, size_t bytes, void** p);
  int release(void* p);
  int trim();  // return cached blocks to the driver
  size_t bytes_in_use() const { return in_use_; }
  size_t bytes_cached() const { return cached_; }

  // CUDA-graph capture: addresses handed out while a stream capture is open
  // are baked into the graph, so every block allocated during the capture
  // is logged, reused only within the capture, and at end_capture handed to
  // the graph (which gives them back with give_back when it is destroyed).
  void begin_capture();
  void end_capture(std::vector<std::pair<void*, size_t>>* owned);
  void give_back(const std::vector<std::pair<void*, size_t>>& owned);
  bool capturing() const { return capturing_; }

 private:
  static size_t round_size(size_t bytes);
  std::mutex mu_;
  std::unordered_map<size_t, std::vector<void*>> free_;
  std::unordered_map<void*, size_t> live_;
  size_t in_use_ = 0, cached_ = 0;
  bool capturing_ = false;
  std::vector<std::pair<void*, size_t>> cap_log_;
  std::unordered_map<size_t, std::vector<void*>> cap_free_;
};

// Eager launch queue (sf_queue.cu): compact descriptors of small primitives,
// executed in push order by one interpreter-kernel launch per flush.
constexpr int kQueueDims = 4;
constexpr int kQueueMaxOps = 64;
constexpr int kQueueThreads = 512;
struct QOp;  // sf_queue.cu
struct QOpSlot {
  alignas(8) unsigned char bytes[152];
};

struct Device {
  int id = 0;
  cudaStream_t stream = nullptr;
  bool external_stream = false;
  Allocator alloc;
  // pinned staging ring for host->device copies: kStageSlots slots, each
  // guarded by the event of the last transfer that read it
  static constexpr int kStageSlots = 16;
  static constexpr size_t kStageSlotBytes = 256u << 10;
  std::mutex stage_mu;
  char* pinned = nullptr;
  cudaEvent_t slot_ready[kStageSlots] = {};
  int next_slot = 0;
  // pinned bounce buffer for large host->device writes (grown on demand),
  // guarded by the event of the last transfer that read it
  char* pinned_h2d = nullptr;
  size_t pinned_h2d_bytes = 0;
  cudaEvent_t h2d_ready = nullptr;
  // pinned bounce buffer for large device->host reads (grown on demand)
  std::mutex d2h_mu;
  char* pinned_d2h = nullptr;
  size_t pinned_d2h_bytes = 0;
  int sm_count = 0;
  // arrival counters of single-launch multi-chunk reductions: zero at rest
  // (the last block of a column group resets its counter), so one array
  // serves every launch on the device's stream, graph replays included
  static constexpr int kRedCounters = 1 << 16;
  unsigned* red_counters = nullptr;
  // device RNG (Philox) state: seed and next counter offset
  unsigned long long rng_seed = 0;
  unsigned long long rng_offset = 0;
  std::mutex rng_mu;
  // eager launch queue: q_pending != 0 while q_ops is non-empty (checked
  // without the lock by every entry point that enqueues stream work)
  std::mutex q_mu;
  std::vector<QOpSlot> q_ops;
  std::atomic<int> q_pending{0};
  int q_max_ops = kQueueMaxOps;
  long long q_max_numel = 16384;
  unsigned long long q_pushed = 0, q_flushes = 0;
};

Device* device(int dev);  // nullptr if invalid
// sets the current device and validates; flushes the device's launch queue
// (every entry point that enqueues stream work calls this first)
int ensure_device(int dev, Device** out);
// the same without the flush (allocation, counters, queue pushes)
int ensure_device_noflush(int dev, Device** out);
int queue_flush(Device* d);
int queue_flush_dev(int dev);
size_t dtype_size(int dtype);
void count_launch(int dev, unsigned long long n = 1);

// Kernel launchers shared between the eager entry points and the plan
// executor (all stream-ordered on d->stream).
int launch_elementwise(Device* d, int op, int dtype, int ndim, const int64_t* shape,
                       void* out, const void* const* ins, const int64_t* const* strides,
                       const double* imms, int n_in);
int launch_reduce(Device* d, int op, int dtype, int ndim, const int64_t* shape,
                  uint32_t axes_mask, const void* in, void* out);
int launch_matmul(Device* d, int dtype, int64_t m, int64_t n, int64_t k, const void* a,
                  int trans_a, const void* b, int trans_b, void* c);
int launch_transpose2d(Device* d, int dtype, int64_t rows, int64_t cols, const void* in,
                       void* out);
int launch_fill(Device* d, int dtype, int64_t n, double value, void* out);
int launch_eye(Device* d, int dtype, int64_t n, void* out);
int launch_rng(Device* d, int kind, int dtype, int64_t n, unsigned long long seed,
               unsigned long long offset, void* out);
int launch_dropout(Device* d, int dtype, int64_t n, const void* x, const void* u,
                   int u_dtype, double rate, void* out, void* mask);
int launch_cast(Device* d, int src_dtype, int dst_dtype, int64_t n, const void* in, void* out);

// reduce_sum/mean geometry: kept and reduced dims (size-1 dims dropped,
// contiguous dims merged), element strides of a row-major input
struct RedGeom {
  long long n_out, r;
  int kept_nd, red_nd;
  long long kept_shape[SF_MAX_DIMS], kept_stride[SF_MAX_DIMS];
  long long red_shape[SF_MAX_DIMS], red_stride[SF_MAX_DIMS];
};
void reduce_geometry(int ndim, const int64_t* shape, uint32_t axes_mask, RedGeom* g);

// NCCL (sf_comm.cpp): grouped in-place all-reduce forked from the device
// stream onto the communicator's stream; comm_join makes the device stream
// wait for everything enqueued so far
int comm_allreduce(void* comm, Device* d, void* const* bufs, const size_t* counts, int n,
                   int dtype, double scale);
int comm_join(void* comm, Device* d);

// Row-kernel constant pool (sf_plan.cpp step kind 1 with a pool section):
// gather the kernel's uniform operands into `image` at their pool offsets
// (rows of N elements padded to Np), then the image is copied into the
// module's __constant__ cpool.
struct CpoolEntry {
  const void* src;
  uint32_t dst_off, n, width, N, Np, pad;
};
int launch_cpool_gather(Device* d, const CpoolEntry* e, int n, void* image);
// device address and size of a jitted kernel's module global (loads the module)
int jit_global(void* kernel, int dev, const char* name, void** ptr, size_t* bytes);
std::mutex& jit_mutex(void* kernel);

}  // namespace sfrt
