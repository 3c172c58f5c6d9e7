// sf_runtime.cu — devices, streams, caching allocator, host<->device copies.
//
// Replaces the reference's storage model: a Tensor there owns a read-only
// numpy buffer (stageflow/tensor.py:38-70) and "device copies" only relabel
// it (stageflow/ops.py:245-286).  Here a tensor's bytes live in HBM, carved
// out of a per-device size-class cache, and every copy is a real transfer
// ordered on the device's single compute stream.
#include <atomic>
#include <memory>

#include "sf_internal.h"

namespace sfrt {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
const char* last_error() { return g_err.c_str(); }

DriverApi drv;

template <class F>
static int resolve(const char* name, F* fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !p) {
    (void)cudaGetLastError();
    set_error(std::string("cannot resolve driver entry point ") + name);
    return SF_ERR_CUDA;
  }
  *fn = reinterpret_cast<F>(p);
  return SF_OK;
}

static std::mutex g_init_mu;
static std::vector<std::unique_ptr<Device>> g_devices;
static bool g_inited = false;
std::atomic<unsigned long long> g_launches[64];

Device* device(int dev) {
  if (dev < 0 || dev >= (int)g_devices.size()) return nullptr;
  return g_devices[dev].get();
}

static thread_local int t_current = -1;

int ensure_device(int dev, Device** out) {
  SF_TRY(ensure_device_noflush(dev, out));
  Device* d = *out;
  if (d->q_pending.load(std::memory_order_acquire)) return queue_flush(d);
  return SF_OK;
}

int ensure_device_noflush(int dev, Device** out) {
  if (!g_inited) {
    int n = 0;
    SF_TRY(sf_init(&n));
  }
  Device* d = device(dev);
  if (!d) {
    set_error("invalid device ordinal " + std::to_string(dev));
    return SF_ERR_NO_DEVICE;
  }
  if (t_current != dev) {
    SF_CHECK_CUDA(cudaSetDevice(dev));
    t_current = dev;
  }
  *out = d;
  return SF_OK;
}

size_t dtype_size(int dtype) {
  switch (dtype) {
    case SF_DTYPE_F32: return 4;
    case SF_DTYPE_F64: return 8;
    case SF_DTYPE_I32: return 4;
    case SF_DTYPE_BOOL: return 1;
    default: return 0;
  }
}

void count_launch(int dev, unsigned long long n) {
  if (dev >= 0 && dev < 64) g_launches[dev].fetch_add(n, std::memory_order_relaxed);
}

// ------------------------------------------------------------- allocator
size_t Allocator::round_size(size_t bytes) {
  if (bytes == 0) bytes = 1;
  if (bytes <= 512) return 512;
  if (bytes <= (1u << 20)) {  // next power of two up to 1 MiB
    size_t s = 1024;
    while (s < bytes) s <<= 1;
    return s;
  }
  const size_t g = 2u << 20;  // 2 MiB granules above
  return (bytes + g - 1) / g * g;
}

int Allocator::alloc(int dev, size_t bytes, void** p) {
  const size_t sz = round_size(bytes);
  {
    std::lock_guard<std::mutex> lk(mu_);
    if (capturing_) {
      auto ct = cap_free_.find(sz);
      if (ct != cap_free_.end() && !ct->second.empty()) {
        *p = ct->second.back();
        ct->second.pop_back();
        live_[*p] = sz;
        in_use_ += sz;
        return SF_OK;
      }
    }
    auto it = free_.find(sz);
    if (it != free_.end() && !it->second.empty()) {
      *p = it->second.back();
      it->second.pop_back();
      live_[*p] = sz;
      in_use_ += sz;
      cached_ -= sz;
      if (capturing_) cap_log_.emplace_back(*p, sz);
      return SF_OK;
    }
  }
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, sz);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    if (capturing_) {
      set_error("device " + std::to_string(dev) + ": out of memory during graph capture");
      return SF_ERR_OOM;
    }
    // Return the cache to the driver and retry once (queued ops may still
    // read cached blocks: launch them first).
    queue_flush_dev(dev);
    cudaDeviceSynchronize();
    trim();
    e = cudaMalloc(&q, sz);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      set_error("device " + std::to_string(dev) + ": out of memory allocating " +
                std::to_string(sz) + " bytes");
      return SF_ERR_OOM;
    }
  }
  std::lock_guard<std::mutex> lk(mu_);
  live_[q] = sz;
  in_use_ += sz;
  if (capturing_) cap_log_.emplace_back(q, sz);
  *p = q;
  return SF_OK;
}

int Allocator::release(void* p) {
  if (!p) return SF_OK;
  std::lock_guard<std::mutex> lk(mu_);
  auto it = live_.find(p);
  if (it == live_.end()) {
    set_error("sf_free: pointer not owned by this device's allocator");
    return SF_ERR_INVALID;
  }
  const size_t sz = it->second;
  live_.erase(it);
  in_use_ -= sz;
  if (capturing_) {
    for (const auto& e : cap_log_) {
      if (e.first == p) {  // captured block: reusable only inside this capture
        cap_free_[sz].push_back(p);
        return SF_OK;
      }
    }
  }
  cached_ += sz;
  free_[sz].push_back(p);
  return SF_OK;
}

void Allocator::begin_capture() {
  std::lock_guard<std::mutex> lk(mu_);
  capturing_ = true;
  cap_log_.clear();
  cap_free_.clear();
}

void Allocator::end_capture(std::vector<std::pair<void*, size_t>>* owned) {
  std::lock_guard<std::mutex> lk(mu_);
  for (const auto& e : cap_log_) {
    auto it = live_.find(e.first);
    if (it == live_.end()) in_use_ += e.second;  // released inside the capture
    else live_.erase(it);
    owned->push_back(e);  // counted in use until the graph gives it back
  }
  cap_log_.clear();
  cap_free_.clear();
  capturing_ = false;
}

void Allocator::give_back(const std::vector<std::pair<void*, size_t>>& owned) {
  std::lock_guard<std::mutex> lk(mu_);
  for (const auto& e : owned) {
    in_use_ -= e.second;
    cached_ += e.second;
    free_[e.second].push_back(e.first);
  }
}

int Allocator::trim() {
  std::lock_guard<std::mutex> lk(mu_);
  for (auto& kv : free_) {
    for (void* p : kv.second) cudaFree(p);
    kv.second.clear();
  }
  cached_ = 0;
  return SF_OK;
}

}  // namespace sfrt

using namespace sfrt;

extern "C" {

const char* sf_last_error(void) { return last_error(); }
int sf_version(void) { return 100; }

int sf_init(int* n_devices) {
  std::lock_guard<std::mutex> lk(g_init_mu);
  if (g_inited) {
    if (n_devices) *n_devices = (int)g_devices.size();
    return SF_OK;
  }
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    (void)cudaGetLastError();
    set_error(std::string("no CUDA device available: ") +
              (e == cudaSuccess ? "device count is 0" : cudaGetErrorString(e)));
    return SF_ERR_NO_DEVICE;
  }
  SF_TRY(resolve("cuGetErrorString", &drv.getErrorString));
  SF_TRY(resolve("cuModuleLoadData", &drv.moduleLoadData));
  SF_TRY(resolve("cuModuleGetFunction", &drv.moduleGetFunction));
  SF_TRY(resolve("cuModuleGetGlobal", &drv.moduleGetGlobal));
  SF_TRY(resolve("cuFuncSetAttribute", &drv.funcSetAttribute));
  SF_TRY(resolve("cuLaunchKernel", &drv.launchKernel));
  SF_TRY(resolve("cuTensorMapEncodeTiled", &drv.tensorMapEncodeTiled));
  if (resolve("cuTensorMapEncodeIm2col", &drv.tensorMapEncodeIm2col) != SF_OK)
    drv.tensorMapEncodeIm2col = nullptr;
  for (int i = 0; i < n && i < 64; ++i) {
    auto d = std::make_unique<Device>();
    d->id = i;
    SF_CHECK_CUDA(cudaSetDevice(i));
    SF_CHECK_CUDA(cudaFree(nullptr));  // create the primary context
    SF_CHECK_CUDA(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
    SF_CHECK_CUDA(cudaDeviceGetAttribute(&d->sm_count, cudaDevAttrMultiProcessorCount, i));
    SF_CHECK_CUDA(cudaMalloc((void**)&d->red_counters, sizeof(unsigned) * Device::kRedCounters));
    SF_CHECK_CUDA(cudaMemset(d->red_counters, 0, sizeof(unsigned) * Device::kRedCounters));
    SF_CHECK_CUDA(cudaMallocHost((void**)&d->pinned, Device::kStageSlots * Device::kStageSlotBytes));
    for (int k = 0; k < Device::kStageSlots; ++k)
      SF_CHECK_CUDA(cudaEventCreateWithFlags(&d->slot_ready[k], cudaEventDisableTiming));
    g_devices.push_back(std::move(d));
    g_launches[i] = 0;
  }
  t_current = -1;
  g_inited = true;
  if (n_devices) *n_devices = (int)g_devices.size();
  return SF_OK;
}

int sf_device_info(int dev, int* sm_count, int* cc_major, int* cc_minor, size_t* total_mem) {
  Device* d;
  SF_TRY(ensure_device_noflush(dev, &d));
  cudaDeviceProp prop;
  SF_CHECK_CUDA(cudaGetDeviceProperties(&prop, dev));
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  if (total_mem) *total_mem = prop.totalGlobalMem;
  return SF_OK;
}

int sf_set_stream(int dev, void* stream) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  SF_CHECK_CUDA(cudaStreamSynchronize(d->stream));
  if (stream == nullptr) {
    if (d->external_stream) {
      SF_CHECK_CUDA(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
      d->external_stream = false;
    }
    return SF_OK;
  }
  if (!d->external_stream) SF_CHECK_CUDA(cudaStreamDestroy(d->stream));
  d->stream = (cudaStream_t)stream;
  d->external_stream = true;
  return SF_OK;
}

int sf_get_stream(int dev, void** stream) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  *stream = (void*)d->stream;
  return SF_OK;
}

int sf_device_sync(int dev) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  SF_CHECK_CUDA(cudaStreamSynchronize(d->stream));
  SF_CHECK_CUDA(cudaGetLastError());
  return SF_OK;
}

int sf_alloc(int dev, size_t bytes, void** p) {
  Device* d;
  SF_TRY(ensure_device_noflush(dev, &d));
  return d->alloc.alloc(dev, bytes, p);
}

int sf_free(int dev, void* p) {
  Device* d = device(dev);
  if (!d) {
    set_error("sf_free: invalid device");
    return SF_ERR_NO_DEVICE;
  }
  return d->alloc.release(p);
}

int sf_reduce_counters(int dev, void** counters) {
  Device* d;
  SF_TRY(ensure_device_noflush(dev, &d));
  *counters = d->red_counters;
  return SF_OK;
}

int sf_mem_stats(int dev, size_t* in_use, size_t* cached) {
  Device* d;
  SF_TRY(ensure_device_noflush(dev, &d));
  if (in_use) *in_use = d->alloc.bytes_in_use();
  if (cached) *cached = d->alloc.bytes_cached();
  return SF_OK;
}

int sf_trim(int dev) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  SF_CHECK_CUDA(cudaStreamSynchronize(d->stream));
  return d->alloc.trim();
}

int sf_host_alloc(size_t bytes, void** p) {
  int n = 0;
  SF_TRY(sf_init(&n));
  SF_CHECK_CUDA(cudaHostAlloc(p, bytes ? bytes : 1, cudaHostAllocPortable));
  return SF_OK;
}

int sf_host_free(void* p) {
  if (p) SF_CHECK_CUDA(cudaFreeHost(p));
  return SF_OK;
}

int sf_memcpy_h2d_immutable(int dev, void* dst, const void* src, size_t bytes, int* async) {
  // The caller guarantees src is immutable and outlives the transfer: a
  // page-locked source is DMA'd asynchronously (no wait), anything else takes
  // the regular path.
  if (async) *async = 0;
  if (bytes == 0) return SF_OK;
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, src) == cudaSuccess && attr.type == cudaMemoryTypeHost) {
    SF_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, d->stream));
    if (async) *async = 1;
    return SF_OK;
  }
  (void)cudaGetLastError();
  return sf_memcpy_h2d(dev, dst, src, bytes);
}

int sf_memcpy_h2d(int dev, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return SF_OK;
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  if (bytes <= Device::kStageSlotBytes) {
    // Stage through the next pinned ring slot: wait until the transfer that
    // last read this slot has executed, copy, enqueue.  The caller's buffer
    // is free on return and the transfer stays asynchronous.
    std::lock_guard<std::mutex> lk(d->stage_mu);
    const int k = d->next_slot;
    d->next_slot = (k + 1) % Device::kStageSlots;
    SF_CHECK_CUDA(cudaEventSynchronize(d->slot_ready[k]));
    char* slot = d->pinned + (size_t)k * Device::kStageSlotBytes;
    std::memcpy(slot, src, bytes);
    SF_CHECK_CUDA(cudaMemcpyAsync(dst, slot, bytes, cudaMemcpyHostToDevice, d->stream));
    SF_CHECK_CUDA(cudaEventRecord(d->slot_ready[k], d->stream));
    return SF_OK;
  }
  {
    // pinned source and an idle stream: DMA straight from the caller's buffer
    // and wait for just that copy (the buffer must be free on return) —
    // saves the host memcpy into the bounce buffer
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, src) == cudaSuccess && attr.type == cudaMemoryTypeHost &&
        cudaStreamQuery(d->stream) == cudaSuccess) {
      SF_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, d->stream));
      SF_CHECK_CUDA(cudaStreamSynchronize(d->stream));
      return SF_OK;
    }
    (void)cudaGetLastError();  // clear cudaErrorNotReady from the query
  }
  if (bytes <= (256u << 20)) {
    // larger transfers: one pinned bounce buffer, asynchronous w.r.t. the stream
    std::lock_guard<std::mutex> lk(d->stage_mu);
    if (d->h2d_ready) SF_CHECK_CUDA(cudaEventSynchronize(d->h2d_ready));
    else SF_CHECK_CUDA(cudaEventCreateWithFlags(&d->h2d_ready, cudaEventDisableTiming));
    if (d->pinned_h2d_bytes < bytes) {
      if (d->pinned_h2d) cudaFreeHost(d->pinned_h2d);
      size_t want = 1u << 20;
      while (want < bytes) want <<= 1;
      SF_CHECK_CUDA(cudaMallocHost((void**)&d->pinned_h2d, want));
      d->pinned_h2d_bytes = want;
    }
    std::memcpy(d->pinned_h2d, src, bytes);
    SF_CHECK_CUDA(cudaMemcpyAsync(dst, d->pinned_h2d, bytes, cudaMemcpyHostToDevice, d->stream));
    SF_CHECK_CUDA(cudaEventRecord(d->h2d_ready, d->stream));
    return SF_OK;
  }
  SF_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, d->stream));
  SF_CHECK_CUDA(cudaStreamSynchronize(d->stream));
  return SF_OK;
}

int sf_memcpy_d2h_enqueue(int dev, void* dst, const void* src, size_t bytes) {
  // dst must be page-locked; the copy completes with the stream's next sync
  if (bytes == 0) return SF_OK;
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, dst) != cudaSuccess || attr.type != cudaMemoryTypeHost) {
    (void)cudaGetLastError();
    set_error("sf_memcpy_d2h_enqueue: destination is not page-locked host memory");
    return SF_ERR_INVALID;
  }
  SF_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, d->stream));
  return SF_OK;
}

int sf_memcpy_d2h(int dev, void* dst, const void* src, size_t bytes) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  if (bytes == 0) {
    SF_CHECK_CUDA(cudaStreamSynchronize(d->stream));
    return SF_OK;
  }
  cudaPointerAttributes attr;
  const bool pinned_dst =
      cudaPointerGetAttributes(&attr, dst) == cudaSuccess && attr.type == cudaMemoryTypeHost;
  (void)cudaGetLastError();
  if (bytes >= (64u << 10) && bytes <= (256u << 20) && !pinned_dst) {
    // DMA into a pinned bounce buffer at full PCIe/C2C speed, then one memcpy
    // (a pinned destination, e.g. sf_host_alloc memory, is written directly)
    std::lock_guard<std::mutex> lk(d->d2h_mu);
    if (d->pinned_d2h_bytes < bytes) {
      if (d->pinned_d2h) cudaFreeHost(d->pinned_d2h);
      size_t want = 1u << 20;
      while (want < bytes) want <<= 1;
      SF_CHECK_CUDA(cudaMallocHost((void**)&d->pinned_d2h, want));
      d->pinned_d2h_bytes = want;
    }
    SF_CHECK_CUDA(cudaMemcpyAsync(d->pinned_d2h, src, bytes, cudaMemcpyDeviceToHost, d->stream));
    SF_CHECK_CUDA(cudaStreamSynchronize(d->stream));
    std::memcpy(dst, d->pinned_d2h, bytes);
    return SF_OK;
  }
  SF_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, d->stream));
  SF_CHECK_CUDA(cudaStreamSynchronize(d->stream));
  return SF_OK;
}

int sf_memcpy_d2d(int dev, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return SF_OK;
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  SF_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, d->stream));
  return SF_OK;
}

int sf_memcpy_p2p(int dst_dev, void* dst, int src_dev, const void* src, size_t bytes) {
  if (bytes == 0) return SF_OK;
  if (dst_dev == src_dev) return sf_memcpy_d2d(dst_dev, dst, src, bytes);
  Device *s, *d;
  SF_TRY(ensure_device(src_dev, &s));
  cudaEvent_t ev;
  SF_CHECK_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  SF_CHECK_CUDA(cudaEventRecord(ev, s->stream));
  SF_TRY(ensure_device(dst_dev, &d));
  SF_CHECK_CUDA(cudaStreamWaitEvent(d->stream, ev, 0));
  SF_CHECK_CUDA(cudaMemcpyPeerAsync(dst, dst_dev, src, src_dev, bytes, d->stream));
  // The source buffer may be freed (and reused) on the source stream right
  // after this call, so make the source stream wait for the transfer too.
  cudaEvent_t done;
  SF_CHECK_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  SF_CHECK_CUDA(cudaEventRecord(done, d->stream));
  SF_TRY(ensure_device(src_dev, &s));
  SF_CHECK_CUDA(cudaStreamWaitEvent(s->stream, done, 0));
  cudaEventDestroy(ev);
  cudaEventDestroy(done);
  return SF_OK;
}

int sf_rng_seed(int dev, uint64_t seed) {
  Device* d;
  SF_TRY(ensure_device_noflush(dev, &d));
  std::lock_guard<std::mutex> lk(d->rng_mu);
  d->rng_seed = seed;
  d->rng_offset = 0;
  return SF_OK;
}

int sf_rng_reserve(int dev, uint64_t n, uint64_t* offset) {
  Device* d;
  SF_TRY(ensure_device_noflush(dev, &d));
  std::lock_guard<std::mutex> lk(d->rng_mu);
  *offset = d->rng_offset;
  d->rng_offset += n;
  return SF_OK;
}

int sf_launch_count(int dev, uint64_t* count) {
  if (dev < 0 || dev >= 64) return SF_ERR_INVALID;
  *count = g_launches[dev].load();
  return SF_OK;
}

}  // extern "C"
