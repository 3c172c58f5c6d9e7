// sf_comm.cpp — NCCL behind the C-ABI (the one exchange step of the build:
// the ResNet-50 data-parallel gradient all-reduce).
//
// libnccl.so.2 is opened at first use (the library itself loads on hosts
// without NCCL or a GPU).  A communicator owns a dedicated comm stream.  An
// all-reduce is forked from the device's compute stream (event record +
// wait), runs grouped and in place on the comm stream, and is joined back
// only when the compute stream next needs the buffers: a plan (sf_plan.cpp
// step kind 12) issues each gradient bucket right after the step that
// produced its last gradient and joins once at the end of the plan, so the
// transfers overlap the rest of the backward.  Inside a CUDA-graph capture
// the fork/join pair pulls the comm stream into the capture (NCCL >= 2.9
// captures collectives).
#include <dlfcn.h>
#include <nccl.h>

#include <map>

#include "sf_internal.h"

namespace sfrt {

struct NcclApi {
  bool loaded = false;
  std::string error;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*redOpCreatePreMulSum)(ncclRedOp_t*, void*, ncclDataType_t,
                                       ncclScalarResidence_t, ncclComm_t) = nullptr;
  ncclResult_t (*redOpDestroy)(ncclRedOp_t, ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*getVersion)(int*) = nullptr;
};

static NcclApi g_nccl;
static std::mutex g_nccl_mu;

template <class F>
static bool sym(void* h, const char* name, F* out) {
  *out = (F)dlsym(h, name);
  return *out != nullptr;
}

static int load_nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.loaded) return SF_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (!h) {
    set_error(std::string("NCCL unavailable: ") + dlerror());
    return SF_ERR_UNSUPPORTED;
  }
  bool ok = sym(h, "ncclGetUniqueId", &g_nccl.getUniqueId) &&
            sym(h, "ncclCommInitRank", &g_nccl.commInitRank) &&
            sym(h, "ncclCommDestroy", &g_nccl.commDestroy) &&
            sym(h, "ncclAllReduce", &g_nccl.allReduce) &&
            sym(h, "ncclGroupStart", &g_nccl.groupStart) &&
            sym(h, "ncclGroupEnd", &g_nccl.groupEnd) &&
            sym(h, "ncclRedOpCreatePreMulSum", &g_nccl.redOpCreatePreMulSum) &&
            sym(h, "ncclRedOpDestroy", &g_nccl.redOpDestroy) &&
            sym(h, "ncclGetErrorString", &g_nccl.getErrorString) &&
            sym(h, "ncclGetVersion", &g_nccl.getVersion);
  if (!ok) {
    set_error("NCCL: libnccl.so.2 lacks a required entry point");
    return SF_ERR_UNSUPPORTED;
  }
  g_nccl.loaded = true;
  return SF_OK;
}

#define SF_CHECK_NCCL(expr)                                                          \
  do {                                                                               \
    ncclResult_t _r = (expr);                                                        \
    if (_r != ncclSuccess) {                                                         \
      ::sfrt::set_error(std::string(#expr) + ": " + g_nccl.getErrorString(_r));     \
      return SF_ERR_CUDA;                                                            \
    }                                                                                \
  } while (0)

struct Comm {
  ncclComm_t comm = nullptr;
  int dev = 0, nranks = 1, rank = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  std::map<std::pair<int, double>, ncclRedOp_t> premul;  // (dtype, scale) -> op
};

static bool nccl_dtype(int dtype, ncclDataType_t* out) {
  switch (dtype) {
    case SF_DTYPE_F32: *out = ncclFloat32; return true;
    case SF_DTYPE_F64: *out = ncclFloat64; return true;
    case SF_DTYPE_I32: *out = ncclInt32; return true;
    default: return false;
  }
}

// Enqueue one grouped in-place all-reduce of n buffers after the work on
// the device stream so far; the buffers are complete once comm_join has
// made the device stream wait.  scale != 1: sum of scale * x (premul sum).
int comm_allreduce(void* handle, Device* d, void* const* bufs, const size_t* counts, int n,
                   int dtype, double scale) {
  Comm* c = (Comm*)handle;
  if (!c || c->dev != d->id) {
    set_error("allreduce: communicator of another device");
    return SF_ERR_INVALID;
  }
  ncclDataType_t dt;
  if (!nccl_dtype(dtype, &dt)) {
    set_error("allreduce: unsupported dtype");
    return SF_ERR_INVALID;
  }
  ncclRedOp_t op = ncclSum;
  if (scale != 1.0) {
    auto key = std::make_pair(dtype, scale);
    auto it = c->premul.find(key);
    if (it == c->premul.end()) {
      ncclRedOp_t nop;
      if (dtype == SF_DTYPE_F64) {
        double s = scale;
        SF_CHECK_NCCL(g_nccl.redOpCreatePreMulSum(&nop, &s, dt, ncclScalarHostImmediate, c->comm));
      } else if (dtype == SF_DTYPE_F32) {
        float s = (float)scale;
        SF_CHECK_NCCL(g_nccl.redOpCreatePreMulSum(&nop, &s, dt, ncclScalarHostImmediate, c->comm));
      } else {
        set_error("allreduce: a scaled reduction needs a float dtype");
        return SF_ERR_INVALID;
      }
      it = c->premul.emplace(key, nop).first;
    }
    op = it->second;
  }
  SF_CHECK_CUDA(cudaEventRecord(c->fork, d->stream));
  SF_CHECK_CUDA(cudaStreamWaitEvent(c->stream, c->fork, 0));
  SF_CHECK_NCCL(g_nccl.groupStart());
  for (int i = 0; i < n; ++i) {
    ncclResult_t r = g_nccl.allReduce(bufs[i], bufs[i], counts[i], dt, op, c->comm, c->stream);
    if (r != ncclSuccess) {
      g_nccl.groupEnd();
      set_error(std::string("ncclAllReduce: ") + g_nccl.getErrorString(r));
      return SF_ERR_CUDA;
    }
  }
  SF_CHECK_NCCL(g_nccl.groupEnd());
  SF_CHECK_CUDA(cudaEventRecord(c->join, c->stream));
  return SF_OK;
}

int comm_join(void* handle, Device* d) {
  Comm* c = (Comm*)handle;
  SF_CHECK_CUDA(cudaStreamWaitEvent(d->stream, c->join, 0));
  return SF_OK;
}

int comm_device(void* handle) { return handle ? ((Comm*)handle)->dev : -1; }

}  // namespace sfrt

using namespace sfrt;

extern "C" {

int sf_comm_unique_id(void* id_out) {
  SF_TRY(load_nccl());
  ncclUniqueId id;
  SF_CHECK_NCCL(g_nccl.getUniqueId(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return SF_OK;
}

int sf_comm_init(int dev, int nranks, int rank, const void* id_in, void** comm) {
  SF_TRY(load_nccl());
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  if (nranks < 1 || rank < 0 || rank >= nranks) {
    set_error("sf_comm_init: bad rank / world size");
    return SF_ERR_INVALID;
  }
  auto c = std::make_unique<Comm>();
  c->dev = dev;
  c->nranks = nranks;
  c->rank = rank;
  ncclUniqueId id;
  std::memcpy(&id, id_in, sizeof(id));
  SF_CHECK_NCCL(g_nccl.commInitRank(&c->comm, nranks, id, rank));
  SF_CHECK_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  SF_CHECK_CUDA(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming));
  SF_CHECK_CUDA(cudaEventCreateWithFlags(&c->join, cudaEventDisableTiming));
  *comm = c.release();
  return SF_OK;
}

int sf_comm_destroy(void* comm) {
  Comm* c = (Comm*)comm;
  if (!c) return SF_OK;
  cudaSetDevice(c->dev);
  cudaStreamSynchronize(c->stream);
  for (auto& kv : c->premul) g_nccl.redOpDestroy(kv.second, c->comm);
  if (c->comm) g_nccl.commDestroy(c->comm);
  if (c->fork) cudaEventDestroy(c->fork);
  if (c->join) cudaEventDestroy(c->join);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return SF_OK;
}

int sf_allreduce(void* comm, void* const* bufs, const size_t* counts, int n, int dtype,
                 double scale) {
  Comm* c = (Comm*)comm;
  if (!c) {
    set_error("sf_allreduce: null communicator");
    return SF_ERR_INVALID;
  }
  Device* d;
  SF_TRY(ensure_device(c->dev, &d));  // (flushes the eager launch queue)
  SF_TRY(comm_allreduce(comm, d, bufs, counts, n, dtype, scale));
  return comm_join(comm, d);
}

int sf_nccl_version(int* version) {
  SF_TRY(load_nccl());
  SF_CHECK_NCCL(g_nccl.getVersion(version));
  return SF_OK;
}

}  // extern "C"
