// sf_jit.cpp — NVRTC compilation of the fused kernels generated for staged
// graph functions (see paper_1903_01855_b200/lowering.py).
//
// The generated source #includes "sf_ops.cuh" (embedded below as a string,
// byte-identical to the header the AOT kernels are built from) and is
// compiled for sm_100a with the same IEEE flags as the AOT kernels, so a
// fused chain reproduces the eager per-op results bit-for-bit.
#include <nvrtc.h>

#include <memory>

#include "sf_internal.h"
#include "sf_ops_embed.h"  // generated: const char* kSfOpsCuh

namespace sfrt {

struct JitKernel {
  std::string name;
  std::vector<char> cubin;
  std::mutex mu;
  CUmodule module[64] = {};
  CUfunction fn[64] = {};
};

static std::mutex g_jit_mu;
static std::unordered_map<std::string, std::unique_ptr<JitKernel>> g_jit_cache;
static thread_local std::string t_jit_log;

static int compile(const std::string& name, const std::string& src, std::vector<char>* cubin) {
  nvrtcProgram prog;
  const char* headers[] = {kSfOpsCuh};
  const char* header_names[] = {"sf_ops.cuh"};
  nvrtcResult r = nvrtcCreateProgram(&prog, src.c_str(), (name + ".cu").c_str(), 1, headers,
                                     header_names);
  if (r != NVRTC_SUCCESS) {
    set_error(std::string("nvrtcCreateProgram: ") + nvrtcGetErrorString(r));
    return SF_ERR_NVRTC;
  }
  const char* opts[] = {"--gpu-architecture=sm_100a", "-fmad=false",     "-prec-div=true",
                        "-prec-sqrt=true",            "-ftz=false",      "-default-device",
                        "-std=c++17",                 "-lineinfo",       "-DSF_JIT=1"};
  r = nvrtcCompileProgram(prog, (int)(sizeof(opts) / sizeof(opts[0])), opts);
  size_t log_size = 0;
  nvrtcGetProgramLogSize(prog, &log_size);
  t_jit_log.assign(log_size, '\0');
  if (log_size) nvrtcGetProgramLog(prog, &t_jit_log[0]);
  if (r != NVRTC_SUCCESS) {
    set_error(std::string("NVRTC compile of ") + name + " failed: " + nvrtcGetErrorString(r) +
              "\n" + t_jit_log);
    nvrtcDestroyProgram(&prog);
    return SF_ERR_NVRTC;
  }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  cubin->resize(n);
  nvrtcGetCUBIN(prog, cubin->data());
  nvrtcDestroyProgram(&prog);
  return SF_OK;
}

int jit_function(JitKernel* k, int dev, CUfunction* out) {
  if (dev < 0 || dev >= 64) return SF_ERR_INVALID;
  if (k->fn[dev]) {
    *out = k->fn[dev];
    return SF_OK;
  }
  std::lock_guard<std::mutex> lk(k->mu);
  if (!k->fn[dev]) {
    SF_CHECK_CU(drv.moduleLoadData(&k->module[dev], k->cubin.data()));
    SF_CHECK_CU(drv.moduleGetFunction(&k->fn[dev], k->module[dev], k->name.c_str()));
  }
  *out = k->fn[dev];
  return SF_OK;
}

int jit_launch(Device* d, void* kernel, unsigned grid, unsigned block, unsigned smem,
               const void* params, size_t params_bytes) {
  CUfunction f;
  SF_TRY(jit_function((JitKernel*)kernel, d->id, &f));
  if (smem > 48 * 1024) {
    SF_CHECK_CU(drv.funcSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem));
  }
  size_t sz = params_bytes;
  void* extra[] = {CU_LAUNCH_PARAM_BUFFER_POINTER, const_cast<void*>(params),
                   CU_LAUNCH_PARAM_BUFFER_SIZE, &sz, CU_LAUNCH_PARAM_END};
  SF_CHECK_CU(drv.launchKernel(f, grid, 1, 1, block, 1, 1, smem, (CUstream)d->stream, nullptr, extra));
  count_launch(d->id);
  return SF_OK;
}

}  // namespace sfrt

using namespace sfrt;

extern "C" {

int sf_jit_compile(const char* kernel_name, const char* source, void** kernel) {
  // Compile-only: no device needed (modules are loaded per device at first
  // launch), so generated code can be validated on a GPU-less build host.
  std::string key = std::string(kernel_name) + '\0' + source;
  {
    std::lock_guard<std::mutex> lk(g_jit_mu);
    auto it = g_jit_cache.find(key);
    if (it != g_jit_cache.end()) {
      *kernel = it->second.get();
      return SF_OK;
    }
  }
  auto k = std::make_unique<JitKernel>();
  k->name = kernel_name;
  SF_TRY(compile(kernel_name, source, &k->cubin));
  std::lock_guard<std::mutex> lk(g_jit_mu);
  auto& slot = g_jit_cache[key];
  if (!slot) slot = std::move(k);
  *kernel = slot.get();
  return SF_OK;
}

const char* sf_jit_log(void) { return t_jit_log.c_str(); }

int sf_jit_launch(int dev, void* kernel, unsigned grid, unsigned block, unsigned smem,
                  const void* params, size_t params_bytes) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  return jit_launch(d, kernel, grid, block, smem, params, params_bytes);
}

}  // extern "C"
