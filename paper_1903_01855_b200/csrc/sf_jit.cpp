// sf_jit.cpp — NVRTC compilation of the fused kernels generated for staged
// graph functions (see paper_1903_01855_b200/lowering.py).
//
// The generated source #includes "sf_ops.cuh" (embedded below as a string,
// byte-identical to the header the AOT kernels are built from) and is
// compiled for sm_100a with the same IEEE flags as the AOT kernels, so a
// fused chain reproduces the eager per-op results bit-for-bit.
#include <nvrtc.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <memory>

#include <atomic>

#include "sf_internal.h"
#include "sf_ops_embed.h"  // generated: const char* kSfOpsCuh

namespace sfrt {

struct JitKernel {
  std::string name;
  std::vector<char> cubin;
  std::mutex mu;
  std::mutex pool_mu;  // constant-pool fill + launch are one unit per module
  CUmodule module[64] = {};
  CUfunction fn[64] = {};
  std::atomic<unsigned> dyn_smem[64] = {};  // dynamic shared memory opted in per device
};

static std::mutex g_jit_mu;
static std::unordered_map<std::string, std::unique_ptr<JitKernel>> g_jit_cache;
static thread_local std::string t_jit_log;

// Persistent compile cache: cubins are stored on disk under
// $SF_JIT_CACHE (default ~/.cache/paper_1903_01855_b200/jit; "0" disables),
// keyed by a 64-bit FNV-1a hash of the kernel name, the generated source, the
// embedded sf_ops.cuh and the NVRTC version, and re-checked against the full
// key stored in the file, so a later process skips NVRTC for every graph it
// has lowered before.
static std::string cache_dir() {
  const char* env = getenv("SF_JIT_CACHE");
  if (env && std::string(env) == "0") return "";
  if (env && *env) return env;
  const char* home = getenv("HOME");
  return home ? std::string(home) + "/.cache/paper_1903_01855_b200/jit" : "";
}

static uint64_t fnv1a(const std::string& s, uint64_t h = 1469598103934665603ull) {
  for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
  return h;
}

// the IEEE flags of the AOT kernels (Makefile), so fused code matches eager bits
static const char* kNvrtcOpts[] = {"--gpu-architecture=sm_100a", "-fmad=false", "-prec-div=true",
                                   "-prec-sqrt=true", "-ftz=false", "-default-device",
                                   "-std=c++17", "-lineinfo", "-DSF_JIT=1"};

static std::string cache_key(const std::string& name, const std::string& src) {
  int major = 0, minor = 0;
  nvrtcVersion(&major, &minor);
  std::string opts;
  for (const char* o : kNvrtcOpts) opts += std::string(o) + ' ';
  return name + '\n' + std::to_string(major) + "." + std::to_string(minor) + '\n' + opts + '\n' +
         std::to_string(fnv1a(kSfOpsCuh)) + '\n' + src;
}

static std::string cache_path(const std::string& key) {
  const std::string dir = cache_dir();
  if (dir.empty()) return "";
  char buf[32];
  snprintf(buf, sizeof(buf), "%016llx", (unsigned long long)fnv1a(key));
  return dir + "/" + buf + ".cubin";
}

static bool cache_load(const std::string& key, std::vector<char>* cubin) {
  const std::string path = cache_path(key);
  if (path.empty()) return false;
  FILE* f = fopen(path.c_str(), "rb");
  if (!f) return false;
  uint64_t klen = 0, clen = 0;
  bool ok = fread(&klen, 8, 1, f) == 1 && klen == key.size();
  std::string stored(ok ? klen : 0, '\0');
  ok = ok && fread(&stored[0], 1, klen, f) == klen && stored == key &&
       fread(&clen, 8, 1, f) == 1 && clen > 0 && clen < (1ull << 30);
  if (ok) {
    cubin->resize(clen);
    ok = fread(cubin->data(), 1, clen, f) == clen;
  }
  fclose(f);
  return ok;
}

static void cache_store(const std::string& key, const std::vector<char>& cubin) {
  const std::string path = cache_path(key);
  if (path.empty()) return;
  std::string cmd_dir = cache_dir();
  // mkdir -p, one component at a time
  for (size_t i = 1; i <= cmd_dir.size(); ++i)
    if (i == cmd_dir.size() || cmd_dir[i] == '/') mkdir(cmd_dir.substr(0, i).c_str(), 0755);
  const std::string tmp = path + ".tmp" + std::to_string((unsigned long long)getpid());
  FILE* f = fopen(tmp.c_str(), "wb");
  if (!f) return;
  const uint64_t klen = key.size(), clen = cubin.size();
  bool ok = fwrite(&klen, 8, 1, f) == 1 && fwrite(key.data(), 1, klen, f) == klen &&
            fwrite(&clen, 8, 1, f) == 1 && fwrite(cubin.data(), 1, clen, f) == clen;
  ok = (fclose(f) == 0) && ok;
  if (ok) rename(tmp.c_str(), path.c_str());  // atomic publish
  else remove(tmp.c_str());
}

static int compile_nvrtc(const std::string& name, const std::string& src,
                         std::vector<char>* cubin);

static int compile(const std::string& name, const std::string& src, std::vector<char>* cubin) {
  const std::string key = cache_key(name, src);
  if (cache_load(key, cubin)) return SF_OK;
  SF_TRY(compile_nvrtc(name, src, cubin));
  cache_store(key, *cubin);
  return SF_OK;
}

static int compile_nvrtc(const std::string& name, const std::string& src,
                         std::vector<char>* cubin) {
  nvrtcProgram prog;
  const char* headers[] = {kSfOpsCuh};
  const char* header_names[] = {"sf_ops.cuh"};
  nvrtcResult r = nvrtcCreateProgram(&prog, src.c_str(), (name + ".cu").c_str(), 1, headers,
                                     header_names);
  if (r != NVRTC_SUCCESS) {
    set_error(std::string("nvrtcCreateProgram: ") + nvrtcGetErrorString(r));
    return SF_ERR_NVRTC;
  }
  r = nvrtcCompileProgram(prog, (int)(sizeof(kNvrtcOpts) / sizeof(kNvrtcOpts[0])), kNvrtcOpts);
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

int jit_global(void* kernel, int dev, const char* name, void** ptr, size_t* bytes) {
  JitKernel* k = (JitKernel*)kernel;
  CUfunction f;
  SF_TRY(jit_function(k, dev, &f));  // loads the module on this device
  CUdeviceptr p = 0;
  size_t n = 0;
  SF_CHECK_CU(drv.moduleGetGlobal(&p, &n, k->module[dev], name));
  *ptr = (void*)p;
  *bytes = n;
  return SF_OK;
}

std::mutex& jit_mutex(void* kernel) { return ((JitKernel*)kernel)->pool_mu; }

int jit_launch(Device* d, void* kernel, unsigned grid, unsigned block, unsigned smem,
               const void* params, size_t params_bytes) {
  CUfunction f;
  SF_TRY(jit_function((JitKernel*)kernel, d->id, &f));
  // any dynamic shared memory is opted in (static + dynamic may pass 48 KB)
  JitKernel* jk = (JitKernel*)kernel;
  if (smem > jk->dyn_smem[d->id].load(std::memory_order_relaxed)) {
    SF_CHECK_CU(drv.funcSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem));
    jk->dyn_smem[d->id].store(smem, std::memory_order_relaxed);
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
