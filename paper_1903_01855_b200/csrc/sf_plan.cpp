// sf_plan.cpp — executor for lowered graph functions.
//
// Replaces execute_graph / _Plan / _run_pooled (reference:
// stageflow/executor.py:58-327).  The reference walks one Python
// instruction per node and keeps every intermediate alive until return
// (:209-213).  A plan here is the graph after lowering (fusion into jitted
// kernels, layout-folded matmuls, aliasing reshapes): a flat list of launch
// steps over value slots, executed by one C call per staged invocation.
// Temporaries are carved from the stream-ordered caching allocator at their
// defining step and returned right after their last use, so peak memory is
// the live set, not the whole graph.
//
// Binary plan format (little-endian; written by executor.py PlanWriter):
//   u32 magic 'SFPL' | u32 version(1) | i32 n_slots | i32 n_inputs |
//   i32 n_outputs | i32 n_steps
//   n_slots x slot:  u8 kind (0 input, 1 const, 2 temp, 3 output) | u8 dtype |
//                    u16 pad | i32 index (input/output ordinal) |
//                    u64 nbytes | u64 const_ptr | i32 def_step | i32 last_step
//   n_steps x step:  u32 kind | u32 payload_bytes | payload
//     kind 1 JIT       u64 kernel | u32 grid | u32 block | u32 smem | u32 n_ptr |
//                      i32 slot[n_ptr] | u32 n_scalar_bytes | bytes (8-aligned)
//                      [| u32 n_patches | {u32 kind, u32 offset, u64 count}[n]
//                      [| u32 pool_bytes | u32 n_pool |
//                         {i32 slot, u32 off, u32 n, u32 width, u32 N, u32 Np}[n]]]
//                      (pool: the kernel's __constant__ cpool is filled from
//                      the slots before every launch)
//     kind 2 MATMUL    i32 dtype | i32 ta | i32 tb | i32 a | i32 b | i32 c | i64 m | i64 n | i64 k
//     kind 3 REDUCE    i32 op | i32 dtype | i32 ndim | u32 axes | i32 in | i32 out | i64 shape[8]
//     kind 4 TRANSPOSE i32 dtype | i32 in | i32 out | i32 pad | i64 rows | i64 cols
//     kind 5 FILL      i32 dtype | i32 out | i64 n | f64 value
//     kind 6 EYE       i32 dtype | i32 out | i64 n
//     kind 7 COPY      i32 in | i32 out | i64 nbytes
//     kind 8 EW        i32 op | i32 dtype | i32 ndim | i32 n_in | i32 slot[3] (-1 = imm) |
//                      i32 out | f64 imm[3] | i64 shape[8] | i64 strides[3][8]
//     kind 9 RNG       i32 kind | i32 dtype | i32 out | i32 pad | i64 n
//     kind 10 DROPOUT  i32 dtype | i32 x | i32 out | i32 mask | i64 n | f64 rate
//     kind 11 CAST     i32 src | i32 dst | i32 in | i32 out | i64 n
//     kind 12 ALLREDUCE u64 comm | i32 dtype | i32 n | f64 scale | i32 slot[n]
//                      (in place, on the communicator's stream, forked after the
//                      steps so far; the plan joins it back after its last step)
#include "sf_internal.h"

namespace sfrt {

int jit_launch(Device* d, void* kernel, unsigned grid, unsigned block, unsigned smem,
               const void* params, size_t params_bytes);

struct Slot {
  uint8_t kind, dtype;
  int32_t index;
  uint64_t nbytes;
  void* const_ptr;
  int32_t def_step, last_step;
};

struct Step {
  uint32_t kind;
  std::vector<char> payload;
  // JIT decoded
  void* kernel = nullptr;
  unsigned grid = 1, block = 1, smem = 0;
  std::vector<int32_t> ptr_slots;
  std::vector<char> scalars;
  // run-time patches of the scalar blob: kind 0 = device RNG seed,
  // kind 1 = reserve `count` Philox counters and write the base offset
  struct Patch {
    uint32_t kind, offset;
    uint64_t count;
  };
  std::vector<Patch> patches;
  // constant pool of a row kernel: bytes, entries (src = slot index)
  uint32_t pool_bytes = 0;
  std::vector<CpoolEntry> pool;
  std::vector<int32_t> pool_slots;
  std::vector<int32_t> frees;  // temp slots to release after this step
  std::vector<int32_t> defs;   // temp/output slots to allocate before this step
};

struct Plan {
  int dev = 0;
  // optional per-step GPU timing (sf_plan_profile): CUDA events around each
  // step, read back after the run's stream synchronisation
  bool profile = false;
  std::vector<cudaEvent_t> ev;
  std::vector<double> step_ms;
  std::vector<uint64_t> step_runs;
  std::vector<Slot> slots;
  std::vector<Step> steps;
  std::vector<int32_t> input_slot;   // input ordinal -> slot
  std::vector<int32_t> output_slot;  // output ordinal -> slot
  int n_launches = 0;
  std::mutex mu;
};

class Reader {
 public:
  Reader(const char* p, size_t n) : p_(p), n_(n) {}
  template <class T>
  bool get(T* v) {
    if (off_ + sizeof(T) > n_) return false;
    std::memcpy(v, p_ + off_, sizeof(T));
    off_ += sizeof(T);
    return true;
  }
  bool bytes(size_t n, std::vector<char>* out) {
    if (off_ + n > n_) return false;
    out->assign(p_ + off_, p_ + off_ + n);
    off_ += n;
    return true;
  }

 private:
  const char* p_;
  size_t n_, off_ = 0;
};

template <class T>
static T at(const std::vector<char>& b, size_t off) {
  T v;
  std::memcpy(&v, b.data() + off, sizeof(T));
  return v;
}

static int bad(const char* what) {
  set_error(std::string("sf_plan_create: malformed plan (") + what + ")");
  return SF_ERR_INVALID;
}

static int run_step(Plan* p, Device* d, Step& s, std::vector<void*>& ptr,
                    std::vector<void*>* comms) {
  const auto& b = s.payload;
  auto P = [&](int32_t slot) -> void* { return slot < 0 ? nullptr : ptr[slot]; };
  switch (s.kind) {
    case 12: {
      void* comm = (void*)at<uint64_t>(b, 0);
      const int32_t dtype = at<int32_t>(b, 8), n = at<int32_t>(b, 12);
      const double scale = at<double>(b, 16);
      std::vector<void*> bufs(n);
      std::vector<size_t> counts(n);
      const size_t w = dtype_size(dtype);
      for (int i = 0; i < n; ++i) {
        const int32_t slot = at<int32_t>(b, 24 + 4 * i);
        bufs[i] = P(slot);
        counts[i] = p->slots[slot].nbytes / w;
      }
      SF_TRY(comm_allreduce(comm, d, bufs.data(), counts.data(), n, dtype, scale));
      for (void* c : *comms)
        if (c == comm) return SF_OK;
      comms->push_back(comm);
      return SF_OK;
    }
    case 1: {  // JIT
      std::vector<char> blob(s.ptr_slots.size() * 8 + s.scalars.size());
      for (size_t i = 0; i < s.ptr_slots.size(); ++i) {
        void* q = P(s.ptr_slots[i]);
        std::memcpy(blob.data() + i * 8, &q, 8);
      }
      if (!s.scalars.empty())
        std::memcpy(blob.data() + s.ptr_slots.size() * 8, s.scalars.data(), s.scalars.size());
      if (!s.patches.empty()) {
        std::lock_guard<std::mutex> lk(d->rng_mu);
        for (const auto& pt : s.patches) {
          uint64_t v = d->rng_seed;
          if (pt.kind == 1) {
            v = d->rng_offset;
            d->rng_offset += pt.count;
          }
          std::memcpy(blob.data() + s.ptr_slots.size() * 8 + pt.offset, &v, 8);
        }
      }
      if (!s.pool_bytes)
        return jit_launch(d, s.kernel, s.grid, s.block, s.smem, blob.data(), blob.size());
      // gather the uniform operands into an image, copy it into the
      // module's __constant__ pool, launch; one unit per module (stream order)
      void* cpool = nullptr;
      size_t cbytes = 0;
      SF_TRY(jit_global(s.kernel, d->id, "cpool", &cpool, &cbytes));
      if (cbytes < s.pool_bytes) {
        set_error("plan: constant pool smaller than its image");
        return SF_ERR_INVALID;
      }
      std::vector<CpoolEntry> ents(s.pool);
      for (size_t i = 0; i < ents.size(); ++i) ents[i].src = P(s.pool_slots[i]);
      std::lock_guard<std::mutex> lk(jit_mutex(s.kernel));
      void* image = nullptr;
      SF_TRY(d->alloc.alloc(d->id, s.pool_bytes, &image));
      int rc = launch_cpool_gather(d, ents.data(), (int)ents.size(), image);
      if (rc == SF_OK) {
        cudaError_t e = cudaMemcpyAsync(cpool, image, s.pool_bytes, cudaMemcpyDeviceToDevice,
                                        d->stream);
        if (e != cudaSuccess) {
          set_error(std::string("plan: constant pool copy: ") + cudaGetErrorString(e));
          rc = SF_ERR_CUDA;
        }
      }
      d->alloc.release(image);  // stream-ordered reuse
      if (rc != SF_OK) return rc;
      return jit_launch(d, s.kernel, s.grid, s.block, s.smem, blob.data(), blob.size());
    }
    case 2:
      return launch_matmul(d, at<int32_t>(b, 0), at<int64_t>(b, 24), at<int64_t>(b, 32),
                           at<int64_t>(b, 40), P(at<int32_t>(b, 12)), at<int32_t>(b, 4),
                           P(at<int32_t>(b, 16)), at<int32_t>(b, 8), P(at<int32_t>(b, 20)));
    case 3: {
      int64_t shape[SF_MAX_DIMS];
      std::memcpy(shape, b.data() + 24, sizeof(shape));
      return launch_reduce(d, at<int32_t>(b, 0), at<int32_t>(b, 4), at<int32_t>(b, 8), shape,
                           at<uint32_t>(b, 12), P(at<int32_t>(b, 16)), P(at<int32_t>(b, 20)));
    }
    case 4:
      return launch_transpose2d(d, at<int32_t>(b, 0), at<int64_t>(b, 16), at<int64_t>(b, 24),
                                P(at<int32_t>(b, 4)), P(at<int32_t>(b, 8)));
    case 5:
      return launch_fill(d, at<int32_t>(b, 0), at<int64_t>(b, 8), at<double>(b, 16),
                         P(at<int32_t>(b, 4)));
    case 6:
      return launch_eye(d, at<int32_t>(b, 0), at<int64_t>(b, 8), P(at<int32_t>(b, 4)));
    case 7: {
      const int64_t n = at<int64_t>(b, 8);
      if (n == 0) return SF_OK;
      SF_CHECK_CUDA(cudaMemcpyAsync(P(at<int32_t>(b, 4)), P(at<int32_t>(b, 0)), (size_t)n,
                                    cudaMemcpyDeviceToDevice, d->stream));
      return SF_OK;
    }
    case 8: {
      const int32_t op = at<int32_t>(b, 0), dtype = at<int32_t>(b, 4), ndim = at<int32_t>(b, 8),
                    n_in = at<int32_t>(b, 12);
      const void* ins[3];
      for (int j = 0; j < 3; ++j) ins[j] = P(at<int32_t>(b, 16 + 4 * j));
      void* out = P(at<int32_t>(b, 28));
      double imm[3];
      std::memcpy(imm, b.data() + 32, sizeof(imm));
      int64_t shape[SF_MAX_DIMS];
      std::memcpy(shape, b.data() + 56, sizeof(shape));
      int64_t strides[3][SF_MAX_DIMS];
      std::memcpy(strides, b.data() + 56 + 64, sizeof(strides));
      const int64_t* sp[3] = {strides[0], strides[1], strides[2]};
      return launch_elementwise(d, op, dtype, ndim, shape, out, ins, sp, imm, n_in);
    }
    case 9: {
      const int64_t n = at<int64_t>(b, 16);
      unsigned long long off;
      {
        std::lock_guard<std::mutex> lk(d->rng_mu);
        off = d->rng_offset;
        d->rng_offset += (unsigned long long)n;
      }
      return launch_rng(d, at<int32_t>(b, 0), at<int32_t>(b, 4), n, d->rng_seed, off,
                        P(at<int32_t>(b, 8)));
    }
    case 10:
      return launch_dropout(d, at<int32_t>(b, 0), at<int64_t>(b, 16), P(at<int32_t>(b, 4)),
                            nullptr, SF_DTYPE_F64, at<double>(b, 24), P(at<int32_t>(b, 8)),
                            P(at<int32_t>(b, 12)));
    case 11:
      return launch_cast(d, at<int32_t>(b, 0), at<int32_t>(b, 4), at<int64_t>(b, 16),
                         P(at<int32_t>(b, 8)), P(at<int32_t>(b, 12)));
    default:
      set_error("plan: unknown step kind");
      return SF_ERR_INVALID;
  }
}

}  // namespace sfrt

using namespace sfrt;

extern "C" {

int sf_plan_create(int dev, const void* desc, size_t desc_bytes, void** out) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  Reader r((const char*)desc, desc_bytes);
  uint32_t magic, version;
  int32_t n_slots, n_inputs, n_outputs, n_steps;
  if (!r.get(&magic) || magic != 0x4C504653u) return bad("magic");
  if (!r.get(&version) || version != 1) return bad("version");
  if (!r.get(&n_slots) || !r.get(&n_inputs) || !r.get(&n_outputs) || !r.get(&n_steps))
    return bad("header");
  auto p = std::make_unique<Plan>();
  p->dev = dev;
  p->input_slot.assign(n_inputs, -1);
  p->output_slot.assign(n_outputs, -1);
  p->slots.resize(n_slots);
  for (int i = 0; i < n_slots; ++i) {
    Slot& s = p->slots[i];
    uint16_t pad;
    uint64_t cptr;
    if (!r.get(&s.kind) || !r.get(&s.dtype) || !r.get(&pad) || !r.get(&s.index) ||
        !r.get(&s.nbytes) || !r.get(&cptr) || !r.get(&s.def_step) || !r.get(&s.last_step))
      return bad("slot");
    s.const_ptr = (void*)cptr;
    if (s.kind == 0) {
      if (s.index < 0 || s.index >= n_inputs) return bad("input index");
      p->input_slot[s.index] = i;
    } else if (s.kind == 3) {
      if (s.index < 0 || s.index >= n_outputs) return bad("output index");
      p->output_slot[s.index] = i;
    }
  }
  p->steps.resize(n_steps);
  for (int i = 0; i < n_steps; ++i) {
    Step& s = p->steps[i];
    uint32_t len;
    if (!r.get(&s.kind) || !r.get(&len) || !r.bytes(len, &s.payload)) return bad("step");
    if (s.kind == 1) {
      const auto& b = s.payload;
      if (b.size() < 28) return bad("jit step");
      s.kernel = (void*)at<uint64_t>(b, 0);
      s.grid = at<uint32_t>(b, 8);
      s.block = at<uint32_t>(b, 12);
      s.smem = at<uint32_t>(b, 16);
      const uint32_t n_ptr = at<uint32_t>(b, 20);
      size_t off = 24;
      for (uint32_t k = 0; k < n_ptr; ++k, off += 4) s.ptr_slots.push_back(at<int32_t>(b, off));
      const uint32_t ns = at<uint32_t>(b, off);
      off += 4;
      if (off + ns > b.size()) return bad("jit scalars");
      s.scalars.assign(b.begin() + off, b.begin() + off + ns);
      off += ns;
      if (off + 4 <= b.size()) {
        const uint32_t np = at<uint32_t>(b, off);
        off += 4;
        for (uint32_t k = 0; k < np; ++k, off += 16) {
          if (off + 16 > b.size()) return bad("jit patches");
          Step::Patch pt{at<uint32_t>(b, off), at<uint32_t>(b, off + 4), at<uint64_t>(b, off + 8)};
          if (pt.offset + 8 > ns) return bad("jit patch offset");
          s.patches.push_back(pt);
        }
      }
      if (off + 8 <= b.size()) {  // constant pool section
        s.pool_bytes = at<uint32_t>(b, off);
        const uint32_t ne = at<uint32_t>(b, off + 4);
        off += 8;
        for (uint32_t k = 0; k < ne; ++k, off += 24) {
          if (off + 24 > b.size()) return bad("jit pool");
          CpoolEntry e{};
          s.pool_slots.push_back(at<int32_t>(b, off));
          e.dst_off = at<uint32_t>(b, off + 4);
          e.n = at<uint32_t>(b, off + 8);
          e.width = at<uint32_t>(b, off + 12);
          e.N = at<uint32_t>(b, off + 16);
          e.Np = at<uint32_t>(b, off + 20);
          if (e.N == 0 || e.Np < e.N || (uint64_t)e.dst_off + (uint64_t)e.Np * e.width *
              ((e.n + e.N - 1) / e.N) > s.pool_bytes)
            return bad("jit pool entry");
          s.pool.push_back(e);
        }
      }
    }
    if (s.kind != 7) ++p->n_launches;
    if (s.kind == 1 && s.pool_bytes) p->n_launches += (int)((s.pool.size() + 959) / 960);
  }
  for (int i = 0; i < n_slots; ++i) {
    const Slot& s = p->slots[i];
    if (s.kind == 2 || s.kind == 3) {
      if (s.def_step < 0 || s.def_step >= n_steps) return bad("def step");
      p->steps[s.def_step].defs.push_back(i);
      if (s.kind == 2) {
        const int last = s.last_step < s.def_step ? s.def_step : s.last_step;
        if (last >= n_steps) return bad("last step");
        p->steps[last].frees.push_back(i);
      }
    }
  }
  for (int k = 0; k < n_inputs; ++k)
    if (p->input_slot[k] < 0) return bad("missing input slot");
  for (int k = 0; k < n_outputs; ++k)
    if (p->output_slot[k] < 0) return bad("missing output slot");
  *out = p.release();
  return SF_OK;
}

int sf_plan_run(void* plan, const void* const* inputs, void** outputs) {
  Plan* p = (Plan*)plan;
  Device* d;
  SF_TRY(ensure_device(p->dev, &d));
  std::vector<void*> ptr(p->slots.size(), nullptr);
  for (size_t i = 0; i < p->slots.size(); ++i) {
    const Slot& s = p->slots[i];
    if (s.kind == 0) ptr[i] = const_cast<void*>(inputs[s.index]);
    else if (s.kind == 1) ptr[i] = s.const_ptr;
  }
  int st = SF_OK;
  size_t k = 0;
  std::vector<void*> comms;  // communicators with an all-reduce in flight
  for (; k < p->steps.size(); ++k) {
    Step& s = p->steps[k];
    for (int32_t slot : s.defs) {
      st = d->alloc.alloc(d->id, p->slots[slot].nbytes, &ptr[slot]);
      if (st != SF_OK) break;
    }
    if (st != SF_OK) break;
    if (p->profile) cudaEventRecord(p->ev[2 * k], d->stream);
    st = run_step(p, d, s, ptr, &comms);
    if (st != SF_OK) break;
    if (p->profile) cudaEventRecord(p->ev[2 * k + 1], d->stream);
    for (int32_t slot : s.frees) {
      d->alloc.release(ptr[slot]);
      ptr[slot] = nullptr;
    }
  }
  for (void* c : comms) {  // the outputs are complete only after the collectives
    const int js = comm_join(c, d);
    if (st == SF_OK) st = js;
  }
  if (st != SF_OK) {
    // release everything this run allocated
    for (size_t i = 0; i < p->slots.size(); ++i) {
      const Slot& s = p->slots[i];
      if ((s.kind == 2 || s.kind == 3) && ptr[i]) d->alloc.release(ptr[i]);
    }
    const std::string msg = last_error();
    set_error("plan step " + std::to_string(k) + ": " + msg);
    return st;
  }
  for (size_t o = 0; o < p->output_slot.size(); ++o) outputs[o] = ptr[p->output_slot[o]];
  if (p->profile) {
    SF_CHECK_CUDA(cudaStreamSynchronize(d->stream));
    for (size_t j = 0; j < p->steps.size(); ++j) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, p->ev[2 * j], p->ev[2 * j + 1]) == cudaSuccess) {
        p->step_ms[j] += ms;
        p->step_runs[j] += 1;
      }
    }
  }
  return SF_OK;
}

int sf_plan_profile(void* plan, int enable) {
  Plan* p = (Plan*)plan;
  Device* d;
  SF_TRY(ensure_device(p->dev, &d));
  if (enable && p->ev.empty()) {
    p->ev.resize(2 * p->steps.size());
    for (auto& e : p->ev) SF_CHECK_CUDA(cudaEventCreate(&e));
  }
  p->step_ms.assign(p->steps.size(), 0.0);
  p->step_runs.assign(p->steps.size(), 0);
  p->profile = enable != 0;
  return SF_OK;
}

int sf_plan_step_stats(void* plan, int step, int* kind, double* total_ms, uint64_t* runs) {
  Plan* p = (Plan*)plan;
  if (step < 0 || step >= (int)p->steps.size()) return SF_ERR_INVALID;
  if (kind) *kind = (int)p->steps[step].kind;
  if (total_ms) *total_ms = p->step_ms.empty() ? 0.0 : p->step_ms[step];
  if (runs) *runs = p->step_runs.empty() ? 0 : p->step_runs[step];
  return SF_OK;
}

int sf_plan_info(void* plan, int* n_inputs, int* n_outputs, int* n_steps, int* n_launches) {
  Plan* p = (Plan*)plan;
  if (n_inputs) *n_inputs = (int)p->input_slot.size();
  if (n_outputs) *n_outputs = (int)p->output_slot.size();
  if (n_steps) *n_steps = (int)p->steps.size();
  if (n_launches) *n_launches = p->n_launches;
  return SF_OK;
}

int sf_plan_destroy(void* plan) {
  delete (Plan*)plan;
  return SF_OK;
}

}  // extern "C"
