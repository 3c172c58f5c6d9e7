// sf_graph.cu — device-side while_loop: a CUDA graph with a WHILE
// conditional node.
//
// Replaces the host loop of the reference's while kernel
// (stageflow/kernels.py:513-538: evaluate cond_gf, read the predicate on the
// host, run body_gf, repeat).  On a GPU that host read is one stream
// synchronisation per iteration.  Here the loop runs inside one CUDA graph:
//
//   graph:  [cond plan -> set_cond]  ->  WHILE(handle) { body plan ->
//            copy new state into the loop-state buffers -> cond plan ->
//            set_cond }
//
// The cond and body plans (sf_plan.cpp) are recorded by stream capture, so
// the graph runs exactly the kernels eager/staged execution runs (same
// bits).  The predicate is consumed on the device by set_cond_kernel, which
// sets the conditional handle; the host never waits inside the loop.
//
// The same object implements cond (stageflow/kernels.py:493-510, which reads
// the predicate on the host): [set_cond(pred)] -> IF(handle) { then plan ->
// copy to the output buffers } ELSE { else plan -> copy }.
//
// Addresses baked into the graph stay valid because the allocator is in
// capture mode while the plans are recorded (Allocator::begin_capture): the
// graph owns every block it was given until sf_while_destroy.
#include "sf_internal.h"

namespace sfrt {

__global__ void set_cond_kernel(cudaGraphConditionalHandle h, const unsigned char* pred) {
  cudaGraphSetConditional(h, pred[0] ? 1u : 0u);
}

// One graph object serves both control-flow ops and whole-program replay:
//   while (is_if = false): parts 0 = prologue, 1 = loop body
//   cond  (is_if = true) : parts 0 = prologue (set_cond from the predicate),
//                          1 = then branch, 2 = else branch (IF node, size 2)
//   plain (plain = true) : part 0 only — a staged program recorded once and
//                          replayed with one cudaGraphLaunch per call
struct WhileGraph {
  Device* d = nullptr;
  bool is_if = false;
  bool plain = false;
  bool captured = false;
  cudaGraph_t graph = nullptr;
  cudaGraph_t body[2] = {nullptr, nullptr};
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle handle{};
  std::vector<std::pair<void*, size_t>> owned;  // blocks baked into the graph
  std::vector<void*> fixed;                      // loop-state / capture buffers
  int capturing = -1;
};

static int check_part(WhileGraph* w, int part) {
  const int last = w->plain ? 0 : w->is_if ? 2 : 1;
  if (part < 0 || part > last) {
    set_error("sf_while: part must be 0 (prologue) or a body index");
    return SF_ERR_INVALID;
  }
  if (part >= 1 && !w->body[0]) {
    set_error("sf_while: the prologue must be captured before the bodies");
    return SF_ERR_INVALID;
  }
  return SF_OK;
}

static int create_graph(int dev, bool is_if, bool plain, void** out) {
  Device* d;
  SF_TRY(ensure_device(dev, &d));
  auto* w = new WhileGraph();
  w->d = d;
  w->is_if = is_if;
  w->plain = plain;
  cudaError_t e = cudaGraphCreate(&w->graph, 0);
  // (a plain graph must not own a conditional handle: an unused handle makes
  // cudaGraphInstantiate fail with "invalid argument")
  if (e == cudaSuccess && !plain)
    e = cudaGraphConditionalHandleCreate(&w->handle, w->graph, 0, cudaGraphCondAssignDefault);
  if (e != cudaSuccess) {
    if (w->graph) cudaGraphDestroy(w->graph);
    delete w;
    set_error(std::string("sf_graph create: ") + cudaGetErrorString(e));
    return SF_ERR_CUDA;
  }
  *out = w;
  return SF_OK;
}

}  // namespace sfrt

using namespace sfrt;

extern "C" {

int sf_while_create(int dev, void** out) { return create_graph(dev, false, false, out); }

int sf_graph_create(int dev, void** out) { return create_graph(dev, false, true, out); }

int sf_cond_create(int dev, void** out) { return create_graph(dev, true, false, out); }

int sf_while_buffer(void* wp, size_t bytes, void** p) {
  auto* w = (WhileGraph*)wp;
  SF_TRY(w->d->alloc.alloc(w->d->id, bytes, p));
  w->fixed.push_back(*p);
  return SF_OK;
}

int sf_while_capture_begin(void* wp, int part) {
  auto* w = (WhileGraph*)wp;
  SF_TRY(check_part(w, part));
  if (w->capturing >= 0 || w->exec) {
    set_error("sf_while_capture_begin: capture already open or graph already built");
    return SF_ERR_INVALID;
  }
  SF_TRY(queue_flush(w->d));  // queued eager ops precede the capture
  w->d->alloc.begin_capture();
  cudaError_t e = cudaStreamBeginCaptureToGraph(w->d->stream,
                                                part ? w->body[part - 1] : w->graph, nullptr,
                                                nullptr, 0, cudaStreamCaptureModeRelaxed);
  if (e != cudaSuccess) {
    w->d->alloc.end_capture(&w->owned);
    set_error(std::string("sf_while_capture_begin: ") + cudaGetErrorString(e));
    return SF_ERR_CUDA;
  }
  w->capturing = part;
  return SF_OK;
}

int sf_while_set_cond(void* wp, const void* pred) {
  auto* w = (WhileGraph*)wp;
  if (w->capturing < 0) {
    set_error("sf_while_set_cond: only valid inside a capture");
    return SF_ERR_INVALID;
  }
  set_cond_kernel<<<1, 1, 0, w->d->stream>>>(w->handle, (const unsigned char*)pred);
  SF_CHECK_CUDA(cudaGetLastError());
  return SF_OK;
}

int sf_while_capture_end(void* wp, int part) {
  auto* w = (WhileGraph*)wp;
  if (w->capturing != part) {
    set_error("sf_while_capture_end: no capture of this part is open");
    return SF_ERR_INVALID;
  }
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(w->d->stream, &g);
  w->d->alloc.end_capture(&w->owned);
  w->capturing = -1;
  if (e != cudaSuccess) {
    set_error(std::string("sf_while_capture_end: ") + cudaGetErrorString(e));
    return SF_ERR_CUDA;
  }
  w->captured = true;
  if (part == 0 && !w->plain) {
    // append the WHILE node after every leaf of the prologue
    size_t n = 0;
    SF_CHECK_CUDA(cudaGraphGetNodes(w->graph, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n), leaves;
    if (n) SF_CHECK_CUDA(cudaGraphGetNodes(w->graph, nodes.data(), &n));
    for (auto nd : nodes) {
      size_t k = 0;
      SF_CHECK_CUDA(cudaGraphNodeGetDependentNodes(nd, nullptr, &k));
      if (k == 0) leaves.push_back(nd);
    }
    cudaGraphNodeParams params = {};
    params.type = cudaGraphNodeTypeConditional;
    params.conditional.handle = w->handle;
    // IF with size 2: body 0 runs when the handle is non-zero, body 1 (else) otherwise
    params.conditional.type = w->is_if ? cudaGraphCondTypeIf : cudaGraphCondTypeWhile;
    params.conditional.size = w->is_if ? 2 : 1;
    cudaGraphNode_t node;
    SF_CHECK_CUDA(cudaGraphAddNode(&node, w->graph, leaves.data(), leaves.size(), &params));
    w->body[0] = params.conditional.phGraph_out[0];
    if (w->is_if) w->body[1] = params.conditional.phGraph_out[1];
  }
  return SF_OK;
}

int sf_while_launch(void* wp) {
  auto* w = (WhileGraph*)wp;
  if ((w->plain ? !w->captured : !w->body[0]) || w->capturing >= 0) {
    set_error("sf_while_launch: graph not captured");
    return SF_ERR_INVALID;
  }
  if (!w->exec) {
    cudaError_t e = cudaGraphInstantiate(&w->exec, w->graph, 0);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      if (const char* dot = getenv("SF_GRAPH_DOT"))  // debugging aid: dump the graph
        cudaGraphDebugDotPrint(w->graph, dot, cudaGraphDebugDotFlagsVerbose);
      w->exec = nullptr;
      set_error(std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
      return SF_ERR_CUDA;
    }
  }
  SF_TRY(queue_flush(w->d));
  SF_CHECK_CUDA(cudaGraphLaunch(w->exec, w->d->stream));
  count_launch(w->d->id);
  return SF_OK;
}

int sf_while_destroy(void* wp) {
  auto* w = (WhileGraph*)wp;
  if (!w) return SF_OK;
  // the graph may still be executing: wait before its blocks are reused
  queue_flush(w->d);
  cudaStreamSynchronize(w->d->stream);
  if (w->exec) cudaGraphExecDestroy(w->exec);
  if (w->graph) cudaGraphDestroy(w->graph);
  w->d->alloc.give_back(w->owned);
  for (void* p : w->fixed) w->d->alloc.release(p);
  delete w;
  return SF_OK;
}

}  // extern "C"
