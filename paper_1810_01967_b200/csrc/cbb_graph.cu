// Device-decided IPG iteration as one CUDA graph (reference: coverblip/solver.py:116-144
// step_shrinkage and :155-257 _solve_core).
//
// The step rule of a trial -- project Z = X - mu G, nd = ||dX||^2, den = ||A dX||^2, accept iff
// mu <= nd / den (den == 0: accept; nd == 0: fixed point), else mu /= zeta (collapse after
// max_shrink shrinks) -- is decided on the device by trial_decide_kernel, which also drives the
// while-conditional node that repeats the trial body.  The host captures one iteration
// (gradient, the conditional trial loop, the apply of the accepted iterate and the residual) and
// replays it with a single synchronisation per iteration, where the host loop synchronised
// after every trial.  mu is kept in fp64 exactly as the host loop keeps it; the prologue reads
// its fp32 image (the same float(mu) the host loop passes).
#include "../../include/coverblip_b200.h"
#include "cbb_common.cuh"

#include <cmath>
#include <new>

namespace cbb {

struct TrialState {
  double mu;        // current trial step (fp64, solver.py:139)
  double mu_base;   // first trial's step of every iteration
  float mu32;       // float(mu): read by the projection prologue
  int shrinks;
  int fixed;        // nd == 0 in the last trial
  int status;       // 1: step-size collapse (shrinks > max_shrink)
  int trials;
};

__global__ void trial_init_kernel(TrialState* ts) {
  ts->mu = ts->mu_base;
  ts->mu32 = float(ts->mu_base);
  ts->shrinks = 0;
  ts->fixed = 0;
  ts->status = 0;
  ts->trials = 0;
}

__global__ void trial_decide_kernel(TrialState* ts, const double* nd, const double* den,
                                    double zeta, int max_shrink,
                                    cudaGraphConditionalHandle handle) {
  const double n_ = *nd, d_ = *den;
  ts->trials += 1;
  unsigned int again = 0;
  if (n_ == 0.0) {
    ts->fixed = 1;
  } else {
    const double ratio = d_ == 0.0 ? INFINITY : n_ / d_;
    if (!(ts->mu <= ratio)) {
      ts->mu /= zeta;
      ts->mu32 = float(ts->mu);
      ts->shrinks += 1;
      if (ts->shrinks > max_shrink) ts->status = 1;
      else again = 1;
    }
  }
  cudaGraphSetConditional(handle, again);
}

__global__ void trial_carry_kernel(TrialState* ts) { ts->mu_base = ts->mu; }

}  // namespace cbb

struct cbb_graph {
  cudaStream_t main = nullptr, body = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle cond = 0;
  bool in_body = false;
};

using cbb::kErrArgument;
using cbb::kErrCuda;
using cbb::kOk;

namespace {
cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
}  // namespace

extern "C" {

size_t cbb_trial_state_bytes(void) { return sizeof(cbb::TrialState); }

int cbb_graph_capture_begin(void* stream, cbb_graph** out) {
  if (!out || !stream) {
    cbb::set_last_error("cbb_graph_capture_begin: needs a (non-default) stream");
    return kErrArgument;
  }
  cbb_graph* g = new (std::nothrow) cbb_graph{};
  if (!g) return kErrArgument;
  g->main = S(stream);
  cudaError_t e = cudaStreamBeginCapture(g->main, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) {
    delete g;
    cbb::set_last_error(cudaGetErrorString(e));
    return kErrCuda;
  }
  *out = g;
  return kOk;
}

int cbb_graph_while_begin(cbb_graph* g, void* body_stream) {
  if (!g || g->in_body || !body_stream) return kErrArgument;
  cudaStreamCaptureStatus st;
  cudaGraph_t graph = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  CBB_CUDA_TRY(cudaStreamGetCaptureInfo(g->main, &st, nullptr, &graph, &deps, &ndeps));
  if (st != cudaStreamCaptureStatusActive) return kErrArgument;
  CBB_CUDA_TRY(cudaGraphConditionalHandleCreate(&g->cond, graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = g->cond;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  CBB_CUDA_TRY(cudaGraphAddNode(&node, graph, deps, ndeps, &p));
  CBB_CUDA_TRY(cudaStreamUpdateCaptureDependencies(g->main, &node, 1,
                                                   cudaStreamSetCaptureDependencies));
  g->body = S(body_stream);
  CBB_CUDA_TRY(cudaStreamBeginCaptureToGraph(g->body, p.conditional.phGraph_out[0], nullptr,
                                             nullptr, 0, cudaStreamCaptureModeThreadLocal));
  g->in_body = true;
  return kOk;
}

int cbb_trial_decide(cbb_graph* g, void* trial_state, const double* nd, const double* den,
                     double zeta, int32_t max_shrink) {
  if (!g || !g->in_body || !trial_state || !nd || !den) return kErrArgument;
  cbb::trial_decide_kernel<<<1, 1, 0, g->body>>>(static_cast<cbb::TrialState*>(trial_state), nd,
                                                 den, zeta, max_shrink, g->cond);
  CBB_CUDA_TRY(cudaGetLastError());
  cbb::count_launches(1);
  return kOk;
}

int cbb_graph_while_end(cbb_graph* g) {
  if (!g || !g->in_body) return kErrArgument;
  cudaGraph_t body = nullptr;
  CBB_CUDA_TRY(cudaStreamEndCapture(g->body, &body));
  g->in_body = false;
  return kOk;
}

int cbb_trial_init(void* trial_state, void* stream) {
  if (!trial_state) return kErrArgument;
  cbb::trial_init_kernel<<<1, 1, 0, S(stream)>>>(static_cast<cbb::TrialState*>(trial_state));
  CBB_CUDA_TRY(cudaGetLastError());
  cbb::count_launches(1);
  return kOk;
}

int cbb_trial_carry(void* trial_state, void* stream) {
  if (!trial_state) return kErrArgument;
  cbb::trial_carry_kernel<<<1, 1, 0, S(stream)>>>(static_cast<cbb::TrialState*>(trial_state));
  CBB_CUDA_TRY(cudaGetLastError());
  cbb::count_launches(1);
  return kOk;
}

int cbb_graph_capture_end(cbb_graph* g) {
  if (!g || g->in_body) return kErrArgument;
  CBB_CUDA_TRY(cudaStreamEndCapture(g->main, &g->graph));
  CBB_CUDA_TRY(cudaGraphInstantiate(&g->exec, g->graph, 0));
  return kOk;
}

int cbb_graph_launch(cbb_graph* g, void* stream) {
  if (!g || !g->exec) return kErrArgument;
  CBB_CUDA_TRY(cudaGraphLaunch(g->exec, S(stream)));
  return kOk;
}

int cbb_graph_destroy(cbb_graph* g) {
  if (!g) return kOk;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
  return kOk;
}

}  // extern "C"
