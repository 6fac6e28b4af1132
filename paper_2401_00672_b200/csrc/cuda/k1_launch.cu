// K1: one launch per schedule step, one thread per row, x~ in global memory (L2-resident).
//
// A sweep (Alg 5 loop body) is the sequence of its steps; a step is one
// category of pairwise-orthogonal rows, whose block projection Eq 1.3
// collapses by Lemma 1 to independent Eq 1.2 row projections
// (PAPER.md:29): one thread per row (common.cuh contract), no atomics (disjoint supports), the
// launch boundary is the step barrier.  Steps whose rows overlap (thr > 0 only) run as two
// launches: all alphas at the same x~, then an fp64-atomic scatter.
//
// The sweep loop is device-driven: the steps + the stop check are the body of a CUDA-graph WHILE
// node whose condition the check kernel clears (no host round trip per sweep).  K1 is the
// general fallback (any size, any thr); K2/K3 are the fast paths.
#include "../plan.h"
#include "common.cuh"

namespace pobk {

namespace {
constexpr int kNT = 128;

__global__ void __launch_bounds__(kNT) k1_step(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                               const double* __restrict__ val, const double* __restrict__ fs,
                                               const double* __restrict__ nrm2, double* __restrict__ x, int s0, int s1) {
  const int s = s0 + blockIdx.x * kNT + threadIdx.x;
  if (s >= s1) return;
  row_project(col, val, rp[s], rp[s + 1], fs[s], nrm2[s], x);
}

// thr > 0, overlapping step: pass 1 -- every alpha at the same x~
__global__ void __launch_bounds__(kNT) k1_alpha(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                const double* __restrict__ val, const double* __restrict__ fs,
                                                const double* __restrict__ nrm2, const double* __restrict__ x,
                                                double* __restrict__ alpha, int s0, int s1) {
  const int s = s0 + blockIdx.x * kNT + threadIdx.x;
  if (s >= s1) return;
  alpha[s - s0] = __ddiv_rn(__dsub_rn(fs[s], row_dot(col, val, rp[s], rp[s + 1], x)), nrm2[s]);
}

// pass 2 -- x~ += alpha_i a~_i^T with fp64 atomics (order nondeterministic: parity at 1e-9)
__global__ void __launch_bounds__(kNT) k1_scatter_atomic(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                         const double* __restrict__ val, const double* __restrict__ alpha,
                                                         double* __restrict__ x, int s0, int s1) {
  const int s = s0 + blockIdx.x * kNT + threadIdx.x;
  if (s >= s1) return;
  const double a = alpha[s - s0];
  for (int p = rp[s]; p < rp[s + 1]; p++) atomicAdd(x + col[p], __dmul_rn(a, val[p]));
}

cudaError_t capture_sweep(Plan& p, cudaStream_t cs, long long& nodes) {
  for (int k = 0; k < p.nsteps; k++) {
    const int s0 = p.h_step_ptr[k], s1 = p.h_step_ptr[k + 1];
    const int grid = (s1 - s0 + kNT - 1) / kNT;
    if (!p.h_overlap[k]) {
      k1_step<<<grid, kNT, 0, cs>>>(p.A.rp, p.A.col, p.A.val, p.d_fs, p.A.nrm2, p.d_xt, s0, s1);
      nodes++;
    } else {
      k1_alpha<<<grid, kNT, 0, cs>>>(p.A.rp, p.A.col, p.A.val, p.d_fs, p.A.nrm2, p.d_xt, p.d_alpha, s0, s1);
      k1_scatter_atomic<<<grid, kNT, 0, cs>>>(p.A.rp, p.A.col, p.A.val, p.d_alpha, p.d_xt, s0, s1);
      nodes += 2;
    }
  }
  return cudaGetLastError();
}

cudaError_t build_graph(Plan& p) {
  cudaError_t e;
  cudaGraph_t g;
  if ((e = cudaGraphCreate(&g, 0)) != cudaSuccess) return e;
  cudaGraphConditionalHandle h;
  if ((e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault)) != cudaSuccess) return e;
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  if ((e = cudaGraphAddNode(&node, g, nullptr, 0, &cp)) != cudaSuccess) return e;
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  cudaStream_t cs;
  if ((e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking)) != cudaSuccess) return e;
  if ((e = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
    return e;
  long long nodes = 0;
  e = capture_sweep(p, cs, nodes);
  cudaError_t e2 = launch_check_graph(p, cs, h);
  nodes++;
  cudaGraph_t out;
  cudaError_t e3 = cudaStreamEndCapture(cs, &out);
  cudaStreamDestroy(cs);
  if (e != cudaSuccess) return e;
  if (e2 != cudaSuccess) return e2;
  if (e3 != cudaSuccess) return e3;
  if ((e = cudaGraphInstantiate(&p.k1_exec, g, 0)) != cudaSuccess) return e;
  p.k1_graph = g;
  p.k1_nodes_per_sweep = nodes;
  return cudaSuccess;
}
}  // namespace

// Precondition: permute-in and ctrl init already enqueued on s.  Runs the sweep loop; the caller
// counts launches from the sweep count (nodes per sweep x sweeps).
cudaError_t k1_solve(Plan& p, cudaStream_t s, long long& launches) {
  cudaError_t e;
  (void)launches;
  if (!p.k1_exec && (e = build_graph(p)) != cudaSuccess) return e;
  return cudaGraphLaunch(p.k1_exec, s);
}

}  // namespace pobk
