// K1: one launch per schedule step, V lanes per row, x~ in global memory (L2-resident).
//
// A sweep (Alg 5 loop body) is the sequence of its steps; a step is one
// category of pairwise-orthogonal rows, whose block projection Eq 1.3
// collapses by Lemma 1 to independent Eq 1.2 row projections
// (PAPER.md:29): one thread vector per row, no atomics (disjoint supports), the launch boundary is
// the step barrier.  Steps whose rows overlap (thr > 0 only) run as two launches: all alphas at
// the same x~, then an fp64-atomic scatter.
//
// The sweep loop is device-driven: the steps + the stop check are the body of a CUDA-graph WHILE
// node whose condition the check kernel clears (no host round trip per sweep).
#include "../plan.h"
#include "common.cuh"

namespace pobk {

cudaError_t launch_check_graph(const Plan& p, cudaStream_t s, cudaGraphConditionalHandle h);

namespace {
constexpr int kNT = 256;

template <int V>
__global__ void __launch_bounds__(kNT) k1_step(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                               const double* __restrict__ val, const double* __restrict__ fs,
                                               const double* __restrict__ nrm2, double* __restrict__ x, int s0, int s1) {
  const int gid = blockIdx.x * kNT + threadIdx.x;
  const int s = s0 + gid / V, lane = gid % V;
  const bool act = s < s1;
  const int p0 = act ? rp[s] : 0, p1 = act ? rp[s + 1] : 0;
  double acc = 0.0;
  for (int p = p0 + lane; p < p1; p += V) acc = fma(val[p], x[col[p]], acc);
  acc = vec_sum<V>(acc);
  if (!act) return;
  const double alpha = (fs[s] - acc) / nrm2[s];
  for (int p = p0 + lane; p < p1; p += V) {
    const int c = col[p];
    x[c] = fma(alpha, val[p], x[c]);
  }
}

// thr > 0, overlapping step: pass 1 -- every alpha at the same x~
template <int V>
__global__ void __launch_bounds__(kNT) k1_alpha(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                const double* __restrict__ val, const double* __restrict__ fs,
                                                const double* __restrict__ nrm2, const double* __restrict__ x,
                                                double* __restrict__ alpha, int s0, int s1) {
  const int gid = blockIdx.x * kNT + threadIdx.x;
  const int s = s0 + gid / V, lane = gid % V;
  const bool act = s < s1;
  const int p0 = act ? rp[s] : 0, p1 = act ? rp[s + 1] : 0;
  double acc = 0.0;
  for (int p = p0 + lane; p < p1; p += V) acc = fma(val[p], x[col[p]], acc);
  acc = vec_sum<V>(acc);
  if (act && lane == 0) alpha[s - s0] = (fs[s] - acc) / nrm2[s];
}

// pass 2 -- x~ += alpha_i a~_i^T with fp64 atomics (order nondeterministic: parity at 1e-9)
template <int V>
__global__ void __launch_bounds__(kNT) k1_scatter_atomic(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                         const double* __restrict__ val, const double* __restrict__ alpha,
                                                         double* __restrict__ x, int s0, int s1) {
  const int gid = blockIdx.x * kNT + threadIdx.x;
  const int s = s0 + gid / V, lane = gid % V;
  if (s >= s1) return;
  const double a = alpha[s - s0];
  for (int p = rp[s] + lane; p < rp[s + 1]; p += V) atomicAdd(x + col[p], a * val[p]);
}

template <int V>
cudaError_t capture_sweep(Plan& p, cudaStream_t cs, long long& nodes) {
  for (int k = 0; k < p.nsteps; k++) {
    const int s0 = p.h_step_ptr[k], s1 = p.h_step_ptr[k + 1];
    const int n = s1 - s0;
    const int grid = (int)(((int64_t)n * V + kNT - 1) / kNT);
    if (!p.h_overlap[k]) {
      k1_step<V><<<grid, kNT, 0, cs>>>(p.A.rp, p.A.col, p.A.val, p.d_fs, p.A.nrm2, p.d_xt, s0, s1);
      nodes++;
    } else {
      k1_alpha<V><<<grid, kNT, 0, cs>>>(p.A.rp, p.A.col, p.A.val, p.d_fs, p.A.nrm2, p.d_xt, p.d_alpha, s0, s1);
      k1_scatter_atomic<V><<<grid, kNT, 0, cs>>>(p.A.rp, p.A.col, p.A.val, p.d_alpha, p.d_xt, s0, s1);
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
  switch (p.V) {
    case 1: e = capture_sweep<1>(p, cs, nodes); break;
    case 2: e = capture_sweep<2>(p, cs, nodes); break;
    case 4: e = capture_sweep<4>(p, cs, nodes); break;
    case 8: e = capture_sweep<8>(p, cs, nodes); break;
    case 16: e = capture_sweep<16>(p, cs, nodes); break;
    default: e = capture_sweep<32>(p, cs, nodes); break;
  }
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

// Precondition: permute-in and ctrl init already enqueued on s.  Runs the sweep loop.
cudaError_t k1_solve(Plan& p, cudaStream_t s, long long& launches) {
  cudaError_t e;
  if (!p.k1_exec && (e = build_graph(p)) != cudaSuccess) return e;
  if ((e = cudaGraphLaunch(p.k1_exec, s)) != cudaSuccess) return e;
  // launches are counted by the caller from the sweep count (nodes per sweep x sweeps)
  (void)launches;
  return cudaSuccess;
}

}  // namespace pobk
