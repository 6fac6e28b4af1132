// K1: one launch per schedule step, one thread per row, x~ in global memory (L2-resident).
//
// A sweep (Alg 5 loop body) is the sequence of its steps; a step is one
// category of pairwise-orthogonal rows, whose block projection Eq 1.3
// collapses by Lemma 1 to independent Eq 1.2 row projections
// (PAPER.md:29): one thread per row (common.cuh contract), no atomics (disjoint supports), the
// launch boundary is the step barrier.  Steps whose rows overlap (thr > 0 only) run as two
// launches: all alphas at the same x~, then the scatter as an ordered fold per column (bitwise the
// oracle's; POBK_THR_ATOMIC=1: an fp64-atomic scatter, order nondeterministic).
//
// The sweep loop is device-driven: the steps + the stop check are the body of a CUDA-graph WHILE
// node whose condition the check kernel clears (no host round trip per sweep).  K1 is the
// general fallback (any size, any thr); K2/K3 are the fast paths.
#include <algorithm>
#include <cstdlib>
#include <vector>

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

// pass 2, ordered (default): one thread per column the step touches, folding the step's
// contributions in ascending schedule position -- x~_c = (x~_c + alpha_i1 a~_i1c) + alpha_i2 a~_i2c
// ..., each product and sum rounded, which is the oracle's order (rows ascending, entries
// ascending): bitwise the oracle's iterates, no atomics
__global__ void __launch_bounds__(kNT) k1_scatter_ordered(const int32_t* __restrict__ cols, const int32_t* __restrict__ eptr,
                                                          const int32_t* __restrict__ es, const double* __restrict__ ev,
                                                          const double* __restrict__ alpha, double* __restrict__ x, int c0,
                                                          int c1) {
  const int t = c0 + blockIdx.x * kNT + threadIdx.x;
  if (t >= c1) return;
  const int c = cols[t];
  double xc = x[c];
  for (int e = eptr[t]; e < eptr[t + 1]; e++) xc = __dadd_rn(xc, __dmul_rn(alpha[es[e]], ev[e]));
  x[c] = xc;
}

cudaError_t capture_sweep(Plan& p, cudaStream_t cs, long long& nodes) {
  const bool atomic = getenv("POBK_THR_ATOMIC") != nullptr;  // the fp64-atomic scatter (order nondeterministic)
  for (int k = 0; k < p.nsteps; k++) {
    const int s0 = p.h_step_ptr[k], s1 = p.h_step_ptr[k + 1];
    const int grid = (s1 - s0 + kNT - 1) / kNT;
    if (!p.h_overlap[k]) {
      k1_step<<<grid, kNT, 0, cs>>>(p.A.rp, p.A.col, p.A.val, p.d_fs, p.A.nrm2, p.d_xt, s0, s1);
      nodes++;
    } else {
      k1_alpha<<<grid, kNT, 0, cs>>>(p.A.rp, p.A.col, p.A.val, p.d_fs, p.A.nrm2, p.d_xt, p.d_alpha, s0, s1);
      nodes++;
      const int c0 = p.h_ov_colptr[k], c1 = p.h_ov_colptr[k + 1];
      if (atomic) {
        k1_scatter_atomic<<<grid, kNT, 0, cs>>>(p.A.rp, p.A.col, p.A.val, p.d_alpha, p.d_xt, s0, s1);
        nodes++;
      } else if (c1 > c0) {
        k1_scatter_ordered<<<(c1 - c0 + kNT - 1) / kNT, kNT, 0, cs>>>(p.ov_cols, p.ov_eptr, p.ov_es, p.ov_ev, p.d_alpha,
                                                                     p.d_xt, c0, c1);
        nodes++;
      }
    }
  }
  return cudaGetLastError();
}

// ---- residual-ordered sweep (opts.order = POBK_ORDER_RESIDUAL, DESIGN.md
// reading R-G): at the start of every sweep, rho_K = ||f~_K - A~_K x~||^2 / ||A~_K||_F^2 per step,
// both sums over the step's rows in schedule order in a fixed two-level grouping (chunks of
// kChunk rows left to right, then the chunk sums left to right -- the oracle's grouping, so
// the same order decisions); steps applied by decreasing rho (ties: ascending index).
constexpr int kChunk = 256;

__global__ void __launch_bounds__(kNT) k1o_resid2(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                  const double* __restrict__ val, const double* __restrict__ fs,
                                                  const double* __restrict__ x, double* __restrict__ rr, int64_t m) {
  const int64_t s = blockIdx.x * (int64_t)kNT + threadIdx.x;
  if (s >= m) return;
  const double r = __dsub_rn(fs[s], row_dot(col, val, rp[s], rp[s + 1], x));
  rr[s] = __dmul_rn(r, r);
}

__global__ void __launch_bounds__(kNT) k1o_chunks(const double* __restrict__ rr, const double* __restrict__ nrm2,
                                                  const int32_t* __restrict__ cb, double* __restrict__ cs,
                                                  double* __restrict__ cn, int nchunks) {
  const int c = blockIdx.x * kNT + threadIdx.x;
  if (c >= nchunks) return;
  double a = 0.0, b = 0.0;
  for (int s = cb[2 * c]; s < cb[2 * c + 1]; s++) {
    a = __dadd_rn(a, rr[s]);
    b = __dadd_rn(b, nrm2[s]);
  }
  cs[c] = a;
  cn[c] = b;
}

// one block: every step's score from its chunk sums, then a stable sort by decreasing score
__global__ void k1o_order(const int32_t* __restrict__ step_chunk, const double* __restrict__ cs,
                          const double* __restrict__ cn, double* __restrict__ rho, int32_t* __restrict__ order,
                          int nsteps) {
  for (int k = threadIdx.x; k < nsteps; k += blockDim.x) {
    double a = 0.0, b = 0.0;
    for (int c = step_chunk[k]; c < step_chunk[k + 1]; c++) {
      a = __dadd_rn(a, cs[c]);
      b = __dadd_rn(b, cn[c]);
    }
    rho[k] = __ddiv_rn(a, b);
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int k = 0; k < nsteps; k++) {  // insertion sort: stable, keys (-rho, index)
    const double r = rho[k];
    int j = k - 1;
    while (j >= 0 && rho[order[j]] < r) {
      order[j + 1] = order[j];
      j--;
    }
    order[j + 1] = k;
  }
}

__global__ void __launch_bounds__(kNT) k1o_step(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                const double* __restrict__ val, const double* __restrict__ fs,
                                                const double* __restrict__ nrm2, double* __restrict__ x,
                                                const int32_t* __restrict__ step_ptr, const int32_t* __restrict__ order,
                                                int j) {
  const int k = order[j];
  const int s = step_ptr[k] + blockIdx.x * kNT + threadIdx.x;
  if (s >= step_ptr[k + 1]) return;
  row_project(col, val, rp[s], rp[s + 1], fs[s], nrm2[s], x);
}

cudaError_t build_graph_ordered(Plan& p) {
  cudaError_t e;
  // chunk list and per-step chunk ranges (host), scratch (device)
  std::vector<int32_t> cb, sc(p.nsteps + 1, 0);
  int32_t maxrows = 1;
  for (int k = 0; k < p.nsteps; k++) {
    const int s0 = p.h_step_ptr[k], s1 = p.h_step_ptr[k + 1];
    maxrows = std::max(maxrows, s1 - s0);
    for (int a = s0; a < s1; a += kChunk) {
      cb.push_back(a);
      cb.push_back(std::min(s1, a + kChunk));
    }
    sc[k + 1] = (int32_t)(cb.size() / 2);
  }
  const int nch = (int)(cb.size() / 2);
  int32_t *d_cb = nullptr, *d_sc = nullptr, *d_order = nullptr;
  double *d_rr = nullptr, *d_cs = nullptr, *d_cn = nullptr, *d_rho = nullptr;
  auto al = [&](void** v, size_t n) { e = cudaMalloc(v, std::max<size_t>(n, 1)); if (e == cudaSuccess) p.allocations.push_back(*v); return e; };
  if (al((void**)&d_cb, cb.size() * 4) || al((void**)&d_sc, sc.size() * 4) || al((void**)&d_order, p.nsteps * 4) ||
      al((void**)&d_rr, p.m * 8) || al((void**)&d_cs, nch * 8) || al((void**)&d_cn, nch * 8) || al((void**)&d_rho, p.nsteps * 8))
    return e;
  if ((e = cudaMemcpy(d_cb, cb.data(), cb.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess) return e;
  if ((e = cudaMemcpy(d_sc, sc.data(), sc.size() * 4, cudaMemcpyHostToDevice)) != cudaSuccess) return e;
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
  k1o_resid2<<<(int)((p.m + kNT - 1) / kNT), kNT, 0, cs>>>(p.A.rp, p.A.col, p.A.val, p.d_fs, p.d_xt, d_rr, p.m);
  k1o_chunks<<<(nch + kNT - 1) / kNT, kNT, 0, cs>>>(d_rr, p.A.nrm2, d_cb, d_cs, d_cn, nch);
  k1o_order<<<1, 256, 0, cs>>>(d_sc, d_cs, d_cn, d_rho, d_order, p.nsteps);
  nodes += 3;
  for (int j = 0; j < p.nsteps; j++) {
    k1o_step<<<(maxrows + kNT - 1) / kNT, kNT, 0, cs>>>(p.A.rp, p.A.col, p.A.val, p.d_fs, p.A.nrm2, p.d_xt, p.k3_step_ptr,
                                                       d_order, j);
    nodes++;
  }
  e = cudaGetLastError();
  cudaError_t e2 = launch_check_graph(p, cs, h);
  nodes++;
  cudaGraph_t out;
  cudaError_t e3 = cudaStreamEndCapture(cs, &out);
  cudaStreamDestroy(cs);
  if (e != cudaSuccess) return e;
  if (e2 != cudaSuccess) return e2;
  if (e3 != cudaSuccess) return e3;
  if ((e = cudaGraphInstantiate(&p.k1o_exec, g, 0)) != cudaSuccess) return e;
  p.k1o_graph = g;
  p.k1o_nodes_per_sweep = nodes;
  return cudaSuccess;
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

// the residual-ordered sweep loop (thr = 0 plans)
cudaError_t k1_solve_ordered(Plan& p, cudaStream_t s, long long& launches) {
  cudaError_t e;
  (void)launches;
  if (!p.k1o_exec && (e = build_graph_ordered(p)) != cudaSuccess) return e;
  return cudaGraphLaunch(p.k1o_exec, s);
}

}  // namespace pobk
