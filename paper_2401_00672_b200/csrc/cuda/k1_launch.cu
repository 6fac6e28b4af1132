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
//
// K1E: the step and alpha kernels read a sliced-ELL copy of A~ (built on the device at the first
// solve) in batches of 16 entries -- a step is a small grid of one-row threads, so the row's
// dependent L2 round trips set its time (config 4: 678 -> 347 us/sweep); bitwise the CSR kernels.
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

// ---- K1E: the same two kernels on the sliced ELL copy (coalesced entry loads: with the CSR a
// warp's 32 rows sit ~200 bytes apart, 32 sectors per load instruction).  Same operations in the
// same order per row (common.cuh contract): bitwise the CSR kernels' iterates.
// Loads in batches of kB entries (all columns, then all x~, then the products, then the ordered
// adds): the row's ~2 x len dependent L2 round trips become ~2 x len / kB.
constexpr int kB = 16;

__device__ __forceinline__ double k1e_dot(const int32_t* __restrict__ ecol, const double* __restrict__ eval, int64_t b,
                                          int len, const double* x) {
  double sum = 0.0;
  for (int j0 = 0; j0 < len; j0 += kB) {
    int c[kB];
    double v[kB], pr[kB];
#pragma unroll
    for (int u = 0; u < kB; u++) {
      const bool on = j0 + u < len;
      c[u] = on ? ecol[b + 32 * (int64_t)(j0 + u)] : -1;
      v[u] = on ? eval[b + 32 * (int64_t)(j0 + u)] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kB; u++) pr[u] = c[u] >= 0 ? x[c[u]] : 0.0;
#pragma unroll
    for (int u = 0; u < kB; u++) pr[u] = pin(__dmul_rn(v[u], pr[u]));
#pragma unroll
    for (int u = 0; u < kB; u++)
      if (c[u] >= 0) sum = __dadd_rn(sum, pr[u]);
  }
  return sum;
}

__device__ __forceinline__ void k1e_row(const int32_t* __restrict__ rp, const int64_t* __restrict__ sptr,
                                        const int32_t* __restrict__ ecol, const double* __restrict__ eval,
                                        const double* __restrict__ fs, const double* __restrict__ nrm2, double* x, int s0,
                                        int s1, int slice0);

__global__ void __launch_bounds__(kNT) k1e_step(const int32_t* __restrict__ rp, const int64_t* __restrict__ sptr,
                                                const int32_t* __restrict__ ecol, const double* __restrict__ eval,
                                                const double* __restrict__ fs, const double* __restrict__ nrm2,
                                                double* x, int s0, int s1, int slice0) {
  k1e_row(rp, sptr, ecol, eval, fs, nrm2, x, s0, s1, slice0);
}

// the residual-ordered loop's step (schedule position j of this sweep's order) on the same layout
__global__ void __launch_bounds__(kNT) k1oe_step(const int32_t* __restrict__ rp, const int64_t* __restrict__ sptr,
                                                 const int32_t* __restrict__ ecol, const double* __restrict__ eval,
                                                 const double* __restrict__ fs, const double* __restrict__ nrm2,
                                                 double* x, const int32_t* __restrict__ step_ptr,
                                                 const int32_t* __restrict__ slice0, const int32_t* __restrict__ order,
                                                 int j) {
  const int k = order[j];
  k1e_row(rp, sptr, ecol, eval, fs, nrm2, x, step_ptr[k], step_ptr[k + 1], slice0[k]);
}

__device__ __forceinline__ void k1e_row(const int32_t* __restrict__ rp, const int64_t* __restrict__ sptr,
                                        const int32_t* __restrict__ ecol, const double* __restrict__ eval,
                                        const double* __restrict__ fs, const double* __restrict__ nrm2, double* x, int s0,
                                        int s1, int slice0) {
  const int s = s0 + blockIdx.x * kNT + threadIdx.x;
  if (s >= s1) return;
  const int len = rp[s + 1] - rp[s];
  const int64_t b = sptr[slice0 + blockIdx.x * (kNT / 32) + (threadIdx.x >> 5)] + (threadIdx.x & 31);
  const double alpha = __ddiv_rn(__dsub_rn(fs[s], k1e_dot(ecol, eval, b, len, x)), nrm2[s]);
  // the row's columns are distinct (strictly increasing, validated), so a batch's x~ loads may
  // all precede its stores
  for (int j0 = 0; j0 < len; j0 += kB) {
    int c[kB];
    double v[kB], xv[kB];
#pragma unroll
    for (int u = 0; u < kB; u++) {
      const bool on = j0 + u < len;
      c[u] = on ? ecol[b + 32 * (int64_t)(j0 + u)] : -1;
      v[u] = on ? eval[b + 32 * (int64_t)(j0 + u)] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kB; u++) xv[u] = c[u] >= 0 ? x[c[u]] : 0.0;
#pragma unroll
    for (int u = 0; u < kB; u++)
      if (c[u] >= 0) x[c[u]] = __dadd_rn(xv[u], __dmul_rn(alpha, v[u]));
  }
}

__global__ void __launch_bounds__(kNT) k1e_alpha(const int32_t* __restrict__ rp, const int64_t* __restrict__ sptr,
                                                 const int32_t* __restrict__ ecol, const double* __restrict__ eval,
                                                 const double* __restrict__ fs, const double* __restrict__ nrm2,
                                                 const double* __restrict__ x, double* __restrict__ alpha, int s0, int s1,
                                                 int slice0) {
  const int s = s0 + blockIdx.x * kNT + threadIdx.x;
  if (s >= s1) return;
  const int len = rp[s + 1] - rp[s];
  const int64_t b = sptr[slice0 + blockIdx.x * (kNT / 32) + (threadIdx.x >> 5)] + (threadIdx.x & 31);
  alpha[s - s0] = __ddiv_rn(__dsub_rn(fs[s], k1e_dot(ecol, eval, b, len, x)), nrm2[s]);
}

// one warp per slice: CSR rows -> the slice's interleaved entries (padding stays zero, never read)
__global__ void __launch_bounds__(kNT) k1e_fill(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                const double* __restrict__ val, const int32_t* __restrict__ srow,
                                                const int64_t* __restrict__ sptr, int32_t* __restrict__ ecol,
                                                double* __restrict__ eval, int nslices) {
  const int sl = blockIdx.x * (kNT / 32) + (threadIdx.x >> 5), l = threadIdx.x & 31;
  if (sl >= nslices) return;
  const int r = srow[2 * sl] + l;
  if (r >= srow[2 * sl + 1]) return;
  const int p0 = rp[r], len = rp[r + 1] - p0;
  const int64_t b = sptr[sl] + l;
  for (int j = 0; j < len; j++) {
    ecol[b + 32 * (int64_t)j] = col[p0 + j];
    eval[b + 32 * (int64_t)j] = val[p0 + j];
  }
}

// Builds the sliced ELL copy (once per plan, before the graph capture).  Any failure (memory)
// leaves k1e_col NULL: the CSR kernels run instead.  POBK_K1_CSR=1 keeps the CSR kernels.
void build_k1e(Plan& p) {
  if (p.k1e_col || getenv("POBK_K1_CSR") != nullptr || p.m == 0) return;
  std::vector<int32_t> rp(p.m + 1), srow;
  if (cudaMemcpy(rp.data(), p.A.rp, (p.m + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  std::vector<int64_t> sptr(1, 0);
  std::vector<int32_t> slice0(p.nsteps, 0);
  for (int k = 0; k < p.nsteps; k++) {
    slice0[k] = (int32_t)(sptr.size() - 1);
    for (int a = p.h_step_ptr[k]; a < p.h_step_ptr[k + 1]; a += 32) {
      const int b = std::min(p.h_step_ptr[k + 1], a + 32);
      int w = 0;
      for (int r = a; r < b; r++) w = std::max(w, rp[r + 1] - rp[r]);
      srow.push_back(a);
      srow.push_back(b);
      sptr.push_back(sptr.back() + 32 * (int64_t)w);
    }
  }
  const int nsl = (int)(sptr.size() - 1);
  const size_t ne = (size_t)std::max<int64_t>(sptr.back(), 1);
  int32_t *ecol = nullptr, *d_srow = nullptr;
  double* eval = nullptr;
  int64_t* d_sptr = nullptr;
  int32_t* d_sl0 = nullptr;
  bool ok = cudaMalloc((void**)&ecol, ne * 4) == cudaSuccess && cudaMalloc((void**)&eval, ne * 8) == cudaSuccess &&
            cudaMalloc((void**)&d_sl0, std::max<size_t>(slice0.size(), 1) * 4) == cudaSuccess &&
            cudaMemcpy(d_sl0, slice0.data(), slice0.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
            cudaMalloc((void**)&d_sptr, sptr.size() * 8) == cudaSuccess &&
            cudaMalloc((void**)&d_srow, std::max<size_t>(srow.size(), 1) * 4) == cudaSuccess;
  ok = ok && cudaMemset(ecol, 0, ne * 4) == cudaSuccess && cudaMemset(eval, 0, ne * 8) == cudaSuccess &&
       cudaMemcpy(d_sptr, sptr.data(), sptr.size() * 8, cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMemcpy(d_srow, srow.data(), srow.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess;
  if (ok && nsl > 0) {
    k1e_fill<<<(nsl + kNT / 32 - 1) / (kNT / 32), kNT>>>(p.A.rp, p.A.col, p.A.val, d_srow, d_sptr, ecol, eval, nsl);
    ok = cudaDeviceSynchronize() == cudaSuccess;
  }
  if (d_srow) cudaFree(d_srow);
  if (!ok) {
    cudaGetLastError();
    if (ecol) cudaFree(ecol);
    if (eval) cudaFree(eval);
    if (d_sptr) cudaFree(d_sptr);
    if (d_sl0) cudaFree(d_sl0);
    return;
  }
  p.allocations.push_back(ecol);
  p.allocations.push_back(eval);
  p.allocations.push_back(d_sptr);
  p.k1e_col = ecol;
  p.k1e_val = eval;
  p.k1e_ptr = d_sptr;
  p.allocations.push_back(d_sl0);
  p.k1e_slice0 = d_sl0;
  p.h_k1e_slice0 = slice0;
}

cudaError_t capture_sweep(Plan& p, cudaStream_t cs, long long& nodes) {
  const bool atomic = getenv("POBK_THR_ATOMIC") != nullptr;  // the fp64-atomic scatter (order nondeterministic)
  const bool ell = p.k1e_col != nullptr;
  for (int k = 0; k < p.nsteps; k++) {
    const int s0 = p.h_step_ptr[k], s1 = p.h_step_ptr[k + 1];
    const int grid = (s1 - s0 + kNT - 1) / kNT;
    if (!p.h_overlap[k]) {
      if (ell)
        k1e_step<<<grid, kNT, 0, cs>>>(p.A.rp, p.k1e_ptr, p.k1e_col, p.k1e_val, p.d_fs, p.A.nrm2, p.d_xt, s0, s1,
                                       p.h_k1e_slice0[k]);
      else
        k1_step<<<grid, kNT, 0, cs>>>(p.A.rp, p.A.col, p.A.val, p.d_fs, p.A.nrm2, p.d_xt, s0, s1);
      nodes++;
    } else {
      if (ell)
        k1e_alpha<<<grid, kNT, 0, cs>>>(p.A.rp, p.k1e_ptr, p.k1e_col, p.k1e_val, p.d_fs, p.A.nrm2, p.d_xt, p.d_alpha, s0,
                                        s1, p.h_k1e_slice0[k]);
      else
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
  build_k1e(p);
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
    if (p.k1e_col)
      k1oe_step<<<(maxrows + kNT - 1) / kNT, kNT, 0, cs>>>(p.A.rp, p.k1e_ptr, p.k1e_col, p.k1e_val, p.d_fs, p.A.nrm2,
                                                          p.d_xt, p.k3_step_ptr, p.k1e_slice0, d_order, j);
    else
      k1o_step<<<(maxrows + kNT - 1) / kNT, kNT, 0, cs>>>(p.A.rp, p.A.col, p.A.val, p.d_fs, p.A.nrm2, p.d_xt,
                                                         p.k3_step_ptr, d_order, j);
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
  build_k1e(p);
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
