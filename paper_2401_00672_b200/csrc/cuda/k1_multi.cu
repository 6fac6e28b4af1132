// K1M: several right-hand sides of one matrix in one sweep loop (the
// north star's "batches of ... right-hand sides"; Ax = f).  The schedule step
// kernel reads each row of A~ ONCE for all R right-hand sides: x~ and f~ are stored R-interleaved
// ([m][R], a column's R values in one 8R-byte run), one thread per row keeps R row sums, and
// applies the per-row contract of common.cuh to each right-hand side separately -- so right-hand
// side r's iterates are bitwise those of its own single solve.  Every right-hand side stops on its
// own RSE rule: the check kernel freezes a stopped right-hand side (the step
// kernel skips it) and clears the graph's WHILE condition when none is left.  thr = 0 plans only
// (disjoint supports: no atomics).
#include <algorithm>
#include <cmath>
#include <vector>

#include "../plan.h"
#include "common.cuh"

namespace pobk {

struct MCtrl {               // one per right-hand side
  long long sweeps;          // sweeps applied to this right-hand side
  long long max_sweeps;      // this call's cap
  long long offset;          // resume numbering
  double tol, value, den;
  int stop_mode, check_every;
  int stopped, term;
};

struct MultiPlan {
  int R = 0, Rcap = 0;
  double *xr = nullptr, *fr = nullptr, *xsr = nullptr;  // [m][R]
  MCtrl* ctrl = nullptr;                                 // [kMaxRHS]
  MCtrl* h_ctrl = nullptr;                               // pinned mirror
  unsigned* active = nullptr;                            // bit r: right-hand side r still iterating
  unsigned* arrive = nullptr;
  double* partials = nullptr;                            // [kMaxReduceBlocks * kMaxRHS]
  const double** ptrs = nullptr;                         // [3 * kMaxRHS] user f, x, x* pointers
  std::vector<const double*> h_ptrs;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int graph_R = 0;
  long long nodes_per_sweep = 0;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // sliced ELL copy of A~ (schedule order): per step, slices of 32 consecutive rows; entry j of
  // the slice's row l at off + 32 j + l (coalesced); padding entries: value +0 on the zero column m
  int64_t* sl_off = nullptr;
  int32_t* sl_w = nullptr;
  int32_t* ecol = nullptr;
  double* eval = nullptr;
  std::vector<int32_t> step_slice0;  // [nsteps] first slice of each step
};

namespace {
constexpr int kNT = 128, kCT = 256;

__global__ void k_mperm_in(int64_t m, int R, const int32_t* __restrict__ perm, const int32_t* __restrict__ orig,
                           const double* const* __restrict__ ptrs, double* __restrict__ fr, double* __restrict__ xr,
                           double* __restrict__ xsr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t o = perm[i], of = orig[i];
    for (int r = 0; r < R; r++) {
      fr[i * R + r] = ptrs[r][of];
      xr[i * R + r] = ptrs[kMaxRHS + r][o];
      if (ptrs[2 * kMaxRHS + r]) xsr[i * R + r] = ptrs[2 * kMaxRHS + r][o];
    }
  }
}

__global__ void k_mperm_out(int64_t m, int R, const int32_t* __restrict__ perm, const double* __restrict__ xr,
                            const double* const* __restrict__ ptrs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t o = perm[i];
    for (int r = 0; r < R; r++) const_cast<double*>(ptrs[kMaxRHS + r])[o] = xr[i * R + r];
  }
}

// sliced ELL (see MultiPlan): scatter the schedule-order CSR into its slices
__global__ void k1m_ell_fill(int64_t m, const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                             const double* __restrict__ val, const int32_t* __restrict__ row_slice,
                             const int64_t* __restrict__ sl_off, const int32_t* __restrict__ sl_w,
                             int32_t* __restrict__ ecol, double* __restrict__ eval, int32_t zero_col) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < m; s += (int64_t)gridDim.x * blockDim.x) {
    const int32_t sl = row_slice[s] >> 5, l = row_slice[s] & 31;
    const int64_t off = sl_off[sl];
    const int w = sl_w[sl], p0 = rp[s], len = rp[s + 1] - p0;
    for (int j = 0; j < w; j++) {
      ecol[off + 32 * j + l] = j < len ? col[p0 + j] : zero_col;
      eval[off + 32 * j + l] = j < len ? val[p0 + j] : 0.0;
    }
  }
}

// one schedule step (a category of pairwise-orthogonal rows), one thread per row:
// the row's (column, value) pairs are read once; right-hand side r follows the common.cuh
// contract: s_r = sum (a_p * x_{c_p, r}) left to right, alpha_r = (f_r - s_r) / ||a||^2,
// x_{c_p, r} += alpha_r * a_p.  Stopped right-hand sides are skipped (frozen).
// (padding entries: +0 * x_zero = +0 added to a sum that starts at +0 -- a bit-exact no-op --
// and no store).  Latency shape: a step has few rows (~30k on config 4), so each thread issues
// its row's column/value loads all at once (a kW-entry register window), then the x~ gathers a
// batch of kB entries at a time, each batch's loads in flight together -- a handful of dependent
// memory round trips per row instead of one per entry.
constexpr int kW = 24;
template <int kR>
__global__ void __launch_bounds__(kNT) k1m_step(const int32_t* __restrict__ rp, const int64_t* __restrict__ sl_off,
                                                const int32_t* __restrict__ sl_w, const int32_t* __restrict__ ecol,
                                                const double* __restrict__ eval, const double* __restrict__ fr,
                                                const double* __restrict__ nrm2, double* __restrict__ xr,
                                                const unsigned* __restrict__ active, int R, int s0, int s1, int slice0) {
  constexpr int kB = kR >= 8 ? 4 : 8;
  const int s = s0 + blockIdx.x * kNT + threadIdx.x;
  if (s >= s1) return;
  const unsigned act = *active;
  const int loc = s - s0, sl = slice0 + (loc >> 5), l = loc & 31;
  const int64_t off = sl_off[sl] + l;
  const int w = sl_w[sl], len = rp[s + 1] - rp[s];
  int c[kW];
  double a[kW];
#pragma unroll
  for (int j = 0; j < kW; j++) {
    c[j] = j < w ? __ldg(ecol + off + 32 * j) : 0;
    a[j] = j < w ? __ldg(eval + off + 32 * j) : 0.0;
  }
  double sum[kR];
#pragma unroll
  for (int r = 0; r < kR; r++) sum[r] = 0.0;
#pragma unroll
  for (int jb = 0; jb < kW; jb += kB) {
    if (jb < w) {
      double xv[kB][kR];
#pragma unroll
      for (int u = 0; u < kB; u++)
#pragma unroll
        for (int r = 0; r < kR; r++) xv[u][r] = (jb + u < w && r < R) ? xr[(size_t)c[jb + u] * R + r] : 0.0;
#pragma unroll
      for (int u = 0; u < kB; u++)
#pragma unroll
        for (int r = 0; r < kR; r++)
          if (r < R) sum[r] = __dadd_rn(sum[r], __dmul_rn(a[jb + u], xv[u][r]));
    }
  }
  for (int j = kW; j < w; j++) {  // rows past the register window
    const double aj = eval[off + 32 * j];
    const double* xc = xr + (size_t)ecol[off + 32 * j] * R;
#pragma unroll
    for (int r = 0; r < kR; r++)
      if (r < R) sum[r] = __dadd_rn(sum[r], __dmul_rn(aj, xc[r]));
  }
  double alpha[kR];
  const double n2 = nrm2[s];
#pragma unroll
  for (int r = 0; r < kR; r++) alpha[r] = r < R ? __ddiv_rn(__dsub_rn(fr[(size_t)s * R + r], sum[r]), n2) : 0.0;
#pragma unroll
  for (int jb = 0; jb < kW; jb += kB) {
    if (jb < len) {
      double xv[kB][kR];
#pragma unroll
      for (int u = 0; u < kB; u++)
#pragma unroll
        for (int r = 0; r < kR; r++) xv[u][r] = (jb + u < len && r < R) ? xr[(size_t)c[jb + u] * R + r] : 0.0;
#pragma unroll
      for (int u = 0; u < kB; u++)
#pragma unroll
        for (int r = 0; r < kR; r++)
          if (jb + u < len && r < R && ((act >> r) & 1u))
            xr[(size_t)c[jb + u] * R + r] = __dadd_rn(xv[u][r], __dmul_rn(alpha[r], a[jb + u]));
    }
  }
  for (int j = kW; j < len; j++) {
    const double aj = eval[off + 32 * j];
    double* xc = xr + (size_t)ecol[off + 32 * j] * R;
#pragma unroll
    for (int r = 0; r < kR; r++)
      if (r < R && ((act >> r) & 1u)) xc[r] = __dadd_rn(xc[r], __dmul_rn(alpha[r], aj));
  }
}

// per right-hand side: den (||x*||^2) -- mode 0 -- or the end-of-sweep RSE decision -- mode 1
// (fixed-order two-level sums; the last block decides)
__global__ void __launch_bounds__(kCT) k_mcheck(MCtrl* __restrict__ c, unsigned* __restrict__ active,
                                                unsigned* __restrict__ arrive, int64_t m, int R,
                                                const double* __restrict__ xr, const double* __restrict__ xsr,
                                                double* __restrict__ partials, int mode, cudaGraphConditionalHandle h,
                                                int use_handle) {
  __shared__ double sh[kCT / 32];
  __shared__ int is_last;
  const int64_t chunk = (m + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * chunk, b1 = min(m, b0 + chunk);
  const unsigned act = *active;
  for (int r = 0; r < R; r++) {
    double local = 0.0;
    if (((act >> r) & 1u) && xsr)
      for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
        const double d = mode == 0 ? xsr[i * R + r] : xr[i * R + r] - xsr[i * R + r];
        local = fma(d, d, local);
      }
    const double bs = block_sum<kCT>(local, sh);
    if (threadIdx.x == 0) partials[(size_t)r * gridDim.x + blockIdx.x] = bs;
  }
  if (threadIdx.x == 0) {
    __threadfence();
    is_last = (atomicAdd(arrive, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last || threadIdx.x != 0) return;
  __threadfence();
  *arrive = 0;
  unsigned still = 0u;
  for (int r = 0; r < R; r++) {
    MCtrl& cr = c[r];
    if (!((act >> r) & 1u)) continue;
    double tot = 0.0;
    for (int b = 0; b < (int)gridDim.x; b++) tot += ld_cg(partials + (size_t)r * gridDim.x + b);
    if (mode == 0) {
      cr.den = tot;
      still |= cr.stopped ? 0u : (1u << r);
      continue;
    }
    const long long s = ++cr.sweeps;
    int stopped = 0;
    if (cr.stop_mode == POBK_STOP_RSE && (((s + cr.offset) % cr.check_every) == 0 || s >= cr.max_sweeps)) {
      const double v = sqrt(tot) / sqrt(cr.den);
      cr.value = v;
      if (!isfinite(v)) { cr.term = POBK_TERM_NONFINITE; stopped = 1; }
      else if (v < cr.tol) { cr.term = POBK_TERM_CONVERGED; stopped = 1; }
    }
    if (!stopped && s >= cr.max_sweeps) { cr.term = POBK_TERM_MAX_SWEEPS; stopped = 1; }
    cr.stopped = stopped;
    still |= stopped ? 0u : (1u << r);
  }
  *active = still;
  if (mode == 1 && still == 0u && use_handle) cudaGraphSetConditional(h, 0);
}

int grid_for(int64_t m) { return (int)std::max<int64_t>(1, std::min<int64_t>((m + 255) / 256, 148 * 8)); }
int reduce_blocks(int64_t m) { return (int)std::max<int64_t>(1, std::min<int64_t>((m + 4 * kCT - 1) / (4 * kCT), 296)); }

template <int kR>
void launch_step(const Plan& p, MultiPlan& mp, cudaStream_t cs, int k) {
  const int s0 = p.h_step_ptr[k], s1 = p.h_step_ptr[k + 1];
  k1m_step<kR><<<(s1 - s0 + kNT - 1) / kNT, kNT, 0, cs>>>(p.A.rp, mp.sl_off, mp.sl_w, mp.ecol, mp.eval, mp.fr, p.A.nrm2, mp.xr,
                                                          mp.active, mp.R, s0, s1, mp.step_slice0[k]);
}

// the sliced ELL copy of the plan's schedule-order CSR (built once per plan)
cudaError_t build_ell(Plan& p, MultiPlan& mp) {
  cudaError_t e;
  std::vector<int32_t> rp(p.m + 1);
  if ((e = cudaMemcpy(rp.data(), p.A.rp, (p.m + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost)) != cudaSuccess) return e;
  std::vector<int64_t> off;
  std::vector<int32_t> w, row_slice(p.m);
  int64_t tot = 0;
  for (int k = 0; k < p.nsteps; k++) {
    const int s0 = p.h_step_ptr[k], s1 = p.h_step_ptr[k + 1];
    mp.step_slice0.push_back((int32_t)off.size());
    for (int a = s0; a < s1; a += 32) {
      int wm = 0;
      for (int r = a; r < std::min(s1, a + 32); r++) {
        wm = std::max(wm, rp[r + 1] - rp[r]);
        row_slice[r] = ((int32_t)off.size() << 5) | (r - a);
      }
      off.push_back(tot);
      w.push_back(wm);
      tot += 32 * (int64_t)wm;
    }
  }
  int32_t* d_rs = nullptr;
  if ((e = cudaMalloc(&mp.sl_off, std::max<size_t>(off.size(), 1) * sizeof(int64_t))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&mp.sl_w, std::max<size_t>(w.size(), 1) * sizeof(int32_t))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&mp.ecol, std::max<int64_t>(tot, 1) * sizeof(int32_t))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&mp.eval, std::max<int64_t>(tot, 1) * sizeof(double))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&d_rs, p.m * sizeof(int32_t))) != cudaSuccess) return e;
  cudaMemcpy(mp.sl_off, off.data(), off.size() * sizeof(int64_t), cudaMemcpyHostToDevice);
  cudaMemcpy(mp.sl_w, w.data(), w.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
  cudaMemcpy(d_rs, row_slice.data(), p.m * sizeof(int32_t), cudaMemcpyHostToDevice);
  k1m_ell_fill<<<grid_for(p.m), 256>>>(p.m, p.A.rp, p.A.col, p.A.val, d_rs, mp.sl_off, mp.sl_w, mp.ecol, mp.eval,
                                         (int32_t)p.m);
  e = cudaDeviceSynchronize();
  cudaFree(d_rs);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t build_graph(Plan& p, MultiPlan& mp) {
  if (mp.exec) {
    cudaGraphExecDestroy(mp.exec);
    cudaGraphDestroy(mp.graph);
    mp.exec = nullptr;
    mp.graph = nullptr;
  }
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
  for (int k = 0; k < p.nsteps; k++) {
    if (mp.R <= 1) launch_step<1>(p, mp, cs, k);
    else if (mp.R <= 2) launch_step<2>(p, mp, cs, k);
    else if (mp.R <= 4) launch_step<4>(p, mp, cs, k);
    else launch_step<kMaxRHS>(p, mp, cs, k);
    nodes++;
  }
  k_mcheck<<<reduce_blocks(p.m), kCT, 0, cs>>>(mp.ctrl, mp.active, mp.arrive, p.m, mp.R, mp.xr, mp.xsr, mp.partials, 1, h, 1);
  nodes++;
  cudaError_t e1 = cudaGetLastError();
  cudaGraph_t out;
  cudaError_t e3 = cudaStreamEndCapture(cs, &out);
  cudaStreamDestroy(cs);
  if (e1 != cudaSuccess) return e1;
  if (e3 != cudaSuccess) return e3;
  if ((e = cudaGraphInstantiate(&mp.exec, g, 0)) != cudaSuccess) return e;
  mp.graph = g;
  mp.graph_R = mp.R;
  mp.nodes_per_sweep = nodes;
  return cudaSuccess;
}

template <typename T>
cudaError_t grow(T** p, size_t n) {
  if (*p) cudaFree(*p);
  *p = nullptr;
  return cudaMalloc((void**)p, std::max<size_t>(n, 1) * sizeof(T));
}
}  // namespace

cudaError_t k1m_solve(Plan& p, int R, const double* const* f, double* const* x, const double* const* xstar,
                      const pobk_solve_opts& o, cudaStream_t s, pobk_report* reps) {
  cudaError_t e;
  if (!p.multi) p.multi = new MultiPlan();
  MultiPlan& mp = *p.multi;
  if (!mp.ecol && (e = build_ell(p, mp)) != cudaSuccess) return e;
  if (R > mp.Rcap) {
    if ((e = grow(&mp.xr, (size_t)(p.m + 1) * R)) != cudaSuccess) return e;  // (+ the zero column m)
    if ((e = grow(&mp.fr, (size_t)p.m * R)) != cudaSuccess) return e;
    if ((e = grow(&mp.xsr, (size_t)p.m * R)) != cudaSuccess) return e;
    mp.Rcap = R;
  }
  if (!mp.ctrl) {
    if ((e = cudaMalloc(&mp.ctrl, kMaxRHS * sizeof(MCtrl))) != cudaSuccess) return e;
    if ((e = cudaMallocHost(&mp.h_ctrl, kMaxRHS * sizeof(MCtrl))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&mp.active, sizeof(unsigned))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&mp.arrive, sizeof(unsigned))) != cudaSuccess) return e;
    if ((e = cudaMemset(mp.arrive, 0, sizeof(unsigned))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&mp.partials, 296 * kMaxRHS * sizeof(double))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&mp.ptrs, 3 * kMaxRHS * sizeof(double*))) != cudaSuccess) return e;
    mp.h_ptrs.assign(3 * kMaxRHS, nullptr);
    for (auto& ev : mp.ev)
      if ((e = cudaEventCreate(&ev)) != cudaSuccess) return e;
  }
  mp.R = R;
  if (!mp.exec || mp.graph_R != R) {
    if ((e = build_graph(p, mp)) != cudaSuccess) return e;
  }
  const long long ncall = o.max_sweeps - o.sweep_offset;
  for (int r = 0; r < R; r++) {
    MCtrl& c = mp.h_ctrl[r];
    c.sweeps = 0;
    c.max_sweeps = ncall;
    c.offset = o.sweep_offset;
    c.tol = o.tol;
    c.value = NAN;
    c.den = 0.0;
    c.stop_mode = o.stop;
    c.check_every = o.check_every;
    c.stopped = ncall <= 0 ? 1 : 0;
    c.term = POBK_TERM_MAX_SWEEPS;
    mp.h_ptrs[r] = f[r];
    mp.h_ptrs[kMaxRHS + r] = x[r];
    mp.h_ptrs[2 * kMaxRHS + r] = o.stop == POBK_STOP_RSE ? xstar[r] : nullptr;
  }
  const unsigned all = ncall > 0 ? (R >= 32 ? 0xffffffffu : ((1u << R) - 1u)) : 0u;
  if ((e = cudaEventRecord(mp.ev[0], s)) != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(mp.ctrl, mp.h_ctrl, R * sizeof(MCtrl), cudaMemcpyHostToDevice, s)) != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(mp.ptrs, mp.h_ptrs.data(), 3 * kMaxRHS * sizeof(double*), cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return e;
  if ((e = cudaMemcpyAsync(mp.active, &all, sizeof(unsigned), cudaMemcpyHostToDevice, s)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(mp.xr + (size_t)p.m * R, 0, R * sizeof(double), s)) != cudaSuccess) return e;  // zero column
  k_mperm_in<<<grid_for(p.m), 256, 0, s>>>(p.m, R, p.d_perm, p.A.orig, mp.ptrs, mp.fr, mp.xr, mp.xsr);
  long long launches = 1;
  if (o.stop == POBK_STOP_RSE) {
    k_mcheck<<<reduce_blocks(p.m), kCT, 0, s>>>(mp.ctrl, mp.active, mp.arrive, p.m, R, mp.xr, mp.xsr, mp.partials, 0, 0, 0);
    launches++;
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = cudaEventRecord(mp.ev[1], s)) != cudaSuccess) return e;
  if (ncall > 0 && (e = cudaGraphLaunch(mp.exec, s)) != cudaSuccess) return e;
  if ((e = cudaEventRecord(mp.ev[2], s)) != cudaSuccess) return e;
  k_mperm_out<<<grid_for(p.m), 256, 0, s>>>(p.m, R, p.d_perm, mp.xr, mp.ptrs);
  launches++;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = cudaEventRecord(mp.ev[3], s)) != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(mp.h_ctrl, mp.ctrl, R * sizeof(MCtrl), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  float t_all = 0.f, t_sw = 0.f;
  cudaEventElapsedTime(&t_all, mp.ev[0], mp.ev[3]);
  cudaEventElapsedTime(&t_sw, mp.ev[1], mp.ev[2]);
  long long maxsw = 0;
  for (int r = 0; r < R; r++) maxsw = std::max(maxsw, mp.h_ctrl[r].sweeps);
  for (int r = 0; r < R && reps; r++) {
    const MCtrl& c = mp.h_ctrl[r];
    pobk_report& rp = reps[r];
    rp.sweeps = c.sweeps;
    rp.termination = c.term;
    rp.kernel = POBK_KERNEL_LAUNCH;
    rp.final_value = o.stop == POBK_STOP_NONE ? NAN : c.value;
    rp.solve_seconds = t_all * 1e-3;
    rp.sweep_seconds = t_sw * 1e-3;
    rp.launches = launches + maxsw * mp.nodes_per_sweep;
    rp.sweeps_total = o.sweep_offset + c.sweeps;
    rp.final_rse = o.stop == POBK_STOP_RSE ? c.value : NAN;
    rp.final_relres = NAN;
  }
  return cudaSuccess;
}

void k1m_free(Plan& p) {
  if (!p.multi) return;
  MultiPlan& mp = *p.multi;
  if (mp.exec) cudaGraphExecDestroy(mp.exec);
  if (mp.graph) cudaGraphDestroy(mp.graph);
  for (void* v : {(void*)mp.xr, (void*)mp.fr, (void*)mp.xsr, (void*)mp.ctrl, (void*)mp.active, (void*)mp.arrive,
                  (void*)mp.partials, (void*)mp.ptrs, (void*)mp.sl_off, (void*)mp.sl_w, (void*)mp.ecol, (void*)mp.eval})
    if (v) cudaFree(v);
  if (mp.h_ctrl) cudaFreeHost(mp.h_ctrl);
  for (auto& ev : mp.ev)
    if (ev) cudaEventDestroy(ev);
  delete p.multi;
  p.multi = nullptr;
}

}  // namespace pobk
