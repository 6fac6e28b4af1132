// Vector-level kernels around the sweep:
//   K6  permute in / out       f~ = P f, x~0 = P x0, x~* = P x* (Eq 3.1);
//                              x = P^T x~
//   K5  stop check             RSE = ||x~ - x~*|| / ||x~*|| every check_every sweeps,
//                              decided on the device (last-block-done, deterministic order)
//   K4  residual               sum (f~_i - a~_i . x~)^2: the fused SpMV + squared norm used by the
//                              RELRES stop and by pobk_residual_norm / pobk_residual_sumsq_rows
// All reductions are two-level and deterministic: block b owns a fixed chunk, a fixed tree per
// block, and the last block to arrive sums the block partials in index order.
#include <cmath>
#include <mutex>
#include <set>
#include <utility>

#include "../plan.h"
#include "common.cuh"

namespace pobk {

namespace {

constexpr int kNT = 256;

int reduce_blocks(int64_t m) {
  int64_t b = (m + 4 * kNT - 1) / (4 * kNT);
  if (b < 1) b = 1;
  if (b > kMaxReduceBlocks) b = kMaxReduceBlocks;
  return (int)b;
}

__global__ void k_permute_in(int64_t m, const int32_t* __restrict__ perm, const int32_t* __restrict__ orig,
                             const double* __restrict__ f, const double* __restrict__ x0,
                             const double* __restrict__ xstar, double* __restrict__ fs, double* __restrict__ xt,
                             double* __restrict__ xst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t o = perm[i];
    if (x0) xt[i] = x0[o];
    if (xstar) xst[i] = xstar[o];
    if (f) fs[i] = f[orig[i]];
  }
}

__global__ void k_permute_out(int64_t m, const int32_t* __restrict__ perm, const double* __restrict__ xt,
                              double* __restrict__ x) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    x[perm[i]] = xt[i];
}

// Sum of squares of row residuals over storage rows [b*chunk, (b+1)*chunk) of this block,
// optionally restricted to user-frame rows [lo, hi).  One thread per row, the row's dot product
// in the contract's order (common.cuh), squares accumulated per thread in a fixed order.
__device__ double residual_chunk(int64_t m, const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                 const double* __restrict__ val, const double* __restrict__ fs,
                                 const double* __restrict__ xt, const int32_t* __restrict__ orig, int64_t lo,
                                 int64_t hi) {
  const int64_t chunk = (m + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * chunk, b1 = min(m, b0 + chunk);
  double acc = 0.0;
  for (int64_t s = b0 + threadIdx.x; s < b1; s += blockDim.x) {
    if (orig && (orig[s] < lo || orig[s] >= hi)) continue;
    const double r = __dsub_rn(fs[s], row_dot(col, val, rp[s], rp[s + 1], xt));
    acc = fma(r, r, acc);
  }
  return acc;
}

// The per-sweep stop check (K5, or K4 for RELRES).  Runs as the last node of every K1 sweep and
// after every K2/K3 sweep is NOT needed (those kernels check internally).
__global__ void __launch_bounds__(kNT) k_check(Ctrl* __restrict__ c, int64_t m, const double* __restrict__ xt,
                                               const double* __restrict__ xst, const int32_t* __restrict__ rp,
                                               const int32_t* __restrict__ col, const double* __restrict__ val,
                                               const double* __restrict__ fs, double* __restrict__ partials,
                                               cudaGraphConditionalHandle h, int use_handle) {
  __shared__ double sh[kNT / 32];
  __shared__ int is_last;
  const long long s = c->sweeps + 1;
  const int mode = c->stop_mode;
  const bool do_check = mode != POBK_STOP_NONE && (((s + c->offset) % c->check_every) == 0 || s >= c->max_sweeps);
  double local = 0.0;
  if (do_check) {
    if (mode == POBK_STOP_RSE) {
      const int64_t chunk = (m + gridDim.x - 1) / gridDim.x;
      const int64_t b0 = blockIdx.x * chunk, b1 = min(m, b0 + chunk);
      for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
        const double d = ld_cg(xt + i) - xst[i];
        local = fma(d, d, local);
      }
    } else {
      local = residual_chunk(m, rp, col, val, fs, xt, nullptr, 0, 0);
    }
  }
  const double bs = block_sum<kNT>(local, sh);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = bs;
    __threadfence();
    is_last = (atomicAdd(&c->arrive, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last || threadIdx.x != 0) return;
  __threadfence();
  double tot = 0.0;
  for (int b = 0; b < (int)gridDim.x; b++) tot += ld_cg(partials + b);
  c->arrive = 0;
  c->sweeps = s;
  int stopped = 0;
  if (do_check) {
    const double v = sqrt(tot) / sqrt(c->den);
    c->value = v;
    if (!isfinite(v)) { c->term = POBK_TERM_NONFINITE; stopped = 1; }
    else if (v < c->tol) { c->term = POBK_TERM_CONVERGED; stopped = 1; }
  }
  if (!stopped && s >= c->max_sweeps) { c->term = POBK_TERM_MAX_SWEEPS; stopped = 1; }
  c->stopped = stopped;
  if (stopped && use_handle) cudaGraphSetConditional(h, 0);
}

// den = ||x~*||^2 (RSE) or ||f~||^2 (RELRES); writes c->den.
__global__ void __launch_bounds__(kNT) k_den(Ctrl* __restrict__ c, int64_t m, const double* __restrict__ v,
                                             double* __restrict__ partials) {
  __shared__ double sh[kNT / 32];
  __shared__ int is_last;
  const int64_t chunk = (m + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * chunk, b1 = min(m, b0 + chunk);
  double local = 0.0;
  if (v)
    for (int64_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) local = fma(v[i], v[i], local);
  const double bs = block_sum<kNT>(local, sh);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = bs;
    __threadfence();
    is_last = (atomicAdd(&c->arrive, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last || threadIdx.x != 0) return;
  __threadfence();
  double tot = 0.0;
  for (int b = 0; b < (int)gridDim.x; b++) tot += ld_cg(partials + b);
  c->arrive = 0;
  c->den = tot;
}

__global__ void __launch_bounds__(kNT) k_resid(int64_t m, const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                               const double* __restrict__ val, const double* __restrict__ fs,
                                               const double* __restrict__ xt, const int32_t* __restrict__ orig,
                                               int64_t lo, int64_t hi, double* __restrict__ partials,
                                               unsigned int* __restrict__ arrive, double* __restrict__ out) {
  __shared__ double sh[kNT / 32];
  __shared__ int is_last;
  const double bs = block_sum<kNT>(residual_chunk(m, rp, col, val, fs, xt, orig, lo, hi), sh);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = bs;
    __threadfence();
    is_last = (atomicAdd(arrive, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last || threadIdx.x != 0) return;
  __threadfence();
  double tot = 0.0;
  for (int b = 0; b < (int)gridDim.x; b++) tot += ld_cg(partials + b);
  *arrive = 0;
  *out = tot;
}

int grid_for(int64_t m) {
  int64_t b = (m + kNT - 1) / kNT;
  if (b > 148 * 8) b = 148 * 8;
  return (int)(b < 1 ? 1 : b);
}

}  // namespace

cudaError_t launch_permute_in(const Plan& p, const double* f, const double* x0, const double* xstar, double* fs,
                              double* xt, double* xst, cudaStream_t s, long long& launches) {
  k_permute_in<<<grid_for(p.m), kNT, 0, s>>>(p.m, p.d_perm, p.A.orig, f, x0, xstar, fs, xt, xst);
  launches++;
  return cudaGetLastError();
}

cudaError_t raise_smem_limit(const void* fn) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(mu);
  if (done.count({fn, dev})) return cudaSuccess;
  // the opt-in per-block budget minus the kernel's static shared memory
  int optin = 0;
  cudaFuncAttributes fa;
  if ((e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess ||
      (e = cudaFuncGetAttributes(&fa, fn)) != cudaSuccess)
    return e;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
  if (e == cudaSuccess) done.insert({fn, dev});
  else (void)cudaGetLastError();  // (not sticky: leave no stale error for the caller's next check)
  return e;
}

cudaError_t launch_permute_out(const Plan& p, double* x, cudaStream_t s, long long& launches) {
  k_permute_out<<<grid_for(p.m), kNT, 0, s>>>(p.m, p.d_perm, p.d_xt, x);
  launches++;
  return cudaGetLastError();
}

cudaError_t launch_permute_out_from(const Plan& p, const double* xt, double* x, cudaStream_t s, long long& launches) {
  k_permute_out<<<grid_for(p.m), kNT, 0, s>>>(p.m, p.d_perm, xt, x);
  launches++;
  return cudaGetLastError();
}

cudaError_t launch_den(const Plan& p, Ctrl* c, const double* v, cudaStream_t s, long long& launches) {
  k_den<<<reduce_blocks(p.m), kNT, 0, s>>>(c, p.m, v, p.d_partials);
  launches++;
  return cudaGetLastError();
}

cudaError_t launch_init_ctrl(const Plan& p, const pobk_solve_opts& o, cudaStream_t s, long long& launches) {
  Ctrl* h = p.h_ctrl;
  h->sweeps = 0;
  h->offset = o.sweep_offset;
  h->max_sweeps = o.max_sweeps - o.sweep_offset;  // (this call's cap; checked >= 0 by the caller)
  h->tol = o.tol;
  h->value = NAN;
  h->den = 0.0;
  h->stop_mode = o.stop;
  h->check_every = o.check_every;
  h->stopped = h->max_sweeps <= 0 ? 1 : 0;
  h->term = POBK_TERM_MAX_SWEEPS;
  h->arrive = 0;
  h->pad = 0;
  cudaError_t e = cudaMemcpyAsync(p.d_ctrl, h, sizeof(Ctrl), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  if (o.stop == POBK_STOP_RSE || o.stop == POBK_STOP_RELRES) {
    k_den<<<reduce_blocks(p.m), kNT, 0, s>>>(p.d_ctrl, p.m, o.stop == POBK_STOP_RSE ? p.d_xst : p.d_fs, p.d_partials);
    launches++;
  }
  return cudaGetLastError();
}

cudaError_t launch_check_graph(const Plan& p, cudaStream_t s, cudaGraphConditionalHandle h) {
  k_check<<<reduce_blocks(p.m), kNT, 0, s>>>(p.d_ctrl, p.m, p.d_xt, p.d_xst, p.A.rp, p.A.col, p.A.val, p.d_fs,
                                             p.d_partials, h, 1);
  return cudaGetLastError();
}

cudaError_t launch_check(const Plan& p, cudaStream_t s) {
  k_check<<<reduce_blocks(p.m), kNT, 0, s>>>(p.d_ctrl, p.m, p.d_xt, p.d_xst, p.A.rp, p.A.col, p.A.val, p.d_fs,
                                             p.d_partials, 0, 0);
  return cudaGetLastError();
}

cudaError_t residual_sumsq(const Plan& p, const double* fs, const double* xt, const int32_t* orig, int64_t lo,
                           int64_t hi, cudaStream_t s, double* host_out, long long& launches) {
  // scratch: partials live in d_partials; the arrive counter and the result live in d_ctrl's
  // spare fields of a private Ctrl (the solve's Ctrl is not in use outside a solve)
  unsigned int* arrive = &p.d_ctrl->arrive;
  double* out = &p.d_ctrl->value;
  cudaError_t e = cudaMemsetAsync(arrive, 0, sizeof(unsigned int), s);
  if (e != cudaSuccess) return e;
  const int B = reduce_blocks(p.m);
  k_resid<<<B, kNT, 0, s>>>(p.m, p.A.rp, p.A.col, p.A.val, fs, xt, orig, lo, hi, p.d_partials, arrive, out);
  launches++;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(host_out, out, sizeof(double), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

}  // namespace pobk
