// K3: the whole system resident in one CTA's shared memory (small systems, e.g. BASELINE config 1:
// m = 1024, 4,992 nnz, ~97 KB).  One launch runs every sweep: per schedule step the CTA's
// threads project one row each (Eq 1.2, per the contract in common.cuh),
// __syncthreads() is the step barrier, and after every due sweep a deterministic block reduction
// evaluates the stop rule.  Latency-bound by design: ~nsteps barriers per sweep,
// no global-memory traffic inside the loop.
#include <algorithm>

#include "../plan.h"
#include "common.cuh"

namespace pobk {

namespace {
constexpr int kNT = 1024;

struct K3Args {
  int m, nnz, nsteps, max_overlap_step;
  const int32_t* rp;
  const int32_t* col;
  const double* val;
  const double* nrm2;
  const double* fs;
  const int32_t* step_ptr;  // [nsteps+1]
  const uint8_t* overlap;   // [nsteps]
  double* xt;
  const double* xst;
  Ctrl* ctrl;
};

__host__ __device__ inline size_t align16(size_t b) { return (b + 15) & ~size_t(15); }

__host__ __device__ inline size_t k3_bytes(int m, int nnz, int nsteps, int max_overlap_step) {
  return align16(8ull * nnz) + align16(8ull * m) * 4 /* x, xs, f, nrm2 */ + align16(8ull * max_overlap_step) +
         align16(4ull * nnz) + align16(4ull * (m + 1)) + align16(4ull * (nsteps + 1)) + align16(nsteps) + 64 * 8;
}

__global__ void __launch_bounds__(kNT, 1) k3_sweeps(K3Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* q = smem;
  auto take = [&](size_t b) { unsigned char* r = q; q += align16(b); return r; };
  double* val = (double*)take(8ull * a.nnz);
  double* x = (double*)take(8ull * a.m);
  double* xs = (double*)take(8ull * a.m);
  double* f = (double*)take(8ull * a.m);
  double* nrm2 = (double*)take(8ull * a.m);
  double* alpha = (double*)take(8ull * a.max_overlap_step);
  int32_t* col = (int32_t*)take(4ull * a.nnz);
  int32_t* rp = (int32_t*)take(4ull * (a.m + 1));
  int32_t* sp = (int32_t*)take(4ull * (a.nsteps + 1));
  uint8_t* ov = (uint8_t*)take(a.nsteps);
  double* red = (double*)take(64 * 8);
  __shared__ int s_stop;

  const int tid = threadIdx.x;
  for (int i = tid; i < a.nnz; i += kNT) { val[i] = a.val[i]; col[i] = a.col[i]; }
  for (int i = tid; i < a.m; i += kNT) {
    x[i] = a.xt[i];
    xs[i] = a.xst ? a.xst[i] : 0.0;
    f[i] = a.fs[i];
    nrm2[i] = a.nrm2[i];
  }
  for (int i = tid; i <= a.m; i += kNT) rp[i] = a.rp[i];
  for (int i = tid; i <= a.nsteps; i += kNT) sp[i] = a.step_ptr[i];
  for (int i = tid; i < a.nsteps; i += kNT) ov[i] = a.overlap[i];
  const long long maxs = a.ctrl->max_sweeps;
  const int mode = a.ctrl->stop_mode, every = a.ctrl->check_every;
  const double tol = a.ctrl->tol, den = a.ctrl->den;
  if (tid == 0) s_stop = maxs <= 0;
  __syncthreads();

  long long sweep = 0;
  double value = NAN;
  int term = POBK_TERM_MAX_SWEEPS;
  while (!s_stop) {
    for (int k = 0; k < a.nsteps; k++) {
      const int s0 = sp[k], s1 = sp[k + 1];
      if (!ov[k]) {
        for (int s = s0 + tid; s < s1; s += kNT) row_project(col, val, rp[s], rp[s + 1], f[s], nrm2[s], x);
      } else {
        for (int s = s0 + tid; s < s1; s += kNT)
          alpha[s - s0] = __ddiv_rn(__dsub_rn(f[s], row_dot(col, val, rp[s], rp[s + 1], x)), nrm2[s]);
        __syncthreads();
        for (int s = s0 + tid; s < s1; s += kNT)
          for (int p = rp[s]; p < rp[s + 1]; p++) atomicAdd(x + col[p], __dmul_rn(alpha[s - s0], val[p]));
      }
      __syncthreads();
    }
    sweep++;
    const bool due = mode != POBK_STOP_NONE && ((sweep % every) == 0 || sweep >= maxs);
    if (due) {
      double loc = 0.0;
      if (mode == POBK_STOP_RSE) {
        for (int i = tid; i < a.m; i += kNT) { const double d = x[i] - xs[i]; loc = fma(d, d, loc); }
      } else {
        for (int s = tid; s < a.m; s += kNT) {
          const double r = __dsub_rn(f[s], row_dot(col, val, rp[s], rp[s + 1], x));
          loc = fma(r, r, loc);
        }
      }
      const double tot = block_sum<kNT>(loc, red);
      if (tid == 0) {
        value = sqrt(tot) / sqrt(den);
        if (!isfinite(value)) { term = POBK_TERM_NONFINITE; s_stop = 1; }
        else if (value < tol) { term = POBK_TERM_CONVERGED; s_stop = 1; }
      }
    }
    if (tid == 0 && !s_stop && sweep >= maxs) { term = POBK_TERM_MAX_SWEEPS; s_stop = 1; }
    __syncthreads();
  }
  for (int i = tid; i < a.m; i += kNT) a.xt[i] = x[i];
  if (tid == 0) {
    a.ctrl->sweeps = sweep;
    a.ctrl->value = value;
    a.ctrl->term = term;
    a.ctrl->stopped = 1;
  }
}

int max_overlap_step(const Plan& p) {
  int mx = 0;
  for (int k = 0; k < p.nsteps; k++)
    if (p.h_overlap[k]) mx = std::max(mx, p.h_step_ptr[k + 1] - p.h_step_ptr[k]);
  return mx;
}

cudaError_t launch(Plan& p, cudaStream_t s) {
  K3Args a;
  a.m = (int)p.m;
  a.nnz = (int)p.nnz;
  a.nsteps = p.nsteps;
  a.max_overlap_step = max_overlap_step(p);
  a.rp = p.A.rp;
  a.col = p.A.col;
  a.val = p.A.val;
  a.nrm2 = p.A.nrm2;
  a.fs = p.d_fs;
  a.step_ptr = p.k3_step_ptr;
  a.overlap = p.k3_overlap;
  a.xt = p.d_xt;
  a.xst = p.d_xst;
  a.ctrl = p.d_ctrl;
  cudaError_t e = cudaFuncSetAttribute(k3_sweeps, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.k3_smem);
  if (e != cudaSuccess) return e;
  k3_sweeps<<<1, kNT, p.k3_smem, s>>>(a);
  return cudaGetLastError();
}
}  // namespace

bool k3_fits(const Plan& p, size_t& bytes) {
  if (p.m > (1 << 20) || p.nnz > (1 << 24)) return false;
  bytes = k3_bytes((int)p.m, (int)p.nnz, p.nsteps, max_overlap_step(p));
  return bytes <= 227 * 1024 - 256;  // sm_100 opt-in limit 232,448 B per CTA minus static smem
}

cudaError_t k3_solve(Plan& p, cudaStream_t s, long long& launches) {
  launches++;
  return launch(p, s);
}

}  // namespace pobk
