// K3: the whole system resident in one CTA's shared memory (small systems, e.g. BASELINE config 1:
// m = 1024, 4,992 nnz, ~97 KB).  One launch runs every sweep: per schedule step the CTA's
// threads project one row each (Eq 1.2, per the contract in common.cuh),
// __syncthreads() is the step barrier, and after every due sweep a deterministic block reduction
// evaluates the stop rule.  Latency-bound by design: ~nsteps barriers per sweep,
// no global-memory traffic inside the loop.
#include <algorithm>
#include <type_traits>
#include <vector>

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
  // overlapping steps: entries by column (plan.h ov_*), the ordered scatter; atomic: fp64 atomics
  const int32_t *ov_colptr, *ov_cols, *ov_eptr, *ov_es;
  const double* ov_ev;
  int atomic;
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
  const long long off = a.ctrl->offset;
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
        if (a.atomic) {
          for (int s = s0 + tid; s < s1; s += kNT)
            for (int p = rp[s]; p < rp[s + 1]; p++) atomicAdd(x + col[p], __dmul_rn(alpha[s - s0], val[p]));
        } else {  // one thread per column: the step's contributions in ascending row order (the oracle's)
          for (int t = a.ov_colptr[k] + tid; t < a.ov_colptr[k + 1]; t += kNT) {
            const int c = a.ov_cols[t];
            double xc = x[c];
            for (int e = a.ov_eptr[t]; e < a.ov_eptr[t + 1]; e++) xc = __dadd_rn(xc, __dmul_rn(alpha[a.ov_es[e]], a.ov_ev[e]));
            x[c] = xc;
          }
        }
      }
      __syncthreads();
    }
    sweep++;
    const bool due = mode != POBK_STOP_NONE && (((sweep + off) % every) == 0 || sweep >= maxs);
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

// ---------------------------------------------------------------------------------------------
// K3E: the same one-CTA solver with the matrix in a thread-major ELL layout (thr = 0 systems whose
// rows have <= kEW entries).  Per step each thread owns one row per round: its kEW columns and
// values sit at e = base + j*kENT + t (coalesced, conflict-free), so every operand load of a row is
// issued at once, the x~ gathers follow in one batch, and the row sum is the oracle's left-to-right
// chain (common.cuh contract: bitwise the oracle's iterates).  Padding entries are value +0 on the
// zero slot x~[m] = +0: adding +0 * +0 to a sum that starts at +0 changes no bit.
constexpr int kENT = 256;  // threads
constexpr int kEW = 16;    // max entries per row held in registers

struct K3EArgs {
  int m, nsteps, nent;
  const int32_t* ecol;      // [nent] ELL columns (RCM frame; m = zero slot)
  const double* eval;       // [nent] ELL values
  const int32_t* einfo;     // [nsteps*4]: {first schedule position, rows, W, ELL base}
  const double* nrm2;       // [m] storage order
  const double* fs;         // [m] storage order
  double* xt;
  const double* xst;
  Ctrl* ctrl;
};

size_t k3e_bytes(int m, int nent, int nsteps) {
  return align16(8ull * nent) + align16(4ull * nent) + align16(8ull * (m + 1)) + 4 * align16(8ull * m) +
         align16(16ull * nsteps) + 64 * 8;
}

// One row of K3E: entries j < EW at e0 + j*kENT; entries j >= W are padding (the zero slot m,
// value +0) selected without branches, so all operand loads of the row issue back to back.
template <int EW>
__device__ __forceinline__ void k3e_row(const int32_t* col, const double* val, double* x, int e0, int W, double fi,
                                        double ni, double yi, int m) {
  int c[EW];
  double av[EW], xv[EW];
#pragma unroll
  for (int j = 0; j < EW; j++) {
    const int jj = j < W ? j : W - 1;
    const int cj = col[e0 + jj * kENT];
    const double aj = val[e0 + jj * kENT];
    c[j] = j < W ? cj : m;
    av[j] = j < W ? aj : 0.0;
  }
#pragma unroll
  for (int j = 0; j < EW; j++) xv[j] = x[c[j]];
  double sum = 0.0, pp[EW];
#pragma unroll
  for (int j = 0; j < EW; j++) pp[j] = pin(__dmul_rn(av[j], xv[j]));  // products first (common.cuh)
#pragma unroll
  for (int j = 0; j < EW; j++) sum = __dadd_rn(sum, pp[j]);  // (+0 * +0 past W: no-ops)
  const double alpha = div_by_rcp(__dsub_rn(fi, sum), ni, yi);  // (= __ddiv_rn: common.cuh)
#pragma unroll
  for (int j = 0; j < EW; j++)
    if (c[j] < m) x[c[j]] = __dadd_rn(xv[j], __dmul_rn(alpha, av[j]));
}

__global__ void __launch_bounds__(kENT, 1) k3e_sweeps(K3EArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* q = smem;
  auto take = [&](size_t b) { unsigned char* r = q; q += align16(b); return r; };
  double* val = (double*)take(8ull * a.nent);
  int32_t* col = (int32_t*)take(4ull * a.nent);
  double* x = (double*)take(8ull * (a.m + 1));
  double* xs = (double*)take(8ull * a.m);
  double* f = (double*)take(8ull * a.m);
  double* nrm2 = (double*)take(8ull * a.m);
  double* rn = (double*)take(8ull * a.m);  // RN(1/nrm2): the division's reciprocal, formed once
  int4* info = (int4*)take(16ull * a.nsteps);
  double* red = (double*)take(64 * 8);

  const int tid = threadIdx.x;
  for (int i = tid; i < a.nent; i += kENT) { val[i] = a.eval[i]; col[i] = a.ecol[i]; }
  for (int i = tid; i < a.m; i += kENT) {
    x[i] = a.xt[i];
    xs[i] = a.xst ? a.xst[i] : 0.0;
    f[i] = a.fs[i];
    nrm2[i] = a.nrm2[i];
    rn[i] = rcp_ahead(a.nrm2[i]);
  }
  for (int i = tid; i < a.nsteps; i += kENT) info[i] = ((const int4*)a.einfo)[i];
  if (tid == 0) x[a.m] = 0.0;  // the zero slot of the ELL padding (never written)
  const long long maxs = a.ctrl->max_sweeps;
  const int mode = a.ctrl->stop_mode, every = a.ctrl->check_every;
  const long long off = a.ctrl->offset;
  const double tol = a.ctrl->tol, den = a.ctrl->den;
  __syncthreads();
  // stop test value = sqrt(tot)/sqrt(den) < tol; above cut_hi it cannot hold
  // (margin >> rounding), so the exact value is formed only near the threshold or at the end
  const double sd = sqrt(den), cut_hi = (den > 0.0 && isfinite(den)) ? (tol * sd) * (tol * sd) * (1.0 + 1e-6) : -1.0;
  long long sweep = 0;
  double value = NAN;
  int term = POBK_TERM_MAX_SWEEPS;
  bool stop = maxs <= 0;
  while (!stop) {
    for (int k = 0; k < a.nsteps; k++) {
      const int4 in = info[k];  // {schedule position, rows, W, ELL base}
      for (int r0 = 0; r0 < in.y; r0 += kENT) {
        const int rr = r0 + tid;
        if (rr < in.y) {
          const int sidx = in.x + rr, W = in.z;
          const int e0 = in.w + (r0 / kENT) * W * kENT + tid;
          if (W <= 8) k3e_row<8>(col, val, x, e0, W, f[sidx], nrm2[sidx], rn[sidx], a.m);
          else k3e_row<kEW>(col, val, x, e0, W, f[sidx], nrm2[sidx], rn[sidx], a.m);
        }
      }
      __syncthreads();
    }
    sweep++;
    const bool due = mode != POBK_STOP_NONE && (((sweep + off) % every) == 0 || sweep >= maxs);
    if (due) {
      double loc = 0.0;
      if (mode == POBK_STOP_RSE) {
        for (int i = tid; i < a.m; i += kENT) { const double d = x[i] - xs[i]; loc = fma(d, d, loc); }
      } else {  // RELRES: ||f~ - A~ x~||^2, row by row from the ELL
        for (int k = 0; k < a.nsteps; k++) {
          const int4 in = info[k];
          for (int rr = tid; rr < in.y; rr += kENT) {
            const int e0 = in.w + (rr / kENT) * in.z * kENT + (rr % kENT);
            double sum = 0.0;
            for (int j = 0; j < in.z; j++) sum = __dadd_rn(sum, __dmul_rn(val[e0 + j * kENT], x[col[e0 + j * kENT]]));
            const double r = __dsub_rn(f[in.x + rr], sum);
            loc = fma(r, r, loc);
          }
        }
      }
      // every thread forms the same total (fixed order: warp butterflies, then the 8 warp sums in
      // order) and takes the stop decision itself: no broadcast barrier.  `red` is next written a
      // whole sweep (nsteps barriers) later.
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) loc += __shfl_xor_sync(0xffffffffu, loc, o);
      if ((tid & 31) == 0) red[tid >> 5] = loc;
      __syncthreads();
      double tot = 0.0;
#pragma unroll
      for (int w = 0; w < kENT / 32; w++) tot += red[w];
      // value = sqrt(tot)/sqrt(den) < tol, evaluated exactly only near the threshold
      // or when the loop ends
      if (!(tot > cut_hi) || !isfinite(tot) || sweep >= maxs) {
        value = sqrt(tot) / sd;
        if (!isfinite(value)) { term = POBK_TERM_NONFINITE; stop = true; }
        else if (value < tol) { term = POBK_TERM_CONVERGED; stop = true; }
      }
    }
    if (!stop && sweep >= maxs) { term = POBK_TERM_MAX_SWEEPS; stop = true; }
  }
  for (int i = tid; i < a.m; i += kENT) a.xt[i] = x[i];
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

cudaError_t launch_e(Plan& p, cudaStream_t s) {
  K3EArgs a;
  a.m = (int)p.m;
  a.nsteps = p.nsteps;
  a.nent = p.k3e_nent;
  a.ecol = p.k3e_col;
  a.eval = p.k3e_val;
  a.einfo = p.k3e_info;
  a.nrm2 = p.A.nrm2;
  a.fs = p.d_fs;
  a.xt = p.d_xt;
  a.xst = p.d_xst;
  a.ctrl = p.d_ctrl;
  cudaError_t e = raise_smem_limit((const void*)k3e_sweeps);
  if (e != cudaSuccess) return e;
  k3e_sweeps<<<1, kENT, p.k3_smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch(Plan& p, cudaStream_t s) {
  if (p.k3e_col) return launch_e(p, s);
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
  a.ov_colptr = p.ov_colptr;
  a.ov_cols = p.ov_cols;
  a.ov_eptr = p.ov_eptr;
  a.ov_es = p.ov_es;
  a.ov_ev = p.ov_ev;
  a.atomic = getenv("POBK_THR_ATOMIC") != nullptr;
  a.xt = p.d_xt;
  a.xst = p.d_xst;
  a.ctrl = p.d_ctrl;
  cudaError_t e = raise_smem_limit((const void*)k3_sweeps);
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

// The K3E layout (when the system has no overlapping step, every row has <= kEW entries and the
// ELL fits): schedule-order CSR in, ELL blocks per step out; *bytes = the kernel's shared memory.
cudaError_t k3e_build(Plan& p, const std::vector<int32_t>& rp, const std::vector<int32_t>& col,
                      const std::vector<double>& val, size_t* bytes, bool* built) {
  *built = false;
  if (p.any_overlap || p.m >= (1 << 24)) return cudaSuccess;
  std::vector<int32_t> info(4 * (size_t)p.nsteps);
  int64_t nent = 0;
  for (int k = 0; k < p.nsteps; k++) {
    const int s0 = p.h_step_ptr[k], s1 = p.h_step_ptr[k + 1];
    int W = 1;
    for (int s = s0; s < s1; s++) W = std::max(W, rp[s + 1] - rp[s]);
    if (W > kEW) return cudaSuccess;
    const int rounds = (s1 - s0 + kENT - 1) / kENT;
    info[4 * k + 0] = s0;
    info[4 * k + 1] = s1 - s0;
    info[4 * k + 2] = W;
    info[4 * k + 3] = (int32_t)nent;
    nent += (int64_t)rounds * W * kENT;
    if (nent > (1 << 24)) return cudaSuccess;
  }
  const size_t b = k3e_bytes((int)p.m, (int)nent, p.nsteps);
  if (b > 227 * 1024 - 256) return cudaSuccess;
  std::vector<int32_t> ecol(std::max<int64_t>(nent, 1), (int32_t)p.m);
  std::vector<double> eval(std::max<int64_t>(nent, 1), 0.0);
  for (int k = 0; k < p.nsteps; k++) {
    const int s0 = info[4 * k], n = info[4 * k + 1], W = info[4 * k + 2], base = info[4 * k + 3];
    for (int rr = 0; rr < n; rr++) {
      const int s = s0 + rr, e0 = base + (rr / kENT) * W * kENT + rr % kENT;
      for (int j = 0; j < rp[s + 1] - rp[s]; j++) {
        ecol[e0 + (size_t)j * kENT] = col[rp[s] + j];
        eval[e0 + (size_t)j * kENT] = val[rp[s] + j];
      }
    }
  }
  cudaError_t e;
  auto up = [&](auto** dst, const auto* src, size_t n) -> cudaError_t {
    void* v = nullptr;
    cudaError_t r = cudaMalloc(&v, n * sizeof(*src));
    if (r != cudaSuccess) return r;
    p.allocations.push_back(v);
    *dst = (std::remove_reference_t<decltype(**dst)>*)v;
    return cudaMemcpy(v, src, n * sizeof(*src), cudaMemcpyHostToDevice);
  };
  if ((e = up(&p.k3e_col, ecol.data(), ecol.size())) != cudaSuccess) return e;
  if ((e = up(&p.k3e_val, eval.data(), eval.size())) != cudaSuccess) return e;
  if ((e = up(&p.k3e_info, info.data(), info.size())) != cudaSuccess) return e;
  p.k3e_nent = (int)nent;
  *bytes = b;
  *built = true;
  return cudaSuccess;
}

cudaError_t k3_solve(Plan& p, cudaStream_t s, long long& launches) {
  launches++;
  return launch(p, s);
}

}  // namespace pobk
