// The C ABI of libpobk.so (include/pobk.h): argument checking, plan construction (host
// preprocessing + device layout), solve orchestration and reports.  No C++ exception crosses
// the ABI; every failure becomes a pobk_status plus a thread-local message.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "plan.h"

namespace pobk {
namespace {

thread_local std::string g_err;

pobk_status fail(pobk_status code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) return fail(POBK_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  bool ok = false;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && cudaSetDevice(dev) == cudaSuccess) ok = true;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <typename T>
cudaError_t dalloc(Plan& p, T** ptr, size_t count) {
  void* v = nullptr;
  cudaError_t e = cudaMalloc(&v, std::max<size_t>(count, 1) * sizeof(T));
  if (e == cudaSuccess) {
    p.allocations.push_back(v);
    *ptr = (T*)v;
  }
  return e;
}

template <typename T>
cudaError_t upload(Plan& p, T** ptr, const T* src, size_t count) {
  cudaError_t e = dalloc(p, ptr, count);
  if (e == cudaSuccess && count) e = cudaMemcpy(*ptr, src, count * sizeof(T), cudaMemcpyHostToDevice);
  return e;
}

void destroy_plan(Plan* p) {
  if (!p) return;
  if (p->device >= 0) {
    DeviceGuard g(p->device);
    if (p->k2) k2_free(*p);
    if (p->k2r) k2r_free(*p);
    if (p->k4) k4_free(*p);
    if (p->k5) k5_free(*p);
    if (p->multi) k1m_free(*p);
    if (p->k1_exec) cudaGraphExecDestroy(p->k1_exec);
    if (p->k1_graph) cudaGraphDestroy(p->k1_graph);
    if (p->k1o_exec) cudaGraphExecDestroy(p->k1o_exec);
    if (p->k1o_graph) cudaGraphDestroy(p->k1o_graph);
    for (void* a : p->allocations) cudaFree(a);
    if (p->h_ctrl) cudaFreeHost(p->h_ctrl);
    for (auto& e : p->ev)
      if (e) cudaEventDestroy(e);
  }
  delete static_cast<pobk_plan_s*>(p);
}

pobk_status build_device(Plan& p, const HostCSR& At, const std::vector<double>& nrm2, int tile_rows) {
  p.k2_tile_rows = tile_rows;
  DeviceGuard g(p.device);
  if (!g.ok) return fail(POBK_ERR_CUDA, "cudaSetDevice(" + std::to_string(p.device) + ") failed");
  const int64_t m = p.m;
  // schedule-order (step-major) CSR
  std::vector<int32_t> rp(m + 1), col(p.nnz), orig(m);
  std::vector<double> val(p.nnz), nrm2_s(m);
  rp[0] = 0;
  for (int64_t s = 0; s < m; s++) {
    const int32_t r = p.sched.rows[s];
    const int64_t b = At.ptr[r], len = At.ptr[r + 1] - b;
    std::memcpy(col.data() + rp[s], At.col.data() + b, len * sizeof(int32_t));
    std::memcpy(val.data() + rp[s], At.val.data() + b, len * sizeof(double));
    rp[s + 1] = rp[s] + (int32_t)len;
    nrm2_s[s] = nrm2[r];
    orig[s] = p.perm[r];
  }
  CUDA_TRY(upload(p, &p.A.rp, rp.data(), m + 1));
  CUDA_TRY(upload(p, &p.A.col, col.data(), p.nnz));
  CUDA_TRY(upload(p, &p.A.val, val.data(), p.nnz));
  CUDA_TRY(upload(p, &p.A.nrm2, nrm2_s.data(), m));
  CUDA_TRY(upload(p, &p.A.orig, orig.data(), m));
  CUDA_TRY(upload(p, &p.d_perm, p.perm.data(), m));
  p.h_step_ptr = p.sched.step_ptr;
  p.h_overlap = p.sched.overlap;
  CUDA_TRY(upload(p, &p.k3_step_ptr, p.h_step_ptr.data(), p.h_step_ptr.size()));
  CUDA_TRY(upload(p, &p.k3_overlap, p.h_overlap.data(), p.h_overlap.size()));
  int32_t max_step = 0;
  for (int32_t k = 0; k < p.nsteps; k++) max_step = std::max(max_step, p.h_step_ptr[k + 1] - p.h_step_ptr[k]);
  CUDA_TRY(dalloc(p, &p.d_xt, m));
  CUDA_TRY(dalloc(p, &p.d_xst, m));
  CUDA_TRY(dalloc(p, &p.d_fs, m));
  CUDA_TRY(dalloc(p, &p.d_alpha, p.any_overlap ? max_step : 1));
  if (p.any_overlap) {  // per overlapping step, its entries by column (ascending schedule position)
    std::vector<int32_t> cols, eptr(1, 0), es;
    std::vector<double> ev;
    std::vector<int32_t> cnt(m, 0), first(m, -1);
    p.h_ov_colptr.assign(p.nsteps + 1, 0);
    for (int32_t k = 0; k < p.nsteps; k++) {
      p.h_ov_colptr[k] = (int32_t)cols.size();
      if (!p.h_overlap[k]) continue;
      const int32_t s0 = p.h_step_ptr[k], s1 = p.h_step_ptr[k + 1];
      const size_t c0 = cols.size();
      for (int32_t s = s0; s < s1; s++)
        for (int32_t q = rp[s]; q < rp[s + 1]; q++) {
          const int32_t c = col[q];
          if (cnt[c]++ == 0) cols.push_back(c);
        }
      const size_t e0 = es.size();
      for (size_t t = c0; t < cols.size(); t++) {  // offsets (entries of the step's columns, in cols order)
        first[cols[t]] = (int32_t)(eptr.back());
        eptr.push_back(eptr.back() + cnt[cols[t]]);
      }
      es.resize(e0 + (size_t)(eptr.back() - (int32_t)e0));
      ev.resize(es.size());
      for (int32_t s = s0; s < s1; s++)  // ascending s: each column's entries in schedule order
        for (int32_t q = rp[s]; q < rp[s + 1]; q++) {
          const int32_t c = col[q];
          es[first[c]] = s - s0;
          ev[first[c]++] = val[q];
        }
      for (size_t t = c0; t < cols.size(); t++) cnt[cols[t]] = 0;
    }
    p.h_ov_colptr[p.nsteps] = (int32_t)cols.size();
    CUDA_TRY(upload(p, &p.ov_colptr, p.h_ov_colptr.data(), p.h_ov_colptr.size()));
    CUDA_TRY(upload(p, &p.ov_cols, cols.data(), std::max<size_t>(cols.size(), 1)));
    CUDA_TRY(upload(p, &p.ov_eptr, eptr.data(), eptr.size()));
    CUDA_TRY(upload(p, &p.ov_es, es.data(), std::max<size_t>(es.size(), 1)));
    CUDA_TRY(upload(p, &p.ov_ev, ev.data(), std::max<size_t>(ev.size(), 1)));
  }
  CUDA_TRY(dalloc(p, &p.d_partials, kMaxReduceBlocks));
  CUDA_TRY(dalloc(p, &p.d_ctrl, 1));
  CUDA_TRY(cudaMemset(p.d_ctrl, 0, sizeof(Ctrl)));
  CUDA_TRY(cudaMallocHost(&p.h_ctrl, sizeof(Ctrl)));
  for (auto& e : p.ev) CUDA_TRY(cudaEventCreate(&e));

  // kernel family: K3 when everything fits one CTA's shared memory, else the K2
  // wavefront when its tiling is valid (m >= 4096: measured faster than K1's launch per step
  // from config 2, 20k rows, upwards), else K1.  Overlapping categories (thr > 0) use K1/K3.
  const int req = p.kernel;
  size_t k3b = 0;
  const bool k3ok = k3_fits(p, k3b);
  if (k3ok) p.k3_smem = k3b;
  std::string why;
  if (k3ok && (req == POBK_KERNEL_SMEM || req == POBK_KERNEL_AUTO) && !getenv("POBK_NO_K3E")) {
    size_t eb = 0;
    bool built = false;
    CUDA_TRY(k3e_build(p, rp, col, val, &eb, &built));
    if (built) p.k3_smem = eb;
  }
  if (req == POBK_KERNEL_SMEM) {
    if (!k3ok) return fail(POBK_ERR_ARG, "kernel=SMEM requested but the system needs " + std::to_string(k3b) + " B of shared memory");
  } else if (req == POBK_KERNEL_WAVEFRONT) {
    if (p.any_overlap) return fail(POBK_ERR_ARG, "kernel=WAVEFRONT does not support overlapping categories (thr > 0)");
    if (!k2_build(p, At, nrm2, tile_rows, why)) return fail(POBK_ERR_ARG, "kernel=WAVEFRONT unavailable: " + why);
  } else if (req == POBK_KERNEL_CLUSTER) {
    if (!k4_build(p, rp, col, val, why)) return fail(POBK_ERR_ARG, "kernel=CLUSTER unavailable: " + why);
  } else if (req == POBK_KERNEL_BLOCKS) {  // the k-block variant: Gram inverses + K5 layout
    std::vector<std::vector<double>> ginv;
    Error err;
    if (!block_gram_inverses(At, p.blocks_host, ginv, err)) return fail(err.code, err.msg);
    if (!k5_build(p, At, std::move(p.blocks_host), std::move(ginv), why)) return fail(POBK_ERR_CUDA, why);
    p.blocks_host = BlockLayout();
  } else if (req == POBK_KERNEL_AUTO) {
    // K3 (one CTA) when the system fits one CTA's shared memory, else the K2 wavefront from
    // m >= 4096, else K1 (K4, one cluster, is explicit-only: slower than K2 where both apply)
    if (k3ok) p.kernel = POBK_KERNEL_SMEM;
    else if (!p.any_overlap && m >= 4096 && k2_build(p, At, nrm2, tile_rows, why)) p.kernel = POBK_KERNEL_WAVEFRONT;
    else p.kernel = POBK_KERNEL_LAUNCH;
  }
  return POBK_OK;
}

pobk_status solve_finish(Plan& p, const pobk_solve_opts& o, pobk_report* rep);

pobk_status solve_device(Plan& p, const double* f, double* x, const double* xstar, const pobk_solve_opts& o,
                         cudaStream_t s, pobk_report* rep, bool defer = false) {
  long long launches = 0;
  CUDA_TRY(cudaEventRecord(p.ev[0], s));
  CUDA_TRY(launch_permute_in(p, f, x, xstar, p.d_fs, p.d_xt, o.stop == POBK_STOP_RSE ? p.d_xst : nullptr, s, launches));
  CUDA_TRY(launch_init_ctrl(p, o, s, launches));
  CUDA_TRY(cudaEventRecord(p.ev[1], s));
  // K2 evaluates RSE, RELRES (a residual pass over each tile's stream) and fixed counts in-kernel;
  // plans with vector boundary slices (opt-in) take RELRES on the K1 graph loop.
  int used = p.kernel;
  if (used == POBK_KERNEL_WAVEFRONT && o.stop == POBK_STOP_RELRES && !k2_relres_ok(p)) used = POBK_KERNEL_LAUNCH;
  const bool ordered = o.order == POBK_ORDER_RESIDUAL;
  if (ordered) used = POBK_KERNEL_LAUNCH;
  if (o.max_sweeps - o.sweep_offset > 0) {
    switch (used) {
      case POBK_KERNEL_SMEM: CUDA_TRY(k3_solve(p, s, launches)); break;
      case POBK_KERNEL_WAVEFRONT: CUDA_TRY(k2_solve(p, f, s, launches)); break;
      case POBK_KERNEL_CLUSTER: CUDA_TRY(k4_solve(p, s, launches)); break;
      case POBK_KERNEL_BLOCKS: CUDA_TRY(k5_solve(p, s, launches)); break;
      default:
        if (ordered) CUDA_TRY(k1_solve_ordered(p, s, launches));
        else CUDA_TRY(k1_solve(p, s, launches));
        break;
    }
  }
  CUDA_TRY(cudaEventRecord(p.ev[2], s));
  CUDA_TRY(launch_permute_out(p, x, s, launches));
  CUDA_TRY(cudaEventRecord(p.ev[3], s));
  CUDA_TRY(cudaMemcpyAsync(p.h_ctrl, p.d_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
  p.pending_launches = launches;
  p.pending_used = used;
  if (defer) return POBK_OK;  // (batch: the caller synchronises, then solve_finish)
  CUDA_TRY(cudaStreamSynchronize(s));
  return solve_finish(p, o, rep);
}

// the report of a solve enqueued by solve_device (its stream synchronised)
pobk_status solve_finish(Plan& p, const pobk_solve_opts& o, pobk_report* rep) {
  long long launches = p.pending_launches;
  const int used = p.pending_used;
  float t_all = 0.f, t_sw = 0.f;
  CUDA_TRY(cudaEventElapsedTime(&t_all, p.ev[0], p.ev[3]));
  CUDA_TRY(cudaEventElapsedTime(&t_sw, p.ev[1], p.ev[2]));
  const Ctrl& c = *p.h_ctrl;
  const bool ran = o.max_sweeps - o.sweep_offset > 0;
  if (used == POBK_KERNEL_LAUNCH && ran) launches += c.sweeps * (o.order == POBK_ORDER_RESIDUAL ? p.k1o_nodes_per_sweep : p.k1_nodes_per_sweep);
  if (used == POBK_KERNEL_BLOCKS && ran) launches += c.sweeps * k5_nodes_per_sweep(p);
  if (rep) {
    rep->sweeps = ran ? c.sweeps : 0;
    rep->termination = c.term;
    rep->kernel = used;
    rep->final_value = (o.stop == POBK_STOP_NONE) ? NAN : c.value;
    rep->sweeps_total = o.sweep_offset + rep->sweeps;
    rep->final_rse = o.stop == POBK_STOP_RSE ? rep->final_value : NAN;
    rep->final_relres = o.stop == POBK_STOP_RELRES ? rep->final_value : NAN;
    rep->solve_seconds = t_all * 1e-3;
    rep->sweep_seconds = t_sw * 1e-3;
    rep->launches = launches;
  }
  return POBK_OK;
}

pobk_status check_solve_args(pobk_plan_t plan, const void* f, const void* x, const void* xstar, pobk_solve_opts& o,
                             const pobk_solve_opts* opts) {
  if (!plan) return fail(POBK_ERR_ARG, "plan is NULL");
  if (plan->device < 0) return fail(POBK_ERR_NO_DEVICE, "plan was built with device = -1 (host-only)");
  if (!f || !x) return fail(POBK_ERR_ARG, "f and x must be non-NULL");
  pobk_solve_opts_default(&o);
  if (opts) o = *opts;
  if (o.stop < POBK_STOP_RSE || o.stop > POBK_STOP_NONE) return fail(POBK_ERR_ARG, "opts.stop out of range");
  if (o.stop == POBK_STOP_RSE && !xstar) return fail(POBK_ERR_ARG, "POBK_STOP_RSE needs xstar");
  if (o.check_every < 1) return fail(POBK_ERR_ARG, "opts.check_every must be >= 1");
  if (o.max_sweeps < 0) return fail(POBK_ERR_ARG, "opts.max_sweeps must be >= 0");
  if (o.sweep_offset < 0) return fail(POBK_ERR_ARG, "opts.sweep_offset must be >= 0");
  if (o.order != POBK_ORDER_SCHEDULE && o.order != POBK_ORDER_RESIDUAL) return fail(POBK_ERR_ARG, "opts.order out of range");
  if (o.order == POBK_ORDER_RESIDUAL && (plan->any_overlap || plan->kernel == POBK_KERNEL_BLOCKS))
    return fail(POBK_ERR_ARG, "the residual order needs a row-level plan with thr = 0");
  if (!(o.tol >= 0.0)) return fail(POBK_ERR_ARG, "opts.tol must be >= 0");
  return POBK_OK;
}

}  // namespace
}  // namespace pobk

using namespace pobk;

extern "C" {

void pobk_preprocess_opts_default(pobk_preprocess_opts* o) {
  if (!o) return;
  o->thr = 0.0;
  o->reorder = 1;
  o->kernel = POBK_KERNEL_AUTO;
  o->tile_rows = 0;
  o->guard = 0;
}

void pobk_solve_opts_default(pobk_solve_opts* o) {
  if (!o) return;
  o->tol = 1e-6;
  o->max_sweeps = 500000;
  o->stop = POBK_STOP_RSE;
  o->check_every = 1;
  o->sweep_offset = 0;
  o->order = POBK_ORDER_SCHEDULE;
}

int32_t pobk_abi_version(void) { return POBK_ABI_VERSION; }

const char* pobk_last_error(void) { return g_err.c_str(); }

pobk_status pobk_preprocess(int64_t m, const int64_t* row_ptr, const int32_t* col, const double* val,
                            const pobk_preprocess_opts* opts, int device, pobk_plan_t* out) {
  g_err.clear();
  if (!out) return fail(POBK_ERR_ARG, "out is NULL");
  *out = nullptr;
  pobk_preprocess_opts o;
  pobk_preprocess_opts_default(&o);
  if (opts) o = *opts;
  if (!(o.thr >= 0.0 && o.thr < 1.0)) return fail(POBK_ERR_ARG, "opts.thr must be in [0, 1)");
  if (o.kernel < POBK_KERNEL_AUTO || o.kernel > POBK_KERNEL_CLUSTER) return fail(POBK_ERR_ARG, "opts.kernel out of range");
  if (device < -1) return fail(POBK_ERR_ARG, "device must be >= -1");
  try {
    auto t0 = std::chrono::steady_clock::now();
    HostCSR A;
    Error err;
    if (!canonicalize(m, row_ptr, col, val, A, err)) return fail(err.code, err.msg);
    Plan* p = new pobk_plan_s();
    p->device = device;
    p->m = m;
    p->nnz = A.nnz();
    p->thr = o.thr;
    p->kernel = o.kernel;
    p->bw_before = bandwidth(A);
    if (o.reorder) rcm_order(A, p->perm);
    else {
      p->perm.resize(m);
      for (int64_t i = 0; i < m; i++) p->perm[i] = (int32_t)i;
    }
    HostCSR At;
    permute_symmetric(A, p->perm, At);
    { HostCSR().ptr.swap(A.ptr); std::vector<int32_t>().swap(A.col); std::vector<double>().swap(A.val); }
    p->bw_after = bandwidth(At);
    std::vector<double> nrm2;
    row_sqnorms(At, nrm2);
    first_fit_colour(At, nrm2, o.thr, p->colour);
    build_schedule(At, p->colour, o.thr > 0.0, p->sched);
    p->nsteps = (int32_t)p->sched.step_ptr.size() - 1;
    p->n_oclass = p->sched.n_oclass;
    for (uint8_t v : p->sched.overlap) p->any_overlap |= (v != 0);
    if (o.thr > 0.0 && o.guard) {
      std::string why;
      if (!gershgorin_guard(At, nrm2, p->colour, why)) {
        destroy_plan(p);
        return fail(POBK_ERR_UNSTABLE_THR, why);
      }
    }
    if (device >= 0) {
      pobk_status st = build_device(*p, At, nrm2, o.tile_rows);
      if (st != POBK_OK) {
        std::string keep = g_err;
        destroy_plan(p);
        g_err = keep;
        return st;
      }
    } else if (p->kernel == POBK_KERNEL_AUTO) {
      p->kernel = POBK_KERNEL_LAUNCH;
    }
    p->prep_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = static_cast<pobk_plan_s*>(p);
    return POBK_OK;
  } catch (const std::bad_alloc&) {
    return fail(POBK_ERR_OOM, "host allocation failed during preprocessing");
  } catch (const std::exception& e) {
    return fail(POBK_ERR_ARG, std::string("preprocessing failed: ") + e.what());
  }
}

pobk_status pobk_blocks_preprocess(int64_t m, const int64_t* row_ptr, const int32_t* col, const double* val,
                                   const pobk_blocks_opts* opts, int device, pobk_plan_t* out) {
  g_err.clear();
  if (!out) return fail(POBK_ERR_ARG, "out is NULL");
  *out = nullptr;
  if (!opts) return fail(POBK_ERR_ARG, "opts is NULL (k has no default)");
  if (device < -1) return fail(POBK_ERR_ARG, "device must be >= -1");
  try {
    auto t0 = std::chrono::steady_clock::now();
    HostCSR A;
    Error err;
    if (!canonicalize(m, row_ptr, col, val, A, err)) return fail(err.code, err.msg);
    Plan* p = new pobk_plan_s();
    p->device = device;
    p->m = m;
    p->nnz = A.nnz();
    p->thr = opts->thr;
    p->kernel = POBK_KERNEL_BLOCKS;
    p->bw_before = bandwidth(A);
    if (opts->reorder) rcm_order(A, p->perm);
    else {
      p->perm.resize(m);
      for (int64_t i = 0; i < m; i++) p->perm[i] = (int32_t)i;
    }
    HostCSR At;
    permute_symmetric(A, p->perm, At);
    { HostCSR().ptr.swap(A.ptr); std::vector<int32_t>().swap(A.col); std::vector<double>().swap(A.val); }
    p->bw_after = bandwidth(At);
    if (!block_layout(At, opts->k, opts->thr, p->blocks_host, err)) {
      destroy_plan(p);
      return fail(err.code, err.msg);
    }
    const BlockLayout& L = p->blocks_host;
    // storage order = RCM order; "categories" = the blocks (colour = block id)
    p->colour.assign(m, 0);
    p->sched.step_ptr.assign(L.k + 1, 0);
    for (int32_t b = 0; b < L.k; b++) {
      p->sched.step_ptr[b + 1] = (int32_t)L.ptr[b + 1];
      for (int64_t r = L.ptr[b]; r < L.ptr[b + 1]; r++) p->colour[r] = b;
    }
    p->sched.rows.resize(m);
    for (int64_t i = 0; i < m; i++) p->sched.rows[i] = (int32_t)i;
    p->sched.n_oclass = (int32_t)(2 * L.pairs.size());
    p->sched.overlap.assign(L.k, 0);
    p->nsteps = L.k;
    p->n_oclass = p->sched.n_oclass;
    if (device >= 0) {
      int64_t bmax = 0;
      for (int32_t b = 0; b < L.k; b++) bmax = std::max<int64_t>(bmax, L.ptr[b + 1] - L.ptr[b]);
      if (bmax > 20000) {
        destroy_plan(p);
        return fail(POBK_ERR_ARG, "blocks of " + std::to_string(bmax) + " rows: the k-block path keeps a dense Gram "
                                  "inverse per block and takes blocks of <= 20,000 rows (raise k)");
      }
      std::vector<double> nrm2;
      row_sqnorms(At, nrm2);
      pobk_status st = build_device(*p, At, nrm2, 0);
      if (st != POBK_OK) {
        std::string keep = g_err;
        destroy_plan(p);
        g_err = keep;
        return st;
      }
    }
    p->prep_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = static_cast<pobk_plan_s*>(p);
    return POBK_OK;
  } catch (const std::bad_alloc&) {
    return fail(POBK_ERR_OOM, "host allocation failed during preprocessing");
  } catch (const std::exception& e) {
    return fail(POBK_ERR_ARG, std::string("preprocessing failed: ") + e.what());
  }
}

pobk_status pobk_blocks_info(pobk_plan_t p, int32_t* k, int64_t* block_ptr, double* cos_table, int32_t* pairs,
                             int32_t* npairs, int32_t* nclass, int32_t* nnclass, double* zn, double* nn) {
  if (!p) return fail(POBK_ERR_ARG, "plan is NULL");
  const BlockLayout* L = p->k5 ? k5_layout(*p) : (p->blocks_host.k > 0 ? &p->blocks_host : nullptr);
  if (!L) return fail(POBK_ERR_ARG, "not a k-block plan (pobk_blocks_preprocess)");
  if (k) *k = L->k;
  if (block_ptr) std::memcpy(block_ptr, L->ptr.data(), L->ptr.size() * sizeof(int64_t));
  if (cos_table) std::memcpy(cos_table, L->cos.data(), L->cos.size() * sizeof(double));
  if (pairs)
    for (size_t i = 0; i < L->pairs.size(); i++) { pairs[2 * i] = L->pairs[i].first; pairs[2 * i + 1] = L->pairs[i].second; }
  if (npairs) *npairs = (int32_t)L->pairs.size();
  if (nclass) std::memcpy(nclass, L->nclass.data(), L->nclass.size() * sizeof(int32_t));
  if (nnclass) *nnclass = (int32_t)L->nclass.size();
  if (zn) *zn = L->zn;
  if (nn) *nn = L->nn;
  return POBK_OK;
}

pobk_status pobk_plan_info(pobk_plan_t p, int64_t* m, int64_t* nnz, int32_t* nsteps, int32_t* n_oclass, int64_t* bw_before,
                           int64_t* bw_after, double* prep) {
  if (!p) return fail(POBK_ERR_ARG, "plan is NULL");
  if (m) *m = p->m;
  if (nnz) *nnz = p->nnz;
  if (nsteps) *nsteps = p->nsteps;
  if (n_oclass) *n_oclass = p->n_oclass;
  if (bw_before) *bw_before = p->bw_before;
  if (bw_after) *bw_after = p->bw_after;
  if (prep) *prep = p->prep_seconds;
  return POBK_OK;
}

pobk_status pobk_plan_get_perm(pobk_plan_t p, int32_t* perm) {
  if (!p || !perm) return fail(POBK_ERR_ARG, "plan and perm must be non-NULL");
  std::memcpy(perm, p->perm.data(), p->m * sizeof(int32_t));
  return POBK_OK;
}

pobk_status pobk_plan_get_partition(pobk_plan_t p, int32_t* colour, int32_t* cat_ptr, int32_t* cat_rows) {
  if (!p) return fail(POBK_ERR_ARG, "plan is NULL");
  if (colour) std::memcpy(colour, p->colour.data(), p->m * sizeof(int32_t));
  if (cat_ptr) std::memcpy(cat_ptr, p->sched.step_ptr.data(), p->sched.step_ptr.size() * sizeof(int32_t));
  if (cat_rows) std::memcpy(cat_rows, p->sched.rows.data(), p->m * sizeof(int32_t));
  return POBK_OK;
}

pobk_status pobk_plan_get_tiles(pobk_plan_t p, int32_t* ntiles, int32_t* tile_of_row) {
  if (!p) return fail(POBK_ERR_ARG, "plan is NULL");
  if (ntiles) *ntiles = p->ntiles;
  if (tile_of_row) {
    if (p->tile_of_row.empty()) return fail(POBK_ERR_ARG, "plan has no K2 tiling");
    std::memcpy(tile_of_row, p->tile_of_row.data(), p->m * sizeof(int32_t));
  }
  return POBK_OK;
}

pobk_status pobk_plan_get_layout_stats(pobk_plan_t p, pobk_layout_stats* out) {
  if (!p || !out) return fail(POBK_ERR_ARG, "plan and out must be non-NULL");
  std::memset(out, 0, sizeof(*out));
  out->kernel = p->kernel;
  K2Stats st;
  if (k2_stats(*p, st)) {
    out->ntiles = st.T;
    out->nchunks = st.nchunks;
    out->threads = st.threads;
    out->private_nnz_frac = st.private_frac;
    out->interior_row_frac = st.interior_frac;
    out->stream_bytes = st.stream_bytes;
  }
  return POBK_OK;
}

pobk_status pobk_solve(pobk_plan_t plan, const double* f, double* x, const double* xstar, const pobk_solve_opts* opts,
                       void* stream, pobk_report* rep) {
  g_err.clear();
  pobk_solve_opts o;
  pobk_status st = check_solve_args(plan, f, x, xstar, o, opts);
  if (st != POBK_OK) return st;
  DeviceGuard g(plan->device);
  if (!g.ok) return fail(POBK_ERR_CUDA, "cudaSetDevice failed");
  return solve_device(*plan, f, x, o.stop == POBK_STOP_RSE ? xstar : nullptr, o, (cudaStream_t)stream, rep);
}

pobk_status pobk_solve_host(pobk_plan_t plan, const double* f, double* x, const double* xstar, const pobk_solve_opts* opts,
                            void* stream, pobk_report* rep) {
  g_err.clear();
  pobk_solve_opts o;
  pobk_status st = check_solve_args(plan, f, x, xstar, o, opts);
  if (st != POBK_OK) return st;
  DeviceGuard g(plan->device);
  if (!g.ok) return fail(POBK_ERR_CUDA, "cudaSetDevice failed");
  Plan& p = *plan;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bytes = p.m * sizeof(double);
  if (!p.d_io) CUDA_TRY(dalloc(p, &p.d_io, 3 * p.m));
  double *df = p.d_io, *dx = p.d_io + p.m, *dxs = p.d_io + 2 * p.m;
  const bool rse = o.stop == POBK_STOP_RSE;
  CUDA_TRY(cudaMemcpyAsync(df, f, bytes, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(dx, x, bytes, cudaMemcpyHostToDevice, s));
  if (rse) CUDA_TRY(cudaMemcpyAsync(dxs, xstar, bytes, cudaMemcpyHostToDevice, s));
  // the solution's copy back is enqueued behind the solve: one host synchronisation per call
  st = solve_device(p, df, dx, rse ? dxs : nullptr, o, s, nullptr, true);
  if (st != POBK_OK) {
    (void)cudaStreamSynchronize(s);  // (nothing of this call outlives it)
    return st;
  }
  CUDA_TRY(cudaMemcpyAsync(x, dx, bytes, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return solve_finish(p, o, rep);
}

// The lanes rule of pobk_solve_batch / pobk_solve_batch_host: when every system is a K2 plan on
// the same device, no plan is named twice, and nl >= 2 of their grids fit side by side (e.g. plans
// built with half-GPU tiles), system b runs on internal stream b mod nl, so nl cooperative sweep
// kernels share the GPU (each system's latency-bound step chain overlaps the others').  Returns
// nl (>= 2), or 1 for back-to-back solves.  Results are those of back-to-back solves (tiling
// never changes them).
static int batch_lane_count(pobk_plan_t* plans, int32_t nb, int& dev) {
  bool lanes = nb >= 2;
  int sms = 148;
  dev = -1;
  for (int32_t b = 0; b < nb && lanes; b++) {
    if (!plans[b] || plans[b]->device < 0 || plans[b]->kernel != POBK_KERNEL_WAVEFRONT || !plans[b]->k2) lanes = false;
    else if (dev >= 0 && plans[b]->device != dev) lanes = false;
    else dev = plans[b]->device;
  }
  // a plan is not re-entrant (its vectors, control block and events serve one solve at a time):
  // a batch that names a plan twice runs back to back, each solve reported before the next
  for (int32_t b = 0; b < nb && lanes; b++)
    for (int32_t c = 0; c < b && lanes; c++)
      if (plans[c] == plans[b]) lanes = false;
  if (!lanes) return 1;
  int v = 0;  // (cudaGetDeviceProperties costs milliseconds; the attribute query does not)
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0) sms = v;
  int tmax = 1;
  for (int32_t b = 0; b < nb; b++) tmax = std::max(tmax, (int)plans[b]->ntiles);
  const int nl = std::min({4, sms / tmax, (int)nb});
  return nl >= 2 && !getenv("POBK_BATCH_SERIAL") ? nl : 1;
}

// internal streams of the batch calls (per host thread and device; created once): the lanes, and
// the host->device / device->host copy streams of pobk_solve_batch_host
struct LaneSet {
  cudaStream_t lane[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
};
static cudaError_t lane_set(int dev, LaneSet** out) {
  static thread_local int lane_dev = -1;
  static thread_local LaneSet set;
  if (lane_dev != dev) {
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < 4 && e == cudaSuccess; i++) e = cudaStreamCreateWithFlags(&set.lane[i], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&set.h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&set.d2h, cudaStreamNonBlocking);
    for (int i = 0; i < 5 && e == cudaSuccess; i++) e = cudaEventCreateWithFlags(&set.ev[i], cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
    lane_dev = dev;
  }
  *out = &set;
  return cudaSuccess;
}

pobk_status pobk_solve_batch(pobk_plan_t* plans, int32_t nb, const double* const* f, double* const* x,
                             const double* const* xstar, const pobk_solve_opts* opts, void* stream, pobk_report* reps) {
  g_err.clear();
  if (nb < 0 || (nb > 0 && (!plans || !f || !x))) return fail(POBK_ERR_ARG, "bad batch arguments");
  // every system's arguments are checked before anything is enqueued (lanes: batch_lane_count)
  std::vector<pobk_solve_opts> os(nb);
  for (int32_t b = 0; b < nb; b++) {
    pobk_status st = check_solve_args(plans[b], f[b], x[b], xstar ? xstar[b] : nullptr, os[b], opts);
    if (st != POBK_OK) {
      g_err = "system " + std::to_string(b) + ": " + g_err;
      return st;
    }
  }
  int dev = -1;
  const int nl = batch_lane_count(plans, nb, dev);
  if (nl < 2) {
    for (int32_t b = 0; b < nb; b++) {
      pobk_status st = pobk_solve(plans[b], f[b], x[b], xstar ? xstar[b] : nullptr, opts, stream, reps ? reps + b : nullptr);
      if (st != POBK_OK) {
        g_err = "system " + std::to_string(b) + ": " + g_err;
        return st;
      }
    }
    return POBK_OK;
  }
  DeviceGuard g(dev);
  if (!g.ok) return fail(POBK_ERR_CUDA, "cudaSetDevice failed");
  LaneSet* ls = nullptr;
  CUDA_TRY(lane_set(dev, &ls));
  cudaStream_t* lane_s = ls->lane;
  cudaEvent_t* lane_ev = ls->ev;
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaEventRecord(lane_ev[4], s));
  for (int i = 0; i < nl; i++) CUDA_TRY(cudaStreamWaitEvent(lane_s[i], lane_ev[4], 0));
  pobk_status enq = POBK_OK;
  for (int32_t b = 0; b < nb && enq == POBK_OK; b++) {
    enq = solve_device(*plans[b], f[b], x[b], os[b].stop == POBK_STOP_RSE && xstar ? xstar[b] : nullptr, os[b], lane_s[b % nl],
                       nullptr, true);
    if (enq != POBK_OK) g_err = "system " + std::to_string(b) + ": " + g_err;
  }
  // (also after a failed enqueue: `stream` is ordered after everything already enqueued and the
  // lanes are drained, so no solve of this call outlives it)
  const std::string keep = g_err;
  for (int i = 0; i < nl; i++) {
    CUDA_TRY(cudaEventRecord(lane_ev[i], lane_s[i]));
    CUDA_TRY(cudaStreamWaitEvent(s, lane_ev[i], 0));
  }
  for (int i = 0; i < nl; i++) CUDA_TRY(cudaStreamSynchronize(lane_s[i]));
  if (enq != POBK_OK) {
    g_err = keep;
    return enq;
  }
  for (int32_t b = 0; b < nb; b++) {
    pobk_status st = solve_finish(*plans[b], os[b], reps ? reps + b : nullptr);
    if (st != POBK_OK) return st;
  }
  return POBK_OK;
}

pobk_status pobk_solve_batch_host(pobk_plan_t* plans, int32_t nb, const double* const* f, double* const* x,
                                  const double* const* xstar, const pobk_solve_opts* opts, void* stream,
                                  pobk_report* reps) {
  g_err.clear();
  if (nb < 0 || (nb > 0 && (!plans || !f || !x))) return fail(POBK_ERR_ARG, "bad batch arguments");
  std::vector<pobk_solve_opts> os(nb);
  for (int32_t b = 0; b < nb; b++) {
    pobk_status st = check_solve_args(plans[b], f[b], x[b], xstar ? xstar[b] : nullptr, os[b], opts);
    if (st != POBK_OK) {
      g_err = "system " + std::to_string(b) + ": " + g_err;
      return st;
    }
  }
  int dev = -1;
  int nl = batch_lane_count(plans, nb, dev);
  if (nl < 2 && nb >= 2) {
    // distinct plans on one device that do not fit side by side: one lane, the copies of the
    // other systems still overlapped with each solve
    bool ok = plans[0] && plans[0]->device >= 0;
    dev = ok ? plans[0]->device : -1;
    for (int32_t b = 1; b < nb && ok; b++) {
      ok = plans[b] && plans[b]->device == dev;
      for (int32_t c = 0; c < b && ok; c++) ok = plans[c] != plans[b];
    }
    nl = ok ? 1 : 0;
  }
  if (nb < 2) nl = 0;
  // the solutions come back concurrently: every system needs its own host x
  for (int32_t b = 0; b < nb; b++)
    for (int32_t c = 0; c < b; c++)
      if (x[c] == x[b]) return fail(POBK_ERR_ARG, "x pointers must be distinct (systems " + std::to_string(c) + " and " + std::to_string(b) + ")");
  if (nl < 1) {  // back to back: each system through pobk_solve_host (copies, solve, copy back)
    for (int32_t b = 0; b < nb; b++) {
      pobk_status st = pobk_solve_host(plans[b], f[b], x[b], xstar ? xstar[b] : nullptr, opts, stream, reps ? reps + b : nullptr);
      if (st != POBK_OK) {
        g_err = "system " + std::to_string(b) + ": " + g_err;
        return st;
      }
    }
    return POBK_OK;
  }
  DeviceGuard g(dev);
  if (!g.ok) return fail(POBK_ERR_CUDA, "cudaSetDevice failed");
  LaneSet* ls = nullptr;
  CUDA_TRY(lane_set(dev, &ls));
  // the plans' staging vectors (f, x, x*), allocated before anything is enqueued
  for (int32_t b = 0; b < nb; b++)
    if (!plans[b]->d_io) {
      DeviceGuard gb(plans[b]->device);
      CUDA_TRY(dalloc(*plans[b], &plans[b]->d_io, 3 * plans[b]->m));
    }
  // per system: inputs arrived (h2d stream -> its lane), solve done (lane -> d2h stream)
  std::vector<cudaEvent_t> ev(2 * (size_t)nb, nullptr);
  auto destroy = [&]() {
    for (cudaEvent_t e : ev)
      if (e) cudaEventDestroy(e);
  };
  for (auto& e : ev)
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
      destroy();
      return fail(POBK_ERR_CUDA, "cudaEventCreate failed");
    }
  cudaStream_t s = (cudaStream_t)stream;
  cudaStream_t* lane_s = ls->lane;
  pobk_status enq = POBK_OK;
  cudaError_t ce = cudaEventRecord(ls->ev[4], s);
  if (ce == cudaSuccess) ce = cudaStreamWaitEvent(ls->h2d, ls->ev[4], 0);
  for (int i = 0; i < nl && ce == cudaSuccess; i++) ce = cudaStreamWaitEvent(lane_s[i], ls->ev[4], 0);
  if (ce == cudaSuccess) ce = cudaStreamWaitEvent(ls->d2h, ls->ev[4], 0);
  if (ce != cudaSuccess) {
    destroy();
    return fail(POBK_ERR_CUDA, cudaGetErrorString(ce));
  }
  // Every system's inputs go in on one copy stream in system order while earlier systems solve on
  // their lanes; each solution comes back on the other copy stream as soon as its solve is done.
  // So only the first round's inputs and the last round's outputs are not hidden behind sweeps.
  for (int32_t b = 0; b < nb && enq == POBK_OK; b++) {
    Plan& p = *plans[b];
    const size_t bytes = p.m * sizeof(double);
    double *df = p.d_io, *dx = p.d_io + p.m, *dxs = p.d_io + 2 * p.m;
    const bool rse = os[b].stop == POBK_STOP_RSE;
    cudaStream_t ln = lane_s[b % nl];
    ce = cudaMemcpyAsync(df, f[b], bytes, cudaMemcpyHostToDevice, ls->h2d);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(dx, x[b], bytes, cudaMemcpyHostToDevice, ls->h2d);
    if (ce == cudaSuccess && rse) ce = cudaMemcpyAsync(dxs, xstar[b], bytes, cudaMemcpyHostToDevice, ls->h2d);
    if (ce == cudaSuccess) ce = cudaEventRecord(ev[2 * b], ls->h2d);
    if (ce == cudaSuccess) ce = cudaStreamWaitEvent(ln, ev[2 * b], 0);
    if (ce != cudaSuccess) {
      enq = fail(POBK_ERR_CUDA, cudaGetErrorString(ce));
      break;
    }
    enq = solve_device(p, df, dx, rse ? dxs : nullptr, os[b], ln, nullptr, true);
    if (enq != POBK_OK) break;
    ce = cudaEventRecord(ev[2 * b + 1], ln);
    if (ce == cudaSuccess) ce = cudaStreamWaitEvent(ls->d2h, ev[2 * b + 1], 0);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(x[b], dx, bytes, cudaMemcpyDeviceToHost, ls->d2h);
    if (ce != cudaSuccess) enq = fail(POBK_ERR_CUDA, cudaGetErrorString(ce));
  }
  if (enq != POBK_OK) g_err = "batch: " + g_err;
  // (also after a failed enqueue: `stream` is ordered after everything already enqueued and the
  // internal streams are drained, so no copy or solve of this call outlives it)
  const std::string keep = g_err;
  ce = cudaSuccess;
  cudaStream_t all[6] = {ls->h2d, ls->d2h, lane_s[0], lane_s[1], lane_s[2], lane_s[3]};
  for (int i = 0; i < 2 + nl; i++) {
    cudaError_t e1 = cudaEventRecord(ls->ev[i < 4 ? i : 3], all[i]);
    if (e1 == cudaSuccess) e1 = cudaStreamWaitEvent(s, ls->ev[i < 4 ? i : 3], 0);
    cudaError_t e2 = cudaStreamSynchronize(all[i]);
    if (ce == cudaSuccess) ce = e1 != cudaSuccess ? e1 : e2;
  }
  destroy();
  if (enq != POBK_OK) {
    g_err = keep;
    return enq;
  }
  if (ce != cudaSuccess) return fail(POBK_ERR_CUDA, cudaGetErrorString(ce));
  for (int32_t b = 0; b < nb; b++) {
    pobk_status st = solve_finish(*plans[b], os[b], reps ? reps + b : nullptr);
    if (st != POBK_OK) return st;
  }
  return POBK_OK;
}

pobk_status pobk_solve_multi(pobk_plan_t plan, int32_t R, const double* const* f, double* const* x,
                             const double* const* xstar, const pobk_solve_opts* opts, void* stream, pobk_report* reps) {
  g_err.clear();
  if (R < 1 || R > kMaxRHS) return fail(POBK_ERR_ARG, "R must be in [1, " + std::to_string(kMaxRHS) + "]");
  if (!f || !x || !reps) return fail(POBK_ERR_ARG, "f, x and reps must be non-NULL");
  pobk_solve_opts o;
  for (int32_t r = 0; r < R; r++) {
    pobk_status st = check_solve_args(plan, f[r], x[r], xstar ? xstar[r] : nullptr, o, opts);
    if (st != POBK_OK) {
      g_err = "right-hand side " + std::to_string(r) + ": " + g_err;
      return st;
    }
  }
  if (o.stop == POBK_STOP_RELRES) return fail(POBK_ERR_ARG, "pobk_solve_multi supports POBK_STOP_RSE and POBK_STOP_NONE");
  if (plan->any_overlap || plan->kernel == POBK_KERNEL_BLOCKS)
    return fail(POBK_ERR_ARG, "pobk_solve_multi needs a row-level plan with thr = 0 (disjoint categories)");
  for (int32_t r = 0; r < R; r++)
    for (int32_t q = 0; q < r; q++)
      if (x[q] == x[r]) return fail(POBK_ERR_ARG, "x pointers must be distinct");
  DeviceGuard g(plan->device);
  if (!g.ok) return fail(POBK_ERR_CUDA, "cudaSetDevice failed");
  Plan& p = *plan;
  cudaStream_t s = (cudaStream_t)stream;
  const bool rse = o.stop == POBK_STOP_RSE;
  // K2 plans: right-hand sides in pairs through the two-RHS K2 plan (A~ streamed once per sweep
  // for both), an odd last one through the plan's own solve; others: K1M (all R in one loop)
  static const bool force_k1m = getenv("POBK_MULTI_KERNEL") && !strcmp(getenv("POBK_MULTI_KERNEL"), "launch");  // (development)
  if (p.k2 && p.kernel == POBK_KERNEL_WAVEFRONT && R >= 2 && !force_k1m) {
    if (!p.k2r) {
      std::string why;
      if (!k2r_build(p, why)) return fail(POBK_ERR_CUDA, "two-RHS K2 plan: " + why);
    }
    for (int32_t r = 0; r + 1 < R; r += 2) {
      const double* ff[2] = {f[r], f[r + 1]};
      double* xx[2] = {x[r], x[r + 1]};
      const double* xs[2] = {rse ? xstar[r] : nullptr, rse ? xstar[r + 1] : nullptr};
      CUDA_TRY(k2r_solve(p, ff, xx, xs, o, s, reps + r));
    }
    if (R & 1) {
      pobk_status st = solve_device(p, f[R - 1], x[R - 1], rse ? xstar[R - 1] : nullptr, o, s, reps + R - 1);
      if (st != POBK_OK) return st;
    }
    return POBK_OK;
  }
  CUDA_TRY(k1m_solve(p, R, f, x, xstar, o, s, reps));
  return POBK_OK;
}

pobk_status pobk_residual_sumsq_rows(pobk_plan_t plan, int64_t lo, int64_t hi, const double* f, const double* x, void* stream,
                                     double* out) {
  g_err.clear();
  if (!plan || !f || !x || !out) return fail(POBK_ERR_ARG, "plan, f, x, out must be non-NULL");
  if (plan->device < 0) return fail(POBK_ERR_NO_DEVICE, "host-only plan");
  if (lo < 0 || hi > plan->m || lo > hi) return fail(POBK_ERR_ARG, "row range out of bounds");
  DeviceGuard g(plan->device);
  if (!g.ok) return fail(POBK_ERR_CUDA, "cudaSetDevice failed");
  Plan& p = *plan;
  cudaStream_t s = (cudaStream_t)stream;
  if (!p.d_tmpvec) CUDA_TRY(dalloc(p, &p.d_tmpvec, p.m));
  if (!p.d_tmpf) CUDA_TRY(dalloc(p, &p.d_tmpf, p.m));
  long long launches = 0;
  CUDA_TRY(launch_permute_in(p, f, x, nullptr, p.d_tmpf, p.d_tmpvec, nullptr, s, launches));
  const bool all = lo == 0 && hi == p.m;
  CUDA_TRY(residual_sumsq(p, p.d_tmpf, p.d_tmpvec, all ? nullptr : p.A.orig, lo, hi, s, out, launches));
  return POBK_OK;
}

pobk_status pobk_residual_norm(pobk_plan_t plan, const double* f, const double* x, void* stream, double* out) {
  if (!plan) return fail(POBK_ERR_ARG, "plan is NULL");
  double ss = 0.0;
  pobk_status st = pobk_residual_sumsq_rows(plan, 0, plan->m, f, x, stream, &ss);
  if (st == POBK_OK && out) *out = std::sqrt(ss);
  return st;
}

void pobk_plan_destroy(pobk_plan_t plan) { destroy_plan(plan); }

}  // extern "C"
