// The plan: everything pobk_preprocess builds, host and device.  Internal to libpobk.so.
#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "internal.h"

namespace pobk {

// Device CSR of A~ in one row order ("storage order"); rows of a schedule step are contiguous
// for the per-step kernels (K1, K3, K4); K2 keeps its own tile-major copy (k2_plan.h).
struct DevCSR {
  int32_t* rp = nullptr;     // [m+1] offsets into col/val (nnz < 2^31)
  int32_t* col = nullptr;    // [nnz] RCM-frame column ids
  double* val = nullptr;     // [nnz]
  double* nrm2 = nullptr;    // [m]   ||a~_i||^2 in storage order
  int32_t* orig = nullptr;   // [m]   user-frame row of each storage row (perm[rcm row])
};

struct K2Plan;  // cuda/k2_wavefront.cu
struct K4Plan;  // cuda/k4_cluster.cu
struct K5Plan;  // cuda/k5_blocks.cu
struct MultiPlan;  // cuda/k1_multi.cu
constexpr int kMaxRHS = 8;  // right-hand sides per pobk_solve_multi call

struct Plan {
  int device = -1;
  int64_t m = 0, nnz = 0;
  int32_t nsteps = 0, n_oclass = 0;
  int64_t bw_before = 0, bw_after = 0;
  double prep_seconds = 0.0;
  double thr = 0.0;
  int kernel = POBK_KERNEL_AUTO;  // family chosen at preprocess
  bool any_overlap = false;

  // host copies (queries, tests)
  std::vector<int32_t> perm, colour;
  Schedule sched;
  std::vector<int32_t> tile_of_row;
  int32_t ntiles = 0;

  // device
  int32_t* d_perm = nullptr;      // [m] new -> old
  DevCSR A;                       // schedule order (step-major)
  std::vector<int32_t> h_step_ptr;
  std::vector<uint8_t> h_overlap;
  double* d_xt = nullptr;         // [m] x~ (RCM frame)
  double* d_xst = nullptr;        // [m] x~* (RCM frame)
  double* d_fs = nullptr;         // [m] f~ in storage order
  double* d_alpha = nullptr;      // [max step size] thr > 0 scratch
  // thr > 0, overlapping steps: the step's entries grouped by column (CSC over its schedule
  // positions, ascending), so the scatter x~_c += sum_i alpha_i a~_ic is one fold per column in
  // the oracle's order (bitwise) -- no atomics (POBK_THR_ATOMIC=1: the fp64-atomic scatter)
  std::vector<int32_t> h_ov_colptr;  // [nsteps+1] offsets into ov_cols (empty range: disjoint step)
  int32_t* ov_colptr = nullptr;   // device copy of h_ov_colptr (K3)
  int32_t* ov_cols = nullptr;     // [ncols] the columns each overlapping step touches
  int32_t* ov_eptr = nullptr;     // [ncols+1] offsets into ov_es / ov_ev
  int32_t* ov_es = nullptr;       // [entries] step-local row index (the alpha slot), ascending per column
  double* ov_ev = nullptr;        // [entries] a~_ic
  double* d_partials = nullptr;   // [kMaxReduceBlocks]
  Ctrl* d_ctrl = nullptr;
  Ctrl* h_ctrl = nullptr;         // pinned mirror
  double* d_tmpvec = nullptr;     // [m] residual_norm scratch (x~ of the caller's x)
  double* d_tmpf = nullptr;       // [m] residual_norm scratch (f in storage order)
  double* d_io = nullptr;         // [3m] pobk_solve_host staging
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};

  // K1 device-driven loop
  cudaGraph_t k1_graph = nullptr;
  cudaGraphExec_t k1_exec = nullptr;
  long long k1_nodes_per_sweep = 0;
  // K1E: sliced ELL of A~ (32-row slices in schedule order, never across a step; entry j of the
  // slice's row l at k1e_ptr[slice] + 32 j + l) so a warp's loads of row entries coalesce
  int32_t* k1e_col = nullptr;
  double* k1e_val = nullptr;
  int64_t* k1e_ptr = nullptr;            // [nslices+1]
  std::vector<int32_t> h_k1e_slice0;     // [nsteps] first slice of each step
  int32_t* k1e_slice0 = nullptr;         // device copy (the residual-ordered loop picks its step on the device)
  cudaGraph_t k1o_graph = nullptr;       // the residual-ordered sweep loop (opts.order)
  cudaGraphExec_t k1o_exec = nullptr;
  long long k1o_nodes_per_sweep = 0;

  K2Plan* k2 = nullptr;
  K2Plan* k2r = nullptr;           // two right-hand sides per sweep (pobk_solve_multi, R = 2)
  int k2_tile_rows = 0;            // the preprocess option K2 was built with (reused by k2r)
  long long pending_launches = 0;  // solve_device -> solve_finish (batched solves)
  int pending_used = 0;
  K4Plan* k4 = nullptr;
  K5Plan* k5 = nullptr;            // the paper-literal k-block variant (pobk_blocks_preprocess)
  MultiPlan* multi = nullptr;      // several right-hand sides in one sweep loop (pobk_solve_multi)
  BlockLayout blocks_host;         // its layout on host-only plans (device = -1)
  size_t k3_smem = 0;
  int32_t* k3_step_ptr = nullptr;  // [nsteps+1] device copy of the schedule steps
  uint8_t* k3_overlap = nullptr;   // [nsteps]
  int32_t* k3e_col = nullptr;      // K3E thread-major ELL (k3_smem.cu); NULL: K3 reads the CSR
  double* k3e_val = nullptr;
  int32_t* k3e_info = nullptr;     // [nsteps*4]
  int k3e_nent = 0;

  std::vector<void*> allocations;
};

constexpr int kMaxReduceBlocks = 296;

// cuda/vec_kernels.cu
// Raise a kernel's dynamic shared-memory limit to the whole per-CTA budget (the device's opt-in
// maximum, 227 KB on B200, minus the kernel's static shared memory), once per
// (kernel, device), never lowering it: changing the attribute while another host thread or lane
// launches the kernel can fail or serialise those launches (thread-safe).
cudaError_t raise_smem_limit(const void* fn);
// f (user frame) -> fs (storage order); x0, xstar (user frame) -> xt, xst (RCM frame); any input may be NULL
cudaError_t launch_permute_in(const Plan& p, const double* f, const double* x0, const double* xstar, double* fs,
                              double* xt, double* xst, cudaStream_t s, long long& launches);
cudaError_t launch_permute_out(const Plan& p, double* x, cudaStream_t s, long long& launches);
cudaError_t launch_permute_out_from(const Plan& p, const double* xt, double* x, cudaStream_t s, long long& launches);
// c->den = ||v||^2 (deterministic two-level sum)
cudaError_t launch_den(const Plan& p, Ctrl* c, const double* v, cudaStream_t s, long long& launches);
cudaError_t launch_init_ctrl(const Plan& p, const pobk_solve_opts& o, cudaStream_t s, long long& launches);
cudaError_t launch_check(const Plan& p, cudaStream_t s);
cudaError_t launch_check_graph(const Plan& p, cudaStream_t s, cudaGraphConditionalHandle h);
cudaError_t residual_sumsq(const Plan& p, const double* fs, const double* xt, const int32_t* orig_lo_hi, int64_t lo,
                           int64_t hi, cudaStream_t s, double* host_out, long long& launches);

// cuda/k1_launch.cu
cudaError_t k1_solve(Plan& p, cudaStream_t s, long long& launches);
cudaError_t k1_solve_ordered(Plan& p, cudaStream_t s, long long& launches);
// cuda/k3_smem.cu
bool k3_fits(const Plan& p, size_t& smem_bytes);
cudaError_t k3e_build(Plan& p, const std::vector<int32_t>& rp, const std::vector<int32_t>& col,
                      const std::vector<double>& val, size_t* smem_bytes, bool* built);
cudaError_t k3_solve(Plan& p, cudaStream_t s, long long& launches);
// cuda/k4_cluster.cu
bool k4_build(Plan& p, const std::vector<int32_t>& rp, const std::vector<int32_t>& col, const std::vector<double>& val,
              std::string& why);
cudaError_t k4_solve(Plan& p, cudaStream_t s, long long& launches);
void k4_free(Plan& p);
int k4_cluster_size(const Plan& p);
// cuda/k1_multi.cu (R right-hand sides, A read once per step for all of them)
cudaError_t k1m_solve(Plan& p, int R, const double* const* f, double* const* x, const double* const* xstar,
                      const pobk_solve_opts& o, cudaStream_t s, pobk_report* reps);
void k1m_free(Plan& p);
// cuda/k5_blocks.cu (the paper-literal k-block variant)
bool k5_build(Plan& p, const HostCSR& At, BlockLayout&& L, std::vector<std::vector<double>>&& ginv, std::string& why);
cudaError_t k5_solve(Plan& p, cudaStream_t s, long long& launches);
long long k5_nodes_per_sweep(const Plan& p);
const BlockLayout* k5_layout(const Plan& p);
void k5_free(Plan& p);
// cuda/k2_wavefront.cu
bool k2_build(Plan& p, const HostCSR& At, const std::vector<double>& nrm2, int tile_rows, std::string& why, int kR = 1);
cudaError_t k2_solve(Plan& p, const double* f_user, cudaStream_t s, long long& launches);
struct K2Stats { int T; double private_frac, interior_frac; long long stream_bytes; int nchunks; int threads; };
bool k2_stats(const Plan& p, K2Stats& st);
bool k2_relres_ok(const Plan& p);
void k2_free(Plan& p);
// the two-RHS K2 plan (pobk_solve_multi with R = 2 on a K2 plan): built on first use
bool k2r_build(Plan& p, std::string& why);
cudaError_t k2r_solve(Plan& p, const double* const* f, double* const* x, const double* const* xstar,
                      const pobk_solve_opts& o, cudaStream_t s, pobk_report* reps);
void k2r_free(Plan& p);

}  // namespace pobk

// The opaque ABI handle is the plan itself.
struct pobk_plan_s : public pobk::Plan {};
