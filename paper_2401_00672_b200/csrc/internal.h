// Internal declarations shared by the host preprocessing (host/*.cpp), the kernels (cuda/*.cu)
// and the C ABI (capi.cpp).  Not installed; the public interface is include/pobk.h.
#pragma once
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "../../include/pobk.h"

namespace pobk {

// ----------------------------------------------------------------------------- host CSR
struct HostCSR {
  int64_t m = 0;
  std::vector<int64_t> ptr;  // [m+1]
  std::vector<int32_t> col;  // [nnz], strictly increasing per row
  std::vector<double> val;   // [nnz], no stored zeros
  int64_t nnz() const { return ptr.empty() ? 0 : ptr[m]; }
};

struct Error {
  pobk_status code = POBK_OK;
  std::string msg;
};

// host/preprocess.cpp -- Alg 5 steps 1-4, DESIGN.md §3.
bool canonicalize(int64_t m, const int64_t* row_ptr, const int32_t* col, const double* val, HostCSR& out, Error& err);
int64_t bandwidth(const HostCSR& A);
void rcm_order(const HostCSR& A, std::vector<int32_t>& perm);                 // perm[new] = old
void permute_symmetric(const HostCSR& A, const std::vector<int32_t>& perm, HostCSR& out);
void row_sqnorms(const HostCSR& A, std::vector<double>& nrm2);
void first_fit_colour(const HostCSR& A, const std::vector<double>& nrm2, double thr, std::vector<int32_t>& colour);
struct Schedule {
  std::vector<int32_t> step_ptr;   // [nsteps+1]
  std::vector<int32_t> rows;       // [m], RCM-frame rows in schedule order
  int32_t n_oclass = 0;
  std::vector<uint8_t> overlap;    // [nsteps] 1 if two rows of the step share a column (thr > 0)
};
void build_schedule(const HostCSR& A, const std::vector<int32_t>& colour, bool check_overlap, Schedule& s);
bool gershgorin_guard(const HostCSR& A, const std::vector<double>& nrm2, const std::vector<int32_t>& colour,
                      std::string& why);

// host/blocks.cpp -- the paper-literal k-block variant (Alg 5 steps 2-4 with k uniform chunks).
struct BlockLayout {
  int32_t k = 0;
  double thr = 0.0;
  std::vector<int64_t> ptr;                        // [k+1] block boundaries (RCM frame)
  std::vector<double> cos;                         // [k*k] centroid cosine table C
  std::vector<std::pair<int32_t, int32_t>> pairs;  // Oclass: class{i} = (i, j)
  std::vector<int32_t> nclass;                     // Nclass blocks, ascending
  std::vector<int32_t> order;                      // one iteration: pairs (tau1, tau2), then Nclass
  double zn = 0.0, nn = 0.0;                       // Definitions 1-2
};
bool block_layout(const HostCSR& At, int32_t k, double thr, BlockLayout& out, Error& err);
bool block_gram_inverses(const HostCSR& At, const BlockLayout& L, std::vector<std::vector<double>>& ginv, Error& err);

// ----------------------------------------------------------------------------- device control block
// One per solve, in device memory.  Written by the check kernels, read back at the end.
struct Ctrl {
  long long sweeps;        // sweeps completed
  long long max_sweeps;
  double tol;
  double value;            // last checked RSE / RELRES
  double den;              // ||x*||^2 (RSE) or ||f||^2 (RELRES)
  int stop_mode;           // POBK_STOP_*
  int check_every;
  int stopped;             // 1 once the loop must end
  int term;                // POBK_TERM_*
  unsigned int arrive;     // last-block-done counter for the check reductions
  unsigned int pad;
  long long offset;        // sweeps done before this call (resume numbering): check when
                           // (offset + sweep) % check_every == 0
};

}  // namespace pobk
