// K5: the paper-literal POBK iteration with k uniform row blocks (Alg 5 loop, PAPER.md:236-243;
// SURVEY.md §8(f) NEXT-2).  One block step (Eq 3.3; A_tau^+ = A_tau^T (A_tau A_tau^T)^-1 for a
// full-row-rank block, Lemma 1) is three launches:
//   k5_resid   r = f~_tau - A_tau x~            one thread per block row (CSR, contract order)
//   k5_gemv    y = G_tau^-1 r                   one warp per row of the dense inverse (coalesced,
//                                               fixed-order lane sums + fixed butterfly)
//   k5_update  x~_c += sum_r a_rc y_r           one thread per column the block touches (the
//                                               block's CSC, rows ascending): no atomics
// An iteration applies the blocks in the plan's order (each Oclass pair tau1 then tau2, then the
// Nclass blocks ascending); the sweep loop is a CUDA-graph WHILE node whose body ends with the
// shared stop-check kernel (RSE / RELRES), as in K1.  HBM-bound on the G^-1 stream (8 b^2 bytes
// per block step); the SpMVs are L2-resident.
#include <algorithm>
#include <string>
#include <vector>

#include "../plan.h"
#include "common.cuh"

namespace pobk {

struct K5Plan {
  BlockLayout L;
  std::vector<int64_t> goff;     // [k] offset of each block's G^-1 in ginv (doubles)
  std::vector<int32_t> cptr_off, ncols;  // per block: offset into ccol/cptr arrays, columns touched
  double* ginv = nullptr;        // concatenated dense G_tau^-1 (row-major)
  int32_t* cptr = nullptr;       // per block [ncols+1] offsets into crow/cval (concatenated)
  int32_t* ccol = nullptr;       // per block [ncols] RCM-frame column ids
  int32_t* crow = nullptr;       // block-local row of each CSC entry
  double* cval = nullptr;
  int64_t centry_off_total = 0;
  std::vector<int64_t> centry_off;  // per block offset into crow/cval
  double* r = nullptr;           // [max block rows]
  double* y = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  long long nodes_per_sweep = 0;
  std::vector<void*> allocs;
};

namespace {
constexpr int kNT = 128;

__global__ void __launch_bounds__(kNT) k5_resid(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                const double* __restrict__ val, const double* __restrict__ fs,
                                                const double* __restrict__ x, double* __restrict__ r, int64_t r0, int b) {
  const int i = blockIdx.x * kNT + threadIdx.x;
  if (i >= b) return;
  const int64_t s = r0 + i;
  r[i] = __dsub_rn(fs[s], row_dot(col, val, rp[s], rp[s + 1], x));
}

__global__ void __launch_bounds__(kNT) k5_gemv(const double* __restrict__ gi, const double* __restrict__ r,
                                               double* __restrict__ y, int b) {
  const int w = blockIdx.x * (kNT / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= b) return;
  const double* row = gi + (size_t)w * b;
  double acc = 0.0;
  for (int j = lane; j < b; j += 32) acc = __dadd_rn(acc, __dmul_rn(row[j], r[j]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
  if (lane == 0) y[w] = acc;
}

__global__ void __launch_bounds__(kNT) k5_update(const int32_t* __restrict__ cptr, const int32_t* __restrict__ ccol,
                                                 const int32_t* __restrict__ crow, const double* __restrict__ cval,
                                                 const double* __restrict__ y, double* __restrict__ x, int ncols) {
  const int t = blockIdx.x * kNT + threadIdx.x;
  if (t >= ncols) return;
  double s = 0.0;
  for (int q = cptr[t]; q < cptr[t + 1]; q++) s = __dadd_rn(s, __dmul_rn(cval[q], y[crow[q]]));
  const int c = ccol[t];
  x[c] = __dadd_rn(x[c], s);
}

template <typename T>
cudaError_t k5_upload(K5Plan& k, T** dst, const T* src, size_t n) {
  void* v = nullptr;
  cudaError_t e = cudaMalloc(&v, std::max<size_t>(n, 1) * sizeof(T));
  if (e != cudaSuccess) return e;
  k.allocs.push_back(v);
  *dst = (T*)v;
  if (n && src) e = cudaMemcpy(v, src, n * sizeof(T), cudaMemcpyHostToDevice);
  return e;
}

cudaError_t capture_sweep(const Plan& p, const K5Plan& k, cudaStream_t cs, long long& nodes) {
  for (int32_t b : k.L.order) {
    const int64_t r0 = k.L.ptr[b];
    const int nb = (int)(k.L.ptr[b + 1] - r0);
    k5_resid<<<(nb + kNT - 1) / kNT, kNT, 0, cs>>>(p.A.rp, p.A.col, p.A.val, p.d_fs, p.d_xt, k.r, r0, nb);
    k5_gemv<<<(nb + kNT / 32 - 1) / (kNT / 32), kNT, 0, cs>>>(k.ginv + k.goff[b], k.r, k.y, nb);
    const int nc = k.ncols[b];
    k5_update<<<(nc + kNT - 1) / kNT, kNT, 0, cs>>>(k.cptr + k.cptr_off[b], k.ccol + k.cptr_off[b] - b, k.crow + k.centry_off[b],
                                                   k.cval + k.centry_off[b], k.y, p.d_xt, nc);
    nodes += 3;
  }
  return cudaGetLastError();
}
}  // namespace

// Device layout of a k-block plan: G_tau^-1 for every block, the blocks' CSC (column lists), and
// scratch vectors.  The CSR of A~ in RCM order (storage order) is the plan's p.A.
bool k5_build(Plan& p, const HostCSR& At, BlockLayout&& L, std::vector<std::vector<double>>&& ginv, std::string& why) {
  K5Plan* k = new K5Plan();
  p.k5 = k;
  k->L = std::move(L);
  const int32_t nb = k->L.k;
  std::vector<double> g;
  int64_t tot = 0, bmax = 1;
  for (int32_t b = 0; b < nb; b++) {
    k->goff.push_back(tot);
    tot += (int64_t)ginv[b].size();
    bmax = std::max<int64_t>(bmax, k->L.ptr[b + 1] - k->L.ptr[b]);
  }
  // CSC per block: columns touched (ascending), entries by row ascending within a column
  std::vector<int32_t> cptr, ccol, crow;
  std::vector<double> cval;
  for (int32_t b = 0; b < nb; b++) {
    const int64_t r0 = k->L.ptr[b], r1 = k->L.ptr[b + 1];
    struct Ent { int32_t col, row; int64_t q; };
    std::vector<Ent> ent;  // block entries in CSR order (rows ascending), then stably by column
    for (int64_t r = r0; r < r1; r++)
      for (int64_t q = At.ptr[r]; q < At.ptr[r + 1]; q++) ent.push_back({At.col[q], (int32_t)(r - r0), q});
    std::stable_sort(ent.begin(), ent.end(), [](const Ent& a, const Ent& c) { return a.col < c.col; });
    k->cptr_off.push_back((int32_t)cptr.size());
    k->centry_off.push_back((int64_t)crow.size());
    int32_t nc = 0;
    const int64_t e0 = (int64_t)crow.size();
    for (size_t e = 0; e < ent.size(); e++) {
      if (e == 0 || ent[e].col != ent[e - 1].col) {
        cptr.push_back((int32_t)((int64_t)crow.size() - e0));
        ccol.push_back(ent[e].col);
        nc++;
      }
      crow.push_back(ent[e].row);
      cval.push_back(At.val[ent[e].q]);
    }
    cptr.push_back((int32_t)((int64_t)crow.size() - e0));
    k->ncols.push_back(nc);
  }
  // (cptr block b occupies ncols[b] + 1 entries from cptr_off[b]; ccol has ncols[b] entries per
  //  block, so block b's ccol starts at cptr_off[b] - b)
  cudaError_t e = cudaSuccess;
  g.reserve(tot);
  for (auto& v : ginv) g.insert(g.end(), v.begin(), v.end());
  std::vector<std::vector<double>>().swap(ginv);
  if (e == cudaSuccess) e = k5_upload(*k, &k->ginv, g.data(), g.size());
  if (e == cudaSuccess) e = k5_upload(*k, &k->cptr, cptr.data(), cptr.size());
  if (e == cudaSuccess) e = k5_upload(*k, &k->ccol, ccol.data(), ccol.size());
  if (e == cudaSuccess) e = k5_upload(*k, &k->crow, crow.data(), crow.size());
  if (e == cudaSuccess) e = k5_upload(*k, &k->cval, cval.data(), cval.size());
  if (e == cudaSuccess) e = k5_upload(*k, &k->r, (const double*)nullptr, (size_t)bmax);
  if (e == cudaSuccess) e = k5_upload(*k, &k->y, (const double*)nullptr, (size_t)bmax);
  if (e != cudaSuccess) {
    why = std::string("device upload failed: ") + cudaGetErrorString(e);
    return false;
  }
  return true;
}

namespace {
cudaError_t build_graph(Plan& p) {
  K5Plan& k = *p.k5;
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
  e = capture_sweep(p, k, cs, nodes);
  cudaError_t e2 = launch_check_graph(p, cs, h);
  nodes++;
  cudaGraph_t out;
  cudaError_t e3 = cudaStreamEndCapture(cs, &out);
  cudaStreamDestroy(cs);
  if (e != cudaSuccess) return e;
  if (e2 != cudaSuccess) return e2;
  if (e3 != cudaSuccess) return e3;
  if ((e = cudaGraphInstantiate(&k.exec, g, 0)) != cudaSuccess) return e;
  k.graph = g;
  k.nodes_per_sweep = nodes;
  return cudaSuccess;
}
}  // namespace

cudaError_t k5_solve(Plan& p, cudaStream_t s, long long& launches) {
  cudaError_t e;
  (void)launches;
  if (!p.k5->exec && (e = build_graph(p)) != cudaSuccess) return e;
  return cudaGraphLaunch(p.k5->exec, s);
}

long long k5_nodes_per_sweep(const Plan& p) { return p.k5 ? p.k5->nodes_per_sweep : 0; }

const BlockLayout* k5_layout(const Plan& p) { return p.k5 ? &p.k5->L : nullptr; }

void k5_free(Plan& p) {
  if (!p.k5) return;
  if (p.k5->exec) cudaGraphExecDestroy(p.k5->exec);
  if (p.k5->graph) cudaGraphDestroy(p.k5->graph);
  for (void* v : p.k5->allocs) cudaFree(v);
  delete p.k5;
  p.k5 = nullptr;
}

}  // namespace pobk
