// K4: one thread-block cluster holds the whole system in distributed shared memory (mid-size
// systems, e.g. BASELINE config 2: m = 20,000, 178k nonzeros, 2.1 MB -- too big for one CTA's
// shared memory).  An explicit option (kernel = CLUSTER), not chosen by AUTO: measured on config 2
// at 89.5 us/sweep vs K2's 72.8 (a step costs ~2.8 us: the cluster barrier, ~450 cycles alone
// (tools/microbench/mb12.cu), waits on every CTA's scattered DSMEM stores, one transaction per
// lane; routing local columns through plain LDS/STS measured slower still, 152 us).
//
// x~ is split by RCM column ranges over the C CTAs of the cluster (C = 16 where the GPU can
// co-schedule it, else 8, 4, 2); a row runs on the CTA that owns its diagonal column.  Each CTA
// keeps its rows as a thread-major ELL per schedule step (as K3E) and reads / writes x~ through
// the cluster's shared-memory window (ld/st.shared::cluster; RCM makes most columns local or on a
// neighbouring CTA).  Rows of one category touch disjoint columns, so the writes of
// a step never collide; one cluster barrier (release/acquire) per step orders the steps (Alg 5
// loop).  Per-row arithmetic: the common.cuh contract, so the iterates are
// bitwise the oracle's.  Stop test: every CTA reduces its owned columns,
// CTA 0's shared memory gathers the C partials, every thread of every CTA forms the same
// fixed-order total and takes the same decision.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>

#include "../plan.h"
#include "common.cuh"

namespace pobk {

namespace {
constexpr int kCNT = 256;  // threads per CTA
constexpr int kCW = 24;    // max entries per row (held in registers)
constexpr int kMaxC = 16;

struct K4Args {
  int m, nsteps, C, chunk;
  int ent_max, slot_max;
  const uint32_t* ecol;  // [C][ent_max] (owner CTA << 24) | local column; padding: own zero slot
  const double* eval;    // [C][ent_max]
  const int2* einfo;     // [C][nsteps] {blocks, first block}
  const int4* eblk;      // [C][blk_max] {ELL base, rows R <= 32, width W, first row slot}
  int blk_max;
  const int32_t* eslot;  // [C][slot_max] storage index of each row slot (-1: none)
  const double* nrm2;    // [m] storage order
  const double* fs;      // [m] storage order
  double* xt;            // [m] RCM frame
  const double* xst;     // [m] RCM frame (RSE) or NULL
  Ctrl* ctrl;
  long long* trace;      // development (POBK_K4_TRACE): [8] mean cycles per phase, CTA 0 warp 0
};

__host__ __device__ inline size_t al16(size_t b) { return (b + 15) & ~size_t(15); }
struct K4Layout {
  size_t o_val, o_col, o_x, o_xs, o_f, o_n, o_info, o_blk, o_part, o_red, bytes;
  __host__ __device__ K4Layout(int ent_max, int slot_max, int chunk, int nsteps, int blk_max) {
    size_t o = 0;
    o_val = o; o += al16(8ull * ent_max);
    o_col = o; o += al16(4ull * ent_max);
    o_x = o; o += al16(8ull * (chunk + 1));
    o_xs = o; o += al16(8ull * chunk);
    o_f = o; o += al16(8ull * slot_max);
    o_n = o; o += al16(8ull * slot_max);
    o_info = o; o += al16(8ull * nsteps);
    o_blk = o; o += al16(16ull * blk_max);
    o_part = o; o += al16(8ull * 2 * kMaxC);
    o_red = o; o += al16(8ull * (kCNT / 32));
    bytes = o;
  }
};

__device__ __forceinline__ unsigned cta_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned mapa(unsigned a, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ double ldc(unsigned a) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
  return v;
}
// eight remote loads in one asm block: all in flight before any consumer (ptxas would otherwise
// hoist each product next to its load and stall the in-order issue on every ~215-cycle access)
__device__ __forceinline__ void ldc8(double (&v)[8], const unsigned (&a)[8]) {
  asm volatile(
      "ld.shared::cluster.f64 %0, [%8];\n ld.shared::cluster.f64 %1, [%9];\n ld.shared::cluster.f64 %2, [%10];\n"
      " ld.shared::cluster.f64 %3, [%11];\n ld.shared::cluster.f64 %4, [%12];\n ld.shared::cluster.f64 %5, [%13];\n"
      " ld.shared::cluster.f64 %6, [%14];\n ld.shared::cluster.f64 %7, [%15];"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]), "=d"(v[4]), "=d"(v[5]), "=d"(v[6]), "=d"(v[7])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7])
      : "memory");
}
__device__ __forceinline__ void stc(unsigned a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

__global__ void __launch_bounds__(kCNT, 1) k4_sweeps(K4Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const K4Layout L(a.ent_max, a.slot_max, a.chunk, a.nsteps, a.blk_max);
  double* val = (double*)(smem + L.o_val);
  uint32_t* col = (uint32_t*)(smem + L.o_col);
  double* x = (double*)(smem + L.o_x);
  double* xs = (double*)(smem + L.o_xs);
  double* f = (double*)(smem + L.o_f);
  double* nr = (double*)(smem + L.o_n);
  int2* info = (int2*)(smem + L.o_info);
  int4* blk = (int4*)(smem + L.o_blk);
  double* part = (double*)(smem + L.o_part);
  double* red = (double*)(smem + L.o_red);
  const unsigned rank = cta_rank();
  const int tid = threadIdx.x;
  const int c0 = (int)rank * a.chunk, nown = max(0, min(a.chunk, a.m - c0));

  for (int i = tid; i < a.ent_max; i += kCNT) {
    val[i] = a.eval[(size_t)rank * a.ent_max + i];
    col[i] = a.ecol[(size_t)rank * a.ent_max + i];
  }
  for (int i = tid; i < a.chunk; i += kCNT) {
    x[i] = i < nown ? a.xt[c0 + i] : 0.0;
    xs[i] = (i < nown && a.xst) ? a.xst[c0 + i] : 0.0;
  }
  if (tid == 0) x[a.chunk] = 0.0;  // zero slot of the ELL padding (never written)
  for (int i = tid; i < a.slot_max; i += kCNT) {
    const int sidx = a.eslot[(size_t)rank * a.slot_max + i];
    f[i] = sidx >= 0 ? a.fs[sidx] : 0.0;
    nr[i] = sidx >= 0 ? a.nrm2[sidx] : 1.0;
  }
  for (int i = tid; i < a.nsteps; i += kCNT) info[i] = a.einfo[(size_t)rank * a.nsteps + i];
  for (int i = tid; i < a.blk_max; i += kCNT) blk[i] = a.eblk[(size_t)rank * a.blk_max + i];
  const int warp = tid >> 5, lane = tid & 31;
  const long long maxs = a.ctrl->max_sweeps;
  const int mode = a.ctrl->stop_mode, every = a.ctrl->check_every;
  const long long off = a.ctrl->offset;
  const double tol = a.ctrl->tol, den = a.ctrl->den;
  cluster_sync();  // every CTA's x~ is in place before any remote access

  const unsigned xbase = (unsigned)__cvta_generic_to_shared(x);
  const unsigned pbase0 = mapa((unsigned)__cvta_generic_to_shared(part), 0u);  // CTA 0's partials
  long long sweep = 0;
  double value = NAN;
  int term = POBK_TERM_MAX_SWEEPS;
  bool stop = maxs <= 0;
  while (!stop) {
    for (int k = 0; k < a.nsteps; k++) {
      long long tk0 = a.trace ? clock64() : 0;
      const int2 in = info[k];  // {blocks, first block}: a step's rows of this CTA, <= 32 per block
      for (int b = warp; b < in.x; b += kCNT / 32) {
        const int4 bk = blk[in.y + b];  // {ELL base, R, W, first slot}
        if (lane < bk.y) {
          const int W = bk.z, R = bk.y, e0 = bk.x + lane, slot = bk.w + lane;
          unsigned ra[kCW];
          double av[kCW], xv[kCW];
          unsigned real = 0u;  // bit j: entry j is a stored nonzero (not ELL padding)
#pragma unroll
          for (int j = 0; j < kCW; j++) {
            const int jj = j < W ? j : W - 1;  // (entries >= W: a valid address, result unused)
            const uint32_t c = col[e0 + jj * R];
            av[j] = j < W ? val[e0 + jj * R] : 0.0;
            ra[j] = mapa(xbase + 8u * (c & 0xffffffu), c >> 24);
            real |= (j < W && (c & 0xffffffu) != (uint32_t)a.chunk) ? (1u << j) : 0u;
          }
#pragma unroll
          for (int jb = 0; jb < kCW; jb += 8)
            if (jb < W) {
              double v8[8];
              unsigned a8[8];
#pragma unroll
              for (int u = 0; u < 8; u++) a8[u] = ra[jb + u];
              ldc8(v8, a8);
#pragma unroll
              for (int u = 0; u < 8; u++) xv[jb + u] = v8[u];
            }
          if (a.trace && rank == 0 && tid == 0) {
#pragma unroll
            for (int j = 0; j < kCW; j++) asm volatile("mov.b64 %0, %0;" : "+d"(xv[j]));
            a.trace[1] += clock64() - tk0;
          }
          double sum = 0.0, pp[kCW];
#pragma unroll
          for (int j = 0; j < kCW; j++)
            if (j < W) pp[j] = pin(__dmul_rn(av[j], xv[j]));
#pragma unroll
          for (int j = 0; j < kCW; j++)
            if (j < W) sum = __dadd_rn(sum, pp[j]);
          const double alpha = __ddiv_rn(__dsub_rn(f[slot], sum), nr[slot]);
          double xn[kCW];
#pragma unroll
          for (int j = 0; j < kCW; j++) xn[j] = __dadd_rn(xv[j], __dmul_rn(alpha, av[j]));
#pragma unroll
          for (int j = 0; j < kCW; j++)  // padding entries (value +0, the zero slot): not stored
            if ((real >> j) & 1u) stc(ra[j], xn[j]);
          if (a.trace && rank == 0 && tid == 0) a.trace[2] += clock64() - tk0;
        }
      }
      if (a.trace && rank == 0 && tid == 0) a.trace[3] += clock64() - tk0;
      cluster_sync();
      if (a.trace && rank == 0 && tid == 0) { a.trace[4] += clock64() - tk0; a.trace[0] += 1; }
    }
    sweep++;
    const bool due = mode != POBK_STOP_NONE && (((sweep + off) % every) == 0 || sweep >= maxs);
    if (due) {
      double loc = 0.0;
      if (mode == POBK_STOP_RSE) {
        for (int i = tid; i < nown; i += kCNT) { const double d = x[i] - xs[i]; loc = fma(d, d, loc); }
      } else {  // RELRES: this CTA's rows, row by row from its ELL (x~ through the window)
        for (int k = 0; k < a.nsteps; k++) {
          const int2 in = info[k];
          for (int b = warp; b < in.x; b += kCNT / 32) {
            const int4 bk = blk[in.y + b];
            if (lane < bk.y) {
              double sum = 0.0;
              for (int j = 0; j < bk.z; j++) {
                const uint32_t c = col[bk.x + lane + j * bk.y];
                sum = __dadd_rn(sum, __dmul_rn(val[bk.x + lane + j * bk.y], ldc(mapa(xbase + 8u * (c & 0xffffffu), c >> 24))));
              }
              const double r = __dsub_rn(f[bk.w + lane], sum);
              loc = fma(r, r, loc);
            }
          }
        }
      }
      const double tot_cta = block_sum<kCNT>(loc, red);
      const int par = (int)(sweep & 1);
      if (tid == 0) stc(pbase0 + 8u * (unsigned)(par * kMaxC + (int)rank), tot_cta);
      cluster_sync();
      double tot = 0.0;  // the same fixed order in every thread of every CTA
      for (int q = 0; q < a.C; q++) tot += ldc(pbase0 + 8u * (unsigned)(par * kMaxC + q));
      value = sqrt(tot) / sqrt(den);
      if (!isfinite(value)) { term = POBK_TERM_NONFINITE; stop = true; }
      else if (value < tol) { term = POBK_TERM_CONVERGED; stop = true; }
    }
    if (!stop && sweep >= maxs) { term = POBK_TERM_MAX_SWEEPS; stop = true; }
  }
  for (int i = tid; i < nown; i += kCNT) a.xt[c0 + i] = x[i];
  if (rank == 0 && tid == 0) {
    a.ctrl->sweeps = sweep;
    a.ctrl->value = value;
    a.ctrl->term = term;
    a.ctrl->stopped = 1;
  }
  cluster_sync();  // no CTA leaves while another may still read its shared memory
}
}  // namespace

struct K4Plan {
  int C = 0, chunk = 0, ent_max = 0, slot_max = 0, blk_max = 0;
  size_t smem = 0;
  uint32_t* ecol = nullptr;
  double* eval = nullptr;
  int2* einfo = nullptr;
  int4* eblk = nullptr;
  int32_t* eslot = nullptr;
};

// Build the cluster layout from the schedule-order CSR (rp/col/val: storage order s, rows of a
// step contiguous; sched.rows[s] = RCM row).  Returns false (with why) when the system does not
// fit a cluster; the plan then uses another kernel family.
bool k4_build(Plan& p, const std::vector<int32_t>& rp, const std::vector<int32_t>& col, const std::vector<double>& val,
              std::string& why) {
  if (p.any_overlap) { why = "overlapping categories"; return false; }
  const int64_t m = p.m;
  for (int64_t s = 0; s < m; s++)
    if (rp[s + 1] - rp[s] > kCW) { why = "a row has more than " + std::to_string(kCW) + " nonzeros"; return false; }
  cudaError_t e = cudaFuncSetAttribute(k4_sweeps, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) { why = cudaGetErrorString(e); return false; }
  const int cmax = getenv("POBK_K4_CMAX") ? atoi(getenv("POBK_K4_CMAX")) : 16;  // development override
  for (int C : {16, 8, 4, 2}) {
    if (C > cmax) continue;
    const int chunk = (int)((m + C - 1) / C);
    if (chunk >= (1 << 24)) continue;
    // rows per (CTA, step) in schedule order, then sorted by length (longest first) and cut into
    // blocks of <= 32 rows with their own ELL width (little padding)
    std::vector<std::vector<int32_t>> srows((size_t)C * p.nsteps);
    for (int k = 0; k < p.nsteps; k++)
      for (int s = p.h_step_ptr[k]; s < p.h_step_ptr[k + 1]; s++) {
        const int q = p.sched.rows[s] / chunk;
        srows[(size_t)q * p.nsteps + k].push_back(s);
      }
    auto len = [&](int32_t s) { return rp[s + 1] - rp[s]; };
    std::vector<int2> hinfo((size_t)C * p.nsteps);
    std::vector<std::vector<int4>> hblk(C);
    std::vector<int> ent(C, 0), slots(C, 0);
    for (int q = 0; q < C; q++)
      for (int k = 0; k < p.nsteps; k++) {
        auto& v = srows[(size_t)q * p.nsteps + k];
        std::stable_sort(v.begin(), v.end(), [&](int32_t x, int32_t y) { return len(x) > len(y); });
        hinfo[(size_t)q * p.nsteps + k] = make_int2(0, (int)hblk[q].size());
        for (size_t b0 = 0; b0 < v.size(); b0 += 32) {
          const int R = (int)std::min<size_t>(32, v.size() - b0), W = std::max(1, len(v[b0]));
          hblk[q].push_back(make_int4(ent[q], R, W, slots[q] + (int)b0));
          hinfo[(size_t)q * p.nsteps + k].x++;
          ent[q] += R * W;
        }
        slots[q] += (int)v.size();
      }
    int blk_max = 1;
    for (int q = 0; q < C; q++) blk_max = std::max(blk_max, (int)hblk[q].size());
    const int ent_max = std::max(1, *std::max_element(ent.begin(), ent.end()));
    const int slot_max = std::max(1, *std::max_element(slots.begin(), slots.end()));
    const K4Layout L(ent_max, slot_max, chunk, p.nsteps, blk_max);
    if (L.bytes > 227 * 1024 - 64) continue;
    // can the GPU co-schedule a cluster of C CTAs with this much shared memory?
    if ((e = raise_smem_limit((const void*)k4_sweeps)) != cudaSuccess) continue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(kCNT);
    cfg.dynamicSmemBytes = L.bytes;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, k4_sweeps, &cfg) != cudaSuccess || nclusters < 1) {
      cudaGetLastError();
      continue;
    }
    // the ELL blocks: entry j of a block's row r at base + j*R + r
    std::vector<uint32_t> ecol((size_t)C * ent_max);
    std::vector<double> eval((size_t)C * ent_max, 0.0);
    std::vector<int32_t> eslot((size_t)C * slot_max, -1);
    std::vector<int4> eblk((size_t)C * blk_max, make_int4(0, 0, 1, 0));
    for (int q = 0; q < C; q++) {
      const uint32_t pad = ((uint32_t)q << 24) | (uint32_t)chunk;  // own zero slot
      std::fill(ecol.begin() + (size_t)q * ent_max, ecol.begin() + (size_t)(q + 1) * ent_max, pad);
      std::copy(hblk[q].begin(), hblk[q].end(), eblk.begin() + (size_t)q * blk_max);
      for (int k = 0; k < p.nsteps; k++) {
        const int2 in = hinfo[(size_t)q * p.nsteps + k];
        const auto& v = srows[(size_t)q * p.nsteps + k];
        for (int b = 0; b < in.x; b++) {
          const int4 bk = hblk[q][in.y + b];
          for (int r = 0; r < bk.y; r++) {
            const int32_t s = v[(size_t)b * 32 + r];
            for (int j = 0; j < len(s); j++) {
              const int32_t c = col[rp[s] + j];
              const size_t e = (size_t)q * ent_max + bk.x + (size_t)j * bk.y + r;
              ecol[e] = ((uint32_t)(c / chunk) << 24) | (uint32_t)(c % chunk);
              eval[e] = val[rp[s] + j];
            }
            eslot[(size_t)q * slot_max + bk.w + r] = s;
          }
        }
      }
    }
    K4Plan* k = new K4Plan();
    k->C = C;
    k->chunk = chunk;
    k->ent_max = ent_max;
    k->slot_max = slot_max;
    k->blk_max = blk_max;
    k->smem = L.bytes;
    auto up = [&](auto** dst, const auto* src, size_t n) -> cudaError_t {
      void* v = nullptr;
      cudaError_t r = cudaMalloc(&v, n * sizeof(*src));
      if (r != cudaSuccess) return r;
      p.allocations.push_back(v);
      *dst = (std::remove_reference_t<decltype(**dst)>*)v;
      return cudaMemcpy(v, src, n * sizeof(*src), cudaMemcpyHostToDevice);
    };
    if ((e = up(&k->ecol, ecol.data(), ecol.size())) != cudaSuccess || (e = up(&k->eval, eval.data(), eval.size())) != cudaSuccess ||
        (e = up(&k->einfo, hinfo.data(), hinfo.size())) != cudaSuccess || (e = up(&k->eblk, eblk.data(), eblk.size())) != cudaSuccess ||
        (e = up(&k->eslot, eslot.data(), eslot.size())) != cudaSuccess) {
      delete k;
      why = std::string("device upload failed: ") + cudaGetErrorString(e);
      return false;
    }
    p.k4 = k;
    if (getenv("POBK_K4_VERBOSE"))
      fprintf(stderr, "[k4] cluster of %d CTAs, %d columns each, %d ELL entries, %d blocks, %zu B shared memory per CTA\n", C,
              chunk, ent_max, blk_max, L.bytes);
    return true;
  }
  why = "the system does not fit one thread-block cluster's shared memory";
  return false;
}

cudaError_t k4_solve(Plan& p, cudaStream_t s, long long& launches) {
  K4Plan& k = *p.k4;
  K4Args a;
  a.m = (int)p.m;
  a.nsteps = p.nsteps;
  a.C = k.C;
  a.chunk = k.chunk;
  a.ent_max = k.ent_max;
  a.slot_max = k.slot_max;
  a.ecol = k.ecol;
  a.eval = k.eval;
  a.einfo = k.einfo;
  a.eblk = k.eblk;
  a.blk_max = k.blk_max;
  a.eslot = k.eslot;
  a.nrm2 = p.A.nrm2;
  a.fs = p.d_fs;
  a.xt = p.d_xt;
  a.xst = p.d_xst;
  a.ctrl = p.d_ctrl;
  a.trace = nullptr;
  static long long* tr = nullptr;
  if (getenv("POBK_K4_TRACE")) {
    if (!tr) cudaMalloc(&tr, 64);
    cudaMemsetAsync(tr, 0, 64, s);
    a.trace = tr;
  }
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k4_sweeps, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess) return e;
  if ((e = raise_smem_limit((const void*)k4_sweeps)) != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(k.C);
  cfg.blockDim = dim3(kCNT);
  cfg.dynamicSmemBytes = k.smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = k.C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  launches++;
  e = cudaLaunchKernelEx(&cfg, k4_sweeps, a);
  if (e == cudaSuccess && a.trace) {
    long long h[8];
    cudaMemcpyAsync(h, a.trace, 64, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (h[0] > 0)
      fprintf(stderr, "[k4 trace] steps %lld, cycles/step: to loaded %.0f, to stored %.0f, to step end %.0f, to after sync %.0f\n",
              h[0], (double)h[1] / h[0], (double)h[2] / h[0], (double)h[3] / h[0], (double)h[4] / h[0]);
  }
  return e;
}

void k4_free(Plan& p) {
  delete p.k4;  // (device buffers are in p.allocations)
  p.k4 = nullptr;
}

int k4_cluster_size(const Plan& p) { return p.k4 ? p.k4->C : 0; }

}  // namespace pobk
