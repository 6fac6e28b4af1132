// K2: persistent tiled wavefront sweep.
//
// The rows of A~ are split into T tiles (one CTA per SM, cooperative launch).  A schedule step
// (a category of pairwise-orthogonal rows) restricted to one tile is a "task".
// Sequential semantics of the sweep (Alg 5 loop) only constrain rows that share
// a column, so a tile's task k may run as soon as every NEIGHBOUR tile (one sharing a column with
// it) has finished its tasks < k: per-tile progress counters (release/acquire at gpu scope)
// replace the grid-wide barrier between categories.  Results are bitwise those of K1/K3 (same
// per-row contract, common.cuh).
//
//   x~ columns touched by one tile only ("private") live in that CTA's shared memory for the
//   whole solve; the rest ("shared") live in global memory and are accessed at L2 (ld/st .cg).
//   Within a task, rows touching only private columns ("interior") run before the neighbour wait;
//   rows touching a shared column ("boundary") run after it.
//
//   The tile's matrix data (val, col, row extents, f~, ||a~_i||^2) is a sequence of <= 28 KB chunks
//   streamed by 1-D TMA (cp.async.bulk) into a 4-slot shared-memory ring, S-1 chunks ahead of the
//   consumer and across task and sweep boundaries (A does not depend on x~).
//
//   The RSE is accumulated by the LAST writer of every column in the sweep (the row
//   of highest step touching it), so no extra pass over x~ is needed; a grid-wide last-arriver
//   reduction in tile order decides the stop once per checked sweep.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <set>
#include <string>
#include <vector>

#include "../plan.h"
#include "common.cuh"

namespace pobk {

namespace {
constexpr int kNT = 1024;          // threads per CTA
constexpr int kSlots = 3;          // TMA ring depth
constexpr int kChunkCap = 40 * 1024;
constexpr int kNbMax = 16;         // max neighbour tiles
constexpr int kMaxChunks = 1024;   // max chunks per tile (chunk metadata lives in shared memory)
constexpr int kFlagStride = 32;    // ints between progress counters (one 128-B line each)
constexpr int kSmemLimit = 227 * 1024;
constexpr unsigned kShared = 0x80000000u, kLast = 0x40000000u, kIdx = 0x3FFFFFFFu;
constexpr int kFirstBoundary = 1, kLastOfTask = 2;

__host__ __device__ inline int a16(long long b) { return (int)((b + 15) & ~15LL); }

// chunk block layout (bytes, each section 16-B aligned): val[nnz] f[rows] nrm2[rows] col[nnz] rp[rows+1]
struct ChunkLayout {
  int o_val, o_f, o_n, o_col, o_rp, bytes;
  __host__ __device__ ChunkLayout(int rows, int nnz) {
    o_val = 0;
    o_f = a16(8LL * nnz);
    o_n = o_f + a16(8LL * rows);
    o_col = o_n + a16(8LL * rows);
    o_rp = o_col + a16(4LL * nnz);
    bytes = o_rp + a16(4LL * (rows + 1));
  }
};

struct ChunkMeta {
  int rows, nnz, step, flags;
  int k_next;   // last chunk of a task: the tile's next task step (>= nsteps: next sweep)
  int pad0, pad1, pad2;
  long long off;  // byte offset of the block in the stream
};

struct SyncState {
  unsigned int arrive[2];
  int pad0[30];
  int epoch;      // = sweeps decided
  int stop;
  int pad1[30];
};

struct K2Args {
  const unsigned char* stream;
  const long long* tile_off;  // [T] byte offset of each tile's first chunk
  const ChunkMeta* meta;
  const int* tile_chunk;  // [T+1]
  const int* nbr;         // [T*kNbMax], -1 padded
  const int* pmap_ptr;    // [T+1]
  const int* pmap;        // private columns (global ids), tile by tile
  const int* k_first;     // [T]
  double* xg;             // x~ (RCM frame); authoritative for shared columns
  const double* xst;      // x~*
  int* progress;          // [T*kFlagStride]
  SyncState* sync;
  double* partials;       // [2*T]
  Ctrl* ctrl;
  int nsteps, T;
  int nck_max, np_max;  // shared-memory sizing
  unsigned long long* prof;  // optional [T*8] phase clocks (POBK_K2_PROFILE=1), else NULL
  int debug;                 // development-only timing experiments (POBK_K2_DEBUG): 1 relaxed publish, 2 no wait
};

// ------------------------------------------------------------------ PTX helpers (TMA, mbarrier)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
// 1-D bulk copy global -> shared, completing on an mbarrier; the matrix stream is read once per
// sweep and must not evict x~ from L2, so it carries an L2 evict-first policy.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* b,
                                            unsigned long long policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ unsigned long long policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}

template <int V>
__global__ void __launch_bounds__(kNT, 1) k2_sweeps(K2Args a) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* ring = smem;                                             // kSlots * kChunkCap
  unsigned long long* mbar = (unsigned long long*)(smem + kSlots * kChunkCap);
  double* red = (double*)(mbar + 4);                                      // 32 doubles (mbar area padded to 32 B)
  int4* cmeta = (int4*)(red + 32);                                        // [nck_max] {rows, nnz, step<<2|flags, k_next}
  int* coff = (int*)(cmeta + a.nck_max);                                  // [nck_max] byte offset from the tile base
  double* xloc = (double*)(coff + ((a.nck_max + 3) & ~3));                // [np_max] private x~
  double* xsloc = xloc + a.np_max;                                        // [np_max] private x~* (RSE stop)
  __shared__ int s_stop;

  const int t = blockIdx.x, tid = threadIdx.x;
  const int c0 = a.tile_chunk[t], nck = a.tile_chunk[t + 1] - c0;
  const int q0 = a.pmap_ptr[t], np = a.pmap_ptr[t + 1] - q0;
  const int nsteps = a.nsteps;
  const long long maxs = a.ctrl->max_sweeps;
  const int mode = a.ctrl->stop_mode, every = a.ctrl->check_every;
  const double tol = a.ctrl->tol, den = a.ctrl->den;
  const unsigned char* tbase = a.stream + a.tile_off[t];

  if (tid == 0) {
    for (int i = 0; i < kSlots; i++) mbar_init(mbar + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_stop = 0;
  }
  for (int j = tid; j < nck; j += kNT) {
    const ChunkMeta mt = a.meta[c0 + j];
    cmeta[j] = make_int4(mt.rows, mt.nnz, (mt.step << 2) | mt.flags, mt.k_next);
    coff[j] = (int)(mt.off - a.tile_off[t]);
  }
  for (int j = tid; j < np; j += kNT) {
    const int gcol = a.pmap[q0 + j];
    xloc[j] = a.xg[gcol];
    xsloc[j] = (mode == POBK_STOP_RSE) ? a.xst[gcol] : 0.0;
  }
  __syncthreads();

  const unsigned long long pol = policy_evict_first();
  auto issue = [&](long long g) {  // thread 0 only
    const int slot = (int)(g % kSlots);
    const int c = (int)(g % nck);
    const int4 mt = cmeta[c];
    const int bytes = ChunkLayout(mt.x, mt.y).bytes;
    mbar_expect_tx(mbar + slot, bytes);
    tma_load_1d(ring + slot * kChunkCap, tbase + coff[c], bytes, mbar + slot, pol);
  };
  long long issued = 0;
  if (tid == 0 && nck > 0)
    for (; issued < kSlots - 1; issued++) issue(issued);

  const int lane = tid % V, vec = tid / V, nvec = kNT / V;
  const int warp = tid >> 5, wl = tid & 31;
  int my_nb = -1;  // warp 0: lane j polls neighbour j
  if (warp == 0 && wl < kNbMax) my_nb = a.nbr[t * kNbMax + wl];
  double acc_rse = 0.0;
  long long sweep = 0, g = 0;
  unsigned long long pr[6] = {0, 0, 0, 0, 0, 0};  // nbwait, mbarwait, compute, publish, barrier, total
  const unsigned long long t_start = clock64();
  while (true) {
    acc_rse = 0.0;  // only the checked sweep's last-writer events count
    for (int i = 0; i < nck; i++, g++) {
      if (tid == 0) {
        issue(issued);
        issued++;
      }
      const int4 mt = cmeta[i];
      const int rows = mt.x, nnz = mt.y, step = mt.z >> 2, flags = mt.z & 3;
      unsigned long long c_a = clock64();
      if ((flags & kFirstBoundary) && !(a.debug & 2)) {
        if (warp == 0) {
          const int need = (int)(sweep * nsteps + step);
          if (my_nb >= 0) {
            const int* pf = a.progress + my_nb * kFlagStride;
            while (ld_acquire(pf) < need) {
            }
          }
          __syncwarp();
        }
        __syncthreads();
      }
      const int slot = (int)(g % kSlots);
      unsigned long long c_b = clock64();
      mbar_wait(mbar + slot, (unsigned)((g / kSlots) & 1));
      unsigned long long c_c = clock64();
      const unsigned char* blk = ring + slot * kChunkCap;
      const ChunkLayout L(rows, nnz);
      const double* val = (const double*)(blk + L.o_val);
      const double* fv = (const double*)(blk + L.o_f);
      const double* nv = (const double*)(blk + L.o_n);
      const unsigned* col = (const unsigned*)(blk + L.o_col);
      const int* rp = (const int*)(blk + L.o_rp);
      for (int base = 0; base < rows; base += nvec) {
        const int r = base + vec;
        const bool act = r < rows;
        const int p0 = act ? rp[r] : 0, p1 = act ? rp[r + 1] : 0;
        constexpr int KC = 4;
        unsigned cc[KC];
        double av[KC], xv[KC], sv[KC];
#pragma unroll
        for (int j = 0; j < KC; j++) {
          const int p = p0 + lane + j * V;
          cc[j] = p < p1 ? col[p] : 0u;
          av[j] = p < p1 ? val[p] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < KC; j++) {
          const int p = p0 + lane + j * V;
          const unsigned c = cc[j], idx = c & kIdx;
          xv[j] = 0.0;
          sv[j] = 0.0;
          if (p < p1) {
            if (c & kShared) {
              xv[j] = ld_cg(a.xg + idx);
              if (c & kLast) sv[j] = __ldg(a.xst + idx);
            } else {
              xv[j] = xloc[idx];
              if (c & kLast) sv[j] = xsloc[idx];
            }
          }
        }
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < KC; j++)
          if (p0 + lane + j * V < p1) acc = fma(av[j], xv[j], acc);
        for (int p = p0 + lane + KC * V; p < p1; p += V) {
          const unsigned c = col[p];
          acc = fma(val[p], (c & kShared) ? ld_cg(a.xg + (c & kIdx)) : xloc[c & kIdx], acc);
        }
        acc = vec_sum<V>(acc);
        if (act) {
          const double alpha = (fv[r] - acc) / nv[r];
#pragma unroll
          for (int j = 0; j < KC; j++)
            if (p0 + lane + j * V < p1) {
              const unsigned c = cc[j], idx = c & kIdx;
              const double xn = fma(alpha, av[j], xv[j]);
              if (c & kShared) st_cg(a.xg + idx, xn);
              else xloc[idx] = xn;
              if (c & kLast) {
                const double d = xn - sv[j];
                acc_rse = fma(d, d, acc_rse);
              }
            }
          for (int p = p0 + lane + KC * V; p < p1; p += V) {
            const unsigned c = col[p], idx = c & kIdx;
            const double xo = (c & kShared) ? ld_cg(a.xg + idx) : xloc[idx];
            const double xn = fma(alpha, val[p], xo);
            if (c & kShared) st_cg(a.xg + idx, xn);
            else xloc[idx] = xn;
            if (c & kLast) {
              const double d = xn - ((c & kShared) ? __ldg(a.xst + idx) : xsloc[idx]);
              acc_rse = fma(d, d, acc_rse);
            }
          }
        }
      }
      __syncthreads();  // slot free; the task's writes are complete before publishing
      unsigned long long c_d = clock64();
      if ((flags & kLastOfTask) && tid == 0) {
        if (a.debug & 1) asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(a.progress + t * kFlagStride), "r"((int)(sweep * nsteps + mt.w)) : "memory");
        else st_release(a.progress + t * kFlagStride, (int)(sweep * nsteps + mt.w));
      }
      if (a.prof && tid == 0) {
        const unsigned long long c_e = clock64();
        pr[0] += c_b - c_a; pr[1] += c_c - c_b; pr[2] += c_d - c_c; pr[3] += c_e - c_d;
      }
    }
    const unsigned long long c_f = clock64();
    sweep++;
    const bool due = mode != POBK_STOP_NONE && ((sweep % every) == 0 || sweep >= maxs);
    if (due) {
      const double part = block_sum<kNT>(mode == POBK_STOP_RSE ? acc_rse : 0.0, red);
      if (tid == 0) {
        const int par = (int)(sweep & 1);
        a.partials[par * a.T + t] = part;
        __threadfence();
        const unsigned old = atomicAdd(&a.sync->arrive[par], 1u);
        if (old == (unsigned)a.T - 1) {
          __threadfence();
          double tot = 0.0;
          for (int b = 0; b < a.T; b++) tot += ld_cg(a.partials + par * a.T + b);
          const double v = sqrt(tot) / sqrt(den);
          int stop = 0, term = POBK_TERM_MAX_SWEEPS;
          if (!isfinite(v)) { stop = 1; term = POBK_TERM_NONFINITE; }
          else if (v < tol) { stop = 1; term = POBK_TERM_CONVERGED; }
          else if (sweep >= maxs) stop = 1;
          a.sync->arrive[par] = 0;
          a.sync->stop = stop;
          a.ctrl->value = v;
          a.ctrl->sweeps = sweep;
          a.ctrl->term = term;
          __threadfence();
          st_release(&a.sync->epoch, (int)sweep);
        } else {
          while (ld_acquire(&a.sync->epoch) < (int)sweep) {
          }
        }
        s_stop = ld_relaxed(&a.sync->stop);
      }
      __syncthreads();
      if (a.prof && tid == 0) pr[4] += clock64() - c_f;
      if (s_stop) break;
    } else if (sweep >= maxs) {
      if (t == 0 && tid == 0) {
        a.ctrl->sweeps = sweep;
        a.ctrl->term = POBK_TERM_MAX_SWEEPS;
      }
      break;
    }
  }
  if (a.prof && tid == 0) {
    pr[5] = clock64() - t_start;
    for (int j = 0; j < 6; j++) a.prof[t * 8 + j] = pr[j];
    a.prof[t * 8 + 6] = (unsigned long long)nck;
  }
  // drain TMA copies issued ahead of the stop point, then write private x~ back
  if (tid == 0)
    for (long long h = g; h < issued; h++) mbar_wait(mbar + (int)(h % kSlots), (unsigned)((h / kSlots) & 1));
  for (int j = tid; j < np; j += kNT) a.xg[a.pmap[q0 + j]] = xloc[j];
}

__global__ void k2_reset(int T, const int* k_first, int* progress, SyncState* sync) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x)
    progress[t * kFlagStride] = k_first[t];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sync->arrive[0] = sync->arrive[1] = 0;
    sync->epoch = 0;
    sync->stop = 0;
  }
}

// f (user frame) into the f~ slots of the chunk stream
__global__ void k2_scatter_f(int64_t m, const int32_t* __restrict__ orig, const int64_t* __restrict__ fslot,
                             const double* __restrict__ f, double* __restrict__ stream_d) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x)
    stream_d[fslot[q]] = f[orig[q]];
}
}  // namespace

struct K2Plan {
  int T = 0;
  size_t smem = 0;
  int nck_max = 1, np_max = 1;
  unsigned char* stream = nullptr;
  long long* tile_off = nullptr;
  unsigned long long* prof = nullptr;
  ChunkMeta* meta = nullptr;
  int *tile_chunk = nullptr, *nbr = nullptr, *pmap_ptr = nullptr, *pmap = nullptr, *k_first = nullptr;
  int* progress = nullptr;
  SyncState* sync = nullptr;
  double* partials = nullptr;
  int32_t* orig_q = nullptr;   // tile-order row -> user-frame row
  int64_t* fslot = nullptr;    // tile-order row -> double index of its f~ slot in the stream
  std::vector<void*> allocs;
  // stats (bench)
  double private_frac = 0.0;   // fraction of nnz whose column is private
  double interior_frac = 0.0;  // fraction of rows that are interior
  long long stream_bytes = 0;
  int nchunks = 0;
};

namespace {
template <typename T>
cudaError_t k2_upload(K2Plan& k, T** dst, const T* src, size_t n) {
  void* v = nullptr;
  cudaError_t e = cudaMalloc(&v, std::max<size_t>(n, 1) * sizeof(T));
  if (e != cudaSuccess) return e;
  k.allocs.push_back(v);
  *dst = (T*)v;
  if (n && src) e = cudaMemcpy(v, src, n * sizeof(T), cudaMemcpyHostToDevice);
  return e;
}

// 1-D tiler: contiguous RCM row ranges with equal nnz.
void tile_1d(const HostCSR& A, int T, std::vector<int32_t>& tile_of_row) {
  const int64_t m = A.m, nnz = A.nnz();
  tile_of_row.resize(m);
  int t = 0;
  for (int64_t i = 0; i < m; i++) {
    while (t < T - 1 && A.ptr[i] >= (int64_t)((double)nnz * (t + 1) / T)) t++;
    tile_of_row[i] = t;
  }
}
}  // namespace

bool k2_build(Plan& p, const HostCSR& At, int tile_rows, std::string& why) {
  if (p.any_overlap) { why = "overlapping categories"; return false; }
  int sms = 148;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, p.device) == cudaSuccess) sms = prop.multiProcessorCount;
  const int64_t m = p.m;
  int T = sms;
  if (tile_rows > 0) T = (int)std::max<int64_t>(1, std::min<int64_t>(sms, (m + tile_rows - 1) / tile_rows));
  T = (int)std::min<int64_t>(T, std::max<int64_t>(1, p.nnz / 4096));
  std::vector<int32_t> tile;
  tile_1d(At, T, tile);

  // step of every RCM row
  std::vector<int32_t> step_of(m);
  for (int k = 0; k < p.nsteps; k++)
    for (int q = p.sched.step_ptr[k]; q < p.sched.step_ptr[k + 1]; q++) step_of[p.sched.rows[q]] = k;

  // columns: private / shared, last writer (row of the highest step touching the column)
  std::vector<int32_t> col_tile(m, -1), last_row(m, -1);
  std::vector<uint8_t> shared(m, 0);
  for (int64_t i = 0; i < m; i++)
    for (int64_t q = At.ptr[i]; q < At.ptr[i + 1]; q++) {
      const int32_t c = At.col[q];
      if (col_tile[c] < 0) col_tile[c] = tile[i];
      else if (col_tile[c] != tile[i]) shared[c] = 1;
      if (last_row[c] < 0 || step_of[i] > step_of[last_row[c]]) last_row[c] = (int32_t)i;
    }
  // private columns per tile (ascending), capped by shared memory
  static_assert(kSlots <= 4, "mbarrier area holds 4");
  const size_t fixed = (size_t)kSlots * kChunkCap + 4 * 8 + 32 * 8;
  const int np_cap = (int)((kSmemLimit - 1024 - fixed - 20 * (size_t)kMaxChunks) / 16);  // x~ and x~* per column
  std::vector<int32_t> local(m, -1);
  std::vector<int> pmap_ptr(T + 1, 0);
  std::vector<int> pmap;
  std::vector<int> np_t(T, 0);
  {
    std::vector<std::vector<int32_t>> per(T);
    for (int64_t c = 0; c < m; c++)
      if (!shared[c] && col_tile[c] >= 0) per[col_tile[c]].push_back((int32_t)c);
    for (int t = 0; t < T; t++) {
      if ((int)per[t].size() > np_cap) {
        for (size_t j = np_cap; j < per[t].size(); j++) shared[per[t][j]] = 1;  // demote the overflow
        per[t].resize(np_cap);
      }
      pmap_ptr[t + 1] = pmap_ptr[t] + (int)per[t].size();
      for (size_t j = 0; j < per[t].size(); j++) { local[per[t][j]] = (int32_t)j; pmap.push_back(per[t][j]); }
      np_t[t] = (int)per[t].size();
    }
  }
  // neighbours: tiles sharing a column
  std::vector<std::set<int>> nbs(T);
  {
    std::vector<int64_t> cptr(m + 1, 0);
    for (int64_t q = 0; q < At.nnz(); q++) cptr[At.col[q] + 1]++;
    for (int64_t c = 0; c < m; c++) cptr[c + 1] += cptr[c];
    std::vector<int32_t> ctile(At.nnz());
    std::vector<int64_t> fill(cptr.begin(), cptr.end() - 1);
    for (int64_t i = 0; i < m; i++)
      for (int64_t q = At.ptr[i]; q < At.ptr[i + 1]; q++) ctile[fill[At.col[q]]++] = tile[i];
    std::vector<int> uniq;
    for (int64_t c = 0; c < m; c++) {
      if (!shared[c]) continue;
      uniq.assign(ctile.begin() + cptr[c], ctile.begin() + cptr[c + 1]);
      std::sort(uniq.begin(), uniq.end());
      uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
      for (size_t x = 0; x < uniq.size(); x++)
        for (size_t y = 0; y < uniq.size(); y++)
          if (x != y) nbs[uniq[x]].insert(uniq[y]);
    }
  }
  std::vector<int> nbr((size_t)T * kNbMax, -1);
  for (int t = 0; t < T; t++) {
    if ((int)nbs[t].size() > kNbMax) {
      why = "tile " + std::to_string(t) + " has " + std::to_string(nbs[t].size()) + " neighbour tiles (> " +
            std::to_string(kNbMax) + ")";
      return false;
    }
    int j = 0;
    for (int n : nbs[t]) nbr[(size_t)t * kNbMax + j++] = n;
  }
  // rows: interior (all columns private) or boundary
  std::vector<uint8_t> boundary(m, 0);
  int64_t n_private_nnz = 0, n_interior = 0;
  for (int64_t i = 0; i < m; i++) {
    for (int64_t q = At.ptr[i]; q < At.ptr[i + 1]; q++) {
      if (shared[At.col[q]]) boundary[i] = 1;
      else n_private_nnz++;
    }
    n_interior += !boundary[i];
  }
  // tasks and chunks, tile by tile
  std::vector<std::vector<std::vector<int32_t>>> rows_tk(T);  // [t][k] rows (interior first)
  for (int t = 0; t < T; t++) rows_tk[t].resize(p.nsteps);
  for (int k = 0; k < p.nsteps; k++) {
    for (int pass = 0; pass < 2; pass++)
      for (int q = p.sched.step_ptr[k]; q < p.sched.step_ptr[k + 1]; q++) {
        const int32_t r = p.sched.rows[q];
        if (boundary[r] == pass) rows_tk[tile[r]][k].push_back(r);
      }
  }
  std::vector<ChunkMeta> meta;
  std::vector<int> tile_chunk(T + 1, 0), k_first(T, p.nsteps);
  std::vector<std::vector<int32_t>> chunk_rows;
  for (int t = 0; t < T; t++) {
    std::vector<int> tasks;
    for (int k = 0; k < p.nsteps; k++)
      if (!rows_tk[t][k].empty()) tasks.push_back(k);
    if (!tasks.empty()) k_first[t] = tasks[0];
    for (size_t ti = 0; ti < tasks.size(); ti++) {
      const int k = tasks[ti];
      const int k_next = ti + 1 < tasks.size() ? tasks[ti + 1] : p.nsteps + tasks[0];
      const auto& rs = rows_tk[t][k];
      size_t a = 0;
      bool first_boundary_done = false;
      while (a < rs.size()) {
        const uint8_t kind = boundary[rs[a]];
        size_t b = a;
        int nnz = 0;
        while (b < rs.size() && boundary[rs[b]] == kind) {
          const int len = (int)(At.ptr[rs[b] + 1] - At.ptr[rs[b]]);
          if (ChunkLayout((int)(b - a + 1), nnz + len).bytes > kChunkCap) break;
          nnz += len;
          b++;
        }
        if (b == a) {
          why = "row " + std::to_string(rs[a]) + " is too long for one " + std::to_string(kChunkCap) + "-byte chunk";
          return false;
        }
        ChunkMeta mt{};
        mt.rows = (int)(b - a);
        mt.nnz = nnz;
        mt.step = k;
        mt.flags = 0;
        if (kind == 1 && !first_boundary_done) { mt.flags |= kFirstBoundary; first_boundary_done = true; }
        if (b == rs.size()) { mt.flags |= kLastOfTask; mt.k_next = k_next; }
        meta.push_back(mt);
        chunk_rows.emplace_back(rs.begin() + a, rs.begin() + b);
        a = b;
      }
    }
    tile_chunk[t + 1] = (int)meta.size();
    if (tile_chunk[t + 1] - tile_chunk[t] > kMaxChunks) {
      why = "tile " + std::to_string(t) + " needs more than " + std::to_string(kMaxChunks) + " chunks";
      return false;
    }
  }
  // stream bytes
  long long off = 0;
  for (auto& mt : meta) {
    mt.off = off;
    off += ChunkLayout(mt.rows, mt.nnz).bytes;
  }
  std::vector<unsigned char> stream(off, 0);
  std::vector<int32_t> orig_q;
  std::vector<int64_t> fslot;
  std::vector<double> nrm2(m);
  for (int64_t i = 0; i < m; i++) {
    double s = 0.0;
    for (int64_t q = At.ptr[i]; q < At.ptr[i + 1]; q++) s = s + At.val[q] * At.val[q];
    nrm2[i] = s;
  }
  p.tile_of_row.assign(tile.begin(), tile.end());
  for (size_t c = 0; c < meta.size(); c++) {
    const ChunkMeta& mt = meta[c];
    const ChunkLayout L(mt.rows, mt.nnz);
    unsigned char* blk = stream.data() + mt.off;
    double* val = (double*)(blk + L.o_val);
    double* nv = (double*)(blk + L.o_n);
    unsigned* col = (unsigned*)(blk + L.o_col);
    int* rp = (int*)(blk + L.o_rp);
    int w = 0;
    rp[0] = 0;
    for (int r = 0; r < mt.rows; r++) {
      const int32_t i = chunk_rows[c][r];
      for (int64_t q = At.ptr[i]; q < At.ptr[i + 1]; q++, w++) {
        const int32_t cg = At.col[q];
        unsigned e = shared[cg] ? (kShared | (unsigned)cg) : (unsigned)local[cg];
        if (last_row[cg] == i) e |= kLast;
        col[w] = e;
        val[w] = At.val[q];
      }
      rp[r + 1] = w;
      nv[r] = nrm2[i];
      orig_q.push_back(p.perm[i]);
      fslot.push_back((mt.off + L.o_f) / 8 + r);
    }
  }
  // upload
  K2Plan* k = new K2Plan();
  p.k2 = k;
  k->T = T;
  int nck_max = 1;
  for (int t = 0; t < T; t++) nck_max = std::max(nck_max, tile_chunk[t + 1] - tile_chunk[t]);
  k->nck_max = nck_max;
  k->np_max = std::max(1, *std::max_element(np_t.begin(), np_t.end()));
  k->smem = fixed + 16 * (size_t)nck_max + 4 * (size_t)((nck_max + 3) & ~3) + 16 * (size_t)k->np_max;
  std::vector<long long> tile_off(T, 0);
  for (int t = 0; t < T; t++) tile_off[t] = tile_chunk[t] < (int)meta.size() ? meta[tile_chunk[t]].off : 0;
  k->private_frac = p.nnz ? (double)n_private_nnz / (double)p.nnz : 0.0;
  k->interior_frac = (double)n_interior / (double)m;
  k->stream_bytes = off;
  k->nchunks = (int)meta.size();
  cudaError_t e = cudaSuccess;
#define K2_UP(dst, src, n) \
  if (e == cudaSuccess) e = k2_upload(*k, dst, src, n)
  K2_UP(&k->stream, stream.data(), stream.size());
  K2_UP(&k->tile_off, tile_off.data(), tile_off.size());
  K2_UP(&k->meta, meta.data(), meta.size());
  K2_UP(&k->tile_chunk, tile_chunk.data(), tile_chunk.size());
  K2_UP(&k->nbr, nbr.data(), nbr.size());
  K2_UP(&k->pmap_ptr, pmap_ptr.data(), pmap_ptr.size());
  K2_UP(&k->pmap, pmap.data(), pmap.size());
  K2_UP(&k->k_first, k_first.data(), k_first.size());
  K2_UP(&k->orig_q, orig_q.data(), orig_q.size());
  K2_UP(&k->fslot, fslot.data(), fslot.size());
  K2_UP(&k->progress, (int*)nullptr, (size_t)T * kFlagStride);
  K2_UP(&k->sync, (SyncState*)nullptr, 1);
  K2_UP(&k->partials, (double*)nullptr, 2 * (size_t)T);
#undef K2_UP
  if (e != cudaSuccess) {
    why = std::string("device upload failed: ") + cudaGetErrorString(e);
    k2_free(p);
    return false;
  }
  p.ntiles = T;
  return true;
}

cudaError_t k2_solve(Plan& p, const double* f_user, cudaStream_t s, long long& launches) {
  K2Plan& k = *p.k2;
  cudaError_t e;
  k2_scatter_f<<<(int)std::min<int64_t>((p.m + 255) / 256, 148 * 8), 256, 0, s>>>(p.m, k.orig_q, k.fslot, f_user,
                                                                                  (double*)k.stream);
  k2_reset<<<1, 256, 0, s>>>(k.T, k.k_first, k.progress, k.sync);
  launches += 2;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  K2Args a;
  a.stream = k.stream;
  a.tile_off = k.tile_off;
  a.nck_max = k.nck_max;
  a.prof = nullptr;
  static const int dbg = getenv("POBK_K2_DEBUG") ? atoi(getenv("POBK_K2_DEBUG")) : 0;
  a.debug = dbg;
  static const bool prof_on = getenv("POBK_K2_PROFILE") != nullptr;
  if (prof_on) {
    if (!k.prof) cudaMalloc(&k.prof, (size_t)k.T * 8 * sizeof(unsigned long long));
    a.prof = k.prof;
  }
  a.np_max = k.np_max;
  a.meta = k.meta;
  a.tile_chunk = k.tile_chunk;
  a.nbr = k.nbr;
  a.pmap_ptr = k.pmap_ptr;
  a.pmap = k.pmap;
  a.k_first = k.k_first;
  a.xg = p.d_xt;
  a.xst = p.d_xst;
  a.progress = k.progress;
  a.sync = k.sync;
  a.partials = k.partials;
  a.ctrl = p.d_ctrl;
  a.nsteps = p.nsteps;
  a.T = k.T;
  void* args[] = {&a};
  const void* fn = nullptr;
  switch (p.V) {
    case 1: fn = (const void*)k2_sweeps<1>; break;
    case 2: fn = (const void*)k2_sweeps<2>; break;
    case 4: fn = (const void*)k2_sweeps<4>; break;
    case 8: fn = (const void*)k2_sweeps<8>; break;
    case 16: fn = (const void*)k2_sweeps<16>; break;
    default: fn = (const void*)k2_sweeps<32>; break;
  }
  if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k.smem)) != cudaSuccess) return e;
  e = cudaLaunchCooperativeKernel(fn, dim3(k.T), dim3(kNT), args, k.smem, s);
  launches++;
  if (e == cudaSuccess && a.prof) {
    std::vector<unsigned long long> h((size_t)k.T * 8);
    cudaStreamSynchronize(s);
    cudaMemcpy(h.data(), a.prof, h.size() * 8, cudaMemcpyDeviceToHost);
    double sum[7] = {0}, mx[7] = {0};
    for (int t = 0; t < k.T; t++)
      for (int j = 0; j < 7; j++) { sum[j] += (double)h[t * 8 + j]; mx[j] = std::max(mx[j], (double)h[t * 8 + j]); }
    fprintf(stderr, "[k2 prof] cycles per tile (mean / max): nbwait %.3g/%.3g mbarwait %.3g/%.3g compute %.3g/%.3g "
                    "publish %.3g/%.3g barrier %.3g/%.3g total %.3g/%.3g chunks %.0f\n",
            sum[0] / k.T, mx[0], sum[1] / k.T, mx[1], sum[2] / k.T, mx[2], sum[3] / k.T, mx[3], sum[4] / k.T, mx[4],
            sum[5] / k.T, mx[5], sum[6] / k.T);
  }
  return e;
}

void k2_free(Plan& p) {
  if (!p.k2) return;
  for (void* v : p.k2->allocs) cudaFree(v);
  if (p.k2->prof) cudaFree(p.k2->prof);
  delete p.k2;
  p.k2 = nullptr;
}

}  // namespace pobk

namespace pobk {
bool k2_stats(const Plan& p, K2Stats& st) {
  if (!p.k2) return false;
  st.T = p.k2->T;
  st.private_frac = p.k2->private_frac;
  st.interior_frac = p.k2->interior_frac;
  st.stream_bytes = p.k2->stream_bytes;
  st.nchunks = p.k2->nchunks;
  return true;
}
}  // namespace pobk
