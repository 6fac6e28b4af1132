// K2: persistent tiled wavefront sweep, warp-specialised.
//
// The rows of A~ are split into T tiles (one CTA per SM, cooperative launch).  A schedule step
// (a category of pairwise-orthogonal rows) restricted to one tile is a "task".  The
// sequential semantics of a sweep (Alg 5 loop) only order rows that share a
// column, so a tile's task k may run once every NEIGHBOUR tile (one sharing a column with it) has
// finished its tasks < k: per-tile progress counters at gpu scope replace the grid-wide barrier
// between categories.  Results are bitwise those of K1/K3 (same per-row contract, common.cuh).
//
//  * x~ columns touched by one tile only ("private") live in that CTA's shared memory for the
//    whole solve; the rest ("shared") live in global memory and are accessed at L2 (ld/st .cg).
//    Within a task, rows touching only private columns ("interior") run before the neighbour
//    wait; rows touching a shared column ("boundary") run after it.
//  * The tile's matrix data (val, col, row extents, f~, ||a~_i||^2) is a sequence of <= 40 KB
//    chunks streamed by 1-D TMA (cp.async.bulk, L2 evict-first) into a 3-slot shared-memory ring,
//    across task and sweep boundaries (A does not depend on x~).
//  * Warp 31 is the CONTROL warp: it issues the TMA copies as slots free up, polls the neighbours'
//    progress for the next boundary task and releases it to the compute warps, publishes the
//    tile's progress when all compute warps finished a task (gpu-scope fence off the compute
//    critical path), and runs the per-sweep stop decision.  Warps 0..30 COMPUTE: they flow
//    through the chunks without CTA-wide barriers; one named barrier per task orders
//    consecutive tasks inside the tile.
//  * The RSE is accumulated by the LAST writer of every column in the sweep (the
//    row of highest step touching it): no extra pass over x~; per-warp partials are reduced in a
//    fixed order, tiles in tile order (deterministic).
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
#ifndef POBK_K2_CPS
#define POBK_K2_CPS 1
#endif
constexpr int kCPS = POBK_K2_CPS;   // CTAs (tiles) per SM
#ifndef POBK_K2_NT
#define POBK_K2_NT 1024
#endif
constexpr int kNT = POBK_K2_NT / kCPS;  // threads per CTA
constexpr int kNCW = kNT / 32 - 1;  // compute warps (the last warp = control)
constexpr int kSlots = 3;           // TMA ring depth
constexpr int kChunkCap = 40 * 1024 / kCPS;
#ifndef POBK_K2_EPT
#define POBK_K2_EPT 4
#endif
constexpr int kEPT = POBK_K2_EPT;   // entries per compute thread per chunk (chunk nnz <= kEPT * compute threads)
constexpr int kNbMax = 32;          // max neighbour tiles (one control-warp lane each)
constexpr int kMaxChunks = 1024;    // max chunks per tile (metadata lives in shared memory)
constexpr int kFlagStride = 32;     // ints between progress counters (one 128-B line each)
constexpr int kSmemLimit = 228 * 1024 / kCPS - 1024;
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
  int rows, nnz, task, flags;  // task = index in the tile's per-sweep task list
  long long off;               // byte offset of the block in the stream
};

struct TaskMeta {
  int step, k_next, boundary, pad;  // k_next >= nsteps: first task of the next sweep
};

struct SyncState {
  unsigned int arrive[2];
  int pad0[30];
  int epoch;  // = sweeps decided
  int stop;
  int pad1[30];
};

struct K2Args {
  const unsigned char* stream;
  const long long* tile_off;  // [T] byte offset of each tile's first chunk
  const ChunkMeta* meta;
  const int* tile_chunk;      // [T+1]
  const TaskMeta* tmeta;
  const int* tile_task;       // [T+1]
  const int* nbr;             // [T*kNbMax], -1 padded
  const int* pmap_ptr;        // [T+1]
  const int* pmap;            // private columns (global ids), tile by tile
  double* xg;                 // x~ (RCM frame); authoritative for shared columns
  const double* xst;          // x~*
  int* progress;              // [T*kFlagStride]
  SyncState* sync;
  double* partials;           // [2*T]
  Ctrl* ctrl;
  int nsteps, T;
  int nck_max, ntask_max, np_max;  // shared-memory sizing
  int debug;                       // development timing experiments (POBK_K2_DEBUG): 2 = no neighbour wait
  unsigned long long* prof;        // optional [T*8] compute-warp phase clocks (POBK_K2_PROFILE=1)
};

// shared-memory control block
struct Ctl {
  unsigned long long full[4];  // TMA completion mbarriers
  int released[4];             // compute-warp releases per slot (cumulative)
  int go;                      // task sequence numbers released to the compute warps
  int done;                    // compute-warp task completions (cumulative)
  int epoch;                   // sweeps decided
  int stop;
  double part[32];             // per-compute-warp RSE partials
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
__device__ __forceinline__ int ld_vol_shared(const int* p) { return *(const volatile int*)p; }
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__global__ void __launch_bounds__(kNT, kCPS) k2_sweeps(K2Args a) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* ring = smem;                                   // kSlots * kChunkCap
  Ctl* ctl = (Ctl*)(smem + kSlots * kChunkCap);
  int4* cmeta = (int4*)(ctl + 1);                               // [nck_max] {rows, nnz, task, flags}
  int* coff = (int*)(cmeta + a.nck_max);                        // [nck_max] byte offset from the tile base
  int4* tmeta = (int4*)(coff + ((a.nck_max + 3) & ~3));          // [ntask_max]
  double* xloc = (double*)(tmeta + a.ntask_max);                // [np_max] private x~
  double* xsloc = xloc + a.np_max;                              // [np_max] private x~* (RSE stop)

  const int t = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, wl = tid & 31;
  const int c0 = a.tile_chunk[t], nck = a.tile_chunk[t + 1] - c0;
  const int j0 = a.tile_task[t], ntask = a.tile_task[t + 1] - j0;
  const int q0 = a.pmap_ptr[t], np = a.pmap_ptr[t + 1] - q0;
  const int nsteps = a.nsteps;
  const long long maxs = a.ctrl->max_sweeps;
  const int mode = a.ctrl->stop_mode, every = a.ctrl->check_every;

  if (tid == 0) {
    for (int i = 0; i < 4; i++) {
      mbar_init(&ctl->full[i], 1);
      ctl->released[i] = 0;
    }
    ctl->go = 0;
    ctl->done = 0;
    ctl->epoch = 0;
    ctl->stop = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int j = tid; j < nck; j += kNT) {
    const ChunkMeta mt = a.meta[c0 + j];
    cmeta[j] = make_int4(mt.rows, mt.nnz, mt.task, mt.flags);
    coff[j] = (int)(mt.off - a.tile_off[t]);
  }
  for (int j = tid; j < ntask; j += kNT) {
    const TaskMeta tm = a.tmeta[j0 + j];
    tmeta[j] = make_int4(tm.step, tm.k_next, tm.boundary, 0);
  }
  for (int j = tid; j < np; j += kNT) {
    const int gcol = a.pmap[q0 + j];
    xloc[j] = a.xg[gcol];
    xsloc[j] = (mode == POBK_STOP_RSE) ? a.xst[gcol] : 0.0;
  }
  __syncthreads();

  if (warp == kNCW) {
    // ================================================================ control warp
    const unsigned long long pol = policy_evict_first();
    const int my_nb = wl < kNbMax ? a.nbr[t * kNbMax + wl] : -1;
    const unsigned char* tbase = a.stream + a.tile_off[t];
    long long g_issue = 0;   // next chunk sequence to issue
    long long j_go = 0;      // next task sequence to release
    long long j_pub = 0;     // next task sequence to publish
    long long sweep = 0;     // sweeps completed (decided)
    bool finished = (maxs <= 0);
    while (!finished) {
      // (1) TMA: keep the ring full (a slot is free once all compute warps released its last use);
      //     never more than one sweep ahead of the decided sweep
      if (nck > 0) {
        while (g_issue < (sweep + 2) * (long long)nck) {
          const int slot = (int)(g_issue % kSlots);
          const long long use = g_issue / kSlots;
          if (use > 0 && ld_vol_shared(&ctl->released[slot]) < (int)(use * kNCW)) break;
          if (wl == 0) {
            const int c = (int)(g_issue % nck);
            const int4 mt = cmeta[c];
            const int bytes = ChunkLayout(mt.x, mt.y).bytes;
            mbar_expect_tx(&ctl->full[slot], bytes);
            tma_load_1d(ring + slot * kChunkCap, tbase + coff[c], bytes, &ctl->full[slot], pol);
          }
          __syncwarp();
          g_issue++;
        }
      }
      // (2) release the next task of this sweep once its neighbours are far enough
      if (ntask > 0 && j_go < (sweep + 1) * (long long)ntask) {
        const int4 tm = tmeta[(int)(j_go % ntask)];
        const long long sw = j_go / ntask;
        bool ok = true;
        if (tm.z && !(a.debug & 2)) {
          const int need = (int)(sw * nsteps + tm.x);
          const int v = my_nb >= 0 ? ld_relaxed(a.progress + my_nb * kFlagStride) : need;
          ok = __all_sync(0xffffffffu, v >= need);
        }
        if (ok) {
          if (tm.z) __threadfence();  // acquire the neighbours' writes at gpu scope ...
          j_go++;
          if (wl == 0) *(volatile int*)&ctl->go = (int)j_go;  // ... and hand them to the CTA
          __syncwarp();
        }
      }
      // (3) publish finished tasks (all compute warps reported the task)
      if (ntask > 0 && j_pub < j_go && ld_vol_shared(&ctl->done) >= (int)((j_pub + 1) * kNCW)) {
        const int4 tm = tmeta[(int)(j_pub % ntask)];
        const long long sw = j_pub / ntask;
        __threadfence();
        if (wl == 0)
          asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(a.progress + t * kFlagStride),
                       "r"((int)(sw * nsteps + tm.y))
                       : "memory");
        __syncwarp();
        j_pub++;
      }
      // (4) end of sweep: every task of the sweep published (or no tasks)
      if ((ntask == 0) || (j_pub >= (sweep + 1) * (long long)ntask)) {
        const long long s1 = sweep + 1;
        const bool due = mode != POBK_STOP_NONE && ((s1 % every) == 0 || s1 >= maxs);
        int stop = 0;
        if (due) {
          if (wl == 0) {
            double part = 0.0;
            if (ntask > 0)
              for (int w = 0; w < kNCW; w++) part += ((volatile double*)ctl->part)[w];
            const int par = (int)(s1 & 1);
            a.partials[par * a.T + t] = part;
            __threadfence();
            const unsigned old = atomicAdd(&a.sync->arrive[par], 1u);
            if (old == (unsigned)a.T - 1) {
              __threadfence();
              double tot = 0.0;
              for (int b = 0; b < a.T; b++) tot += ld_cg(a.partials + par * a.T + b);
              const double v = sqrt(tot) / sqrt(a.ctrl->den);
              int st = 0, term = POBK_TERM_MAX_SWEEPS;
              if (!isfinite(v)) { st = 1; term = POBK_TERM_NONFINITE; }
              else if (v < a.ctrl->tol) { st = 1; term = POBK_TERM_CONVERGED; }
              else if (s1 >= maxs) st = 1;
              a.sync->arrive[par] = 0;
              a.sync->stop = st;
              a.ctrl->value = v;
              a.ctrl->sweeps = s1;
              a.ctrl->term = term;
              __threadfence();
              st_release(&a.sync->epoch, (int)s1);
            } else {
              while (ld_relaxed(&a.sync->epoch) < (int)s1) {
              }
              __threadfence();
            }
            stop = ld_relaxed(&a.sync->stop);
          }
          stop = __shfl_sync(0xffffffffu, stop, 0);
        } else if (s1 >= maxs) {
          stop = 1;
          if (t == 0 && wl == 0) {
            a.ctrl->sweeps = s1;
            a.ctrl->term = POBK_TERM_MAX_SWEEPS;
          }
        }
        sweep = s1;
        if (wl == 0) {
          *(volatile int*)&ctl->stop = stop;
          __threadfence_block();
          *(volatile int*)&ctl->epoch = (int)sweep;
        }
        __syncwarp();
        if (stop) finished = true;
      }
    }
    // drain the TMA copies issued beyond the consumed ones
    if (wl == 0 && nck > 0) {
      const long long consumed = sweep * nck;
      for (long long h = consumed; h < g_issue; h++)
        mbar_wait(&ctl->full[(int)(h % kSlots)], (unsigned)((h / kSlots) & 1));
    }
  } else {
    // ================================================================ compute warps
    // Entry-parallel, three phases per chunk (the oracle's arithmetic, common.cuh):
    //   A  every thread takes entries p = cid + e*NC: gathers x~ (smem or L2) and forms
    //      a_p * x_p, written in place over val[p] in the ring slot (val kept in registers)
    //   B  one thread per row sums its products left to right, alpha = (f - s) / nrm2, and
    //      broadcasts alpha over the row's entry slots
    //   C  every thread scatters x_p + alpha * a_p for its entries (smem or L2), and the last
    //      writer of a column adds (x - x*)^2 to the RSE partial
    constexpr int NC = kNCW * 32;
    const int cid = tid;
    double acc_rse = 0.0;
    long long sweep = 0, g = 0;
    unsigned long long pf_go = 0, pf_full = 0, pf_bar = 0, pf_epoch = 0;
    unsigned long long pf_a = 0, pf_ab = 0, pf_b = 0, pf_bb = 0, pf_c = 0;
    const unsigned long long pf_t0 = clock64();
    while (sweep < maxs) {
      acc_rse = 0.0;
      for (int i = 0; i < nck; i++, g++) {
        const int4 mt = cmeta[i];
        const int rows = mt.x, nnz = mt.y, flags = mt.w;
        unsigned long long pc0 = clock64();
        if (flags & kFirstBoundary) {
          const int jtask = (int)(sweep * ntask + mt.z);
          while (ld_vol_shared(&ctl->go) <= jtask) {
          }
          __threadfence_block();
        }
        unsigned long long pc1 = clock64();
        const int slot = (int)(g % kSlots);
        mbar_wait(&ctl->full[slot], (unsigned)((g / kSlots) & 1));
        unsigned long long pc2 = clock64();
        pf_go += pc1 - pc0;
        pf_full += pc2 - pc1;
        unsigned char* blk = ring + slot * kChunkCap;
        const ChunkLayout L(rows, nnz);
        double* val = (double*)(blk + L.o_val);
        const double* fv = (const double*)(blk + L.o_f);
        const double* nv = (const double*)(blk + L.o_n);
        const unsigned* col = (const unsigned*)(blk + L.o_col);
        const int* rp = (const int*)(blk + L.o_rp);
        unsigned cc[kEPT];
        double av[kEPT], xv[kEPT], sv[kEPT];
        // ---- A: gather and products
#pragma unroll
        for (int e = 0; e < kEPT; e++) {
          const int p = cid + e * NC;
          cc[e] = 0u;
          av[e] = 0.0;
          xv[e] = 0.0;
          sv[e] = 0.0;
          if (p < nnz) {
            cc[e] = col[p];
            av[e] = val[p];
          }
        }
#pragma unroll
        for (int e = 0; e < kEPT; e++) {
          const int p = cid + e * NC;
          if (p < nnz) {
            const unsigned c = cc[e], idx = c & kIdx;
            if (c & kShared) {
              xv[e] = ld_cg(a.xg + idx);
              if (c & kLast) sv[e] = __ldg(a.xst + idx);
            } else {
              xv[e] = xloc[idx];
              if (c & kLast) sv[e] = xsloc[idx];
            }
          }
        }
#pragma unroll
        for (int e = 0; e < kEPT; e++) {
          const int p = cid + e * NC;
          if (p < nnz) val[p] = __dmul_rn(av[e], xv[e]);
        }
        unsigned long long pA = clock64();
        named_bar(1, NC);
        unsigned long long pA2 = clock64();
        // ---- B: per-row sums (left to right), alpha, broadcast
        for (int r = cid; r < rows; r += NC) {
          const int p0 = rp[r], p1 = rp[r + 1];
          double sum = 0.0;
          int p = p0;
          for (; p + 8 <= p1; p += 8) {  // batch the loads, keep the left-to-right additions
            double v[8];
#pragma unroll
            for (int j = 0; j < 8; j++) v[j] = val[p + j];
#pragma unroll
            for (int j = 0; j < 8; j++) sum = __dadd_rn(sum, v[j]);
          }
          for (; p < p1; p++) sum = __dadd_rn(sum, val[p]);
          const double alpha = __ddiv_rn(__dsub_rn(fv[r], sum), nv[r]);
          for (p = p0; p < p1; p++) val[p] = alpha;
        }
        unsigned long long pB = clock64();
        named_bar(1, NC);
        unsigned long long pB2 = clock64();
        // ---- C: scatter
#pragma unroll
        for (int e = 0; e < kEPT; e++) {
          const int p = cid + e * NC;
          if (p < nnz) {
            const unsigned c = cc[e], idx = c & kIdx;
            const double xn = __dadd_rn(xv[e], __dmul_rn(val[p], av[e]));
            if (c & kShared) st_cg(a.xg + idx, xn);
            else xloc[idx] = xn;
            if (c & kLast) {
              const double d = xn - sv[e];
              acc_rse = fma(d, d, acc_rse);
            }
          }
        }
        unsigned long long pC = clock64();
        pf_a += pA - pc2; pf_ab += pA2 - pA; pf_b += pB - pA2; pf_bb += pB2 - pB; pf_c += pC - pB2;
        if ((flags & kLastOfTask) && i == nck - 1 && mode == POBK_STOP_RSE) {
          // this warp's RSE partial (fixed lane order) before it reports the sweep's last task
          double w = acc_rse;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
          if (wl == 0) ctl->part[warp] = w;
        }
        // generic-proxy writes to the slot (products, alphas) before the next TMA refill
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (wl == 0) {
          __threadfence_block();
          atomicAdd(&ctl->released[slot], 1);
          if (flags & kLastOfTask) atomicAdd(&ctl->done, 1);
        }
        if (flags & kLastOfTask) {
          const unsigned long long pb = clock64();
          named_bar(1, NC);  // task k before task k+1 inside the tile
          pf_bar += clock64() - pb;
        }
      }
      sweep++;
      const bool due = mode != POBK_STOP_NONE && ((sweep % every) == 0 || sweep >= maxs);
      if (due) {
        const unsigned long long pe = clock64();
        while (ld_vol_shared(&ctl->epoch) < (int)sweep) {
        }
        __threadfence_block();
        pf_epoch += clock64() - pe;
        if (ld_vol_shared(&ctl->stop)) break;
      }
    }
    if (a.prof && tid == 0) {
      unsigned long long* o = a.prof + t * 16;
      o[0] = pf_go; o[1] = pf_full; o[2] = pf_bar; o[3] = pf_epoch; o[4] = clock64() - pf_t0; o[5] = nck;
      o[6] = pf_a; o[7] = pf_ab; o[8] = pf_b; o[9] = pf_bb; o[10] = pf_c;
    }
  }
  __syncthreads();
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
  int nck_max = 1, ntask_max = 1, np_max = 1;
  unsigned char* stream = nullptr;
  long long* tile_off = nullptr;
  unsigned long long* prof = nullptr;
  ChunkMeta* meta = nullptr;
  TaskMeta* tmeta = nullptr;
  int *tile_chunk = nullptr, *tile_task = nullptr, *nbr = nullptr, *pmap_ptr = nullptr, *pmap = nullptr;
  int* k_first = nullptr;
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
  else if (n) e = cudaMemset(v, 0, n * sizeof(T));
  return e;
}

// Tilers.  Tiles only change WHERE rows run, never the result.
//
// 2-D tiler: S slabs of consecutive RCM rows (equal nnz); inside a slab -- a band of consecutive
// BFS fronts -- rows are ordered by their BFS distance from a far end of the slab's own graph
// (the direction ALONG the fronts) and cut into P pieces of equal nnz.  On mesh-like matrices this
// yields compact patches, so far fewer x~ columns are shared between tiles than with 1-D ranges.
// S = T, P = 1 is the plain 1-D tiling.
void tile_2d(const HostCSR& A, int S, int P, std::vector<int32_t>& tile_of_row) {
  const int64_t m = A.m, nnz = A.nnz();
  tile_of_row.assign(m, 0);
  std::vector<int64_t> cut(S + 1, m);
  cut[0] = 0;
  {
    int s = 0;
    for (int64_t i = 0; i < m && s < S - 1; i++)
      while (s < S - 1 && A.ptr[i] >= (int64_t)((double)nnz * (s + 1) / S)) cut[++s] = i;
    for (int k = s + 1; k < S; k++) cut[k] = m;
  }
  std::vector<int32_t> dist(m, -1), q;
  for (int s = 0; s < S; s++) {
    const int64_t b = cut[s], e = std::max(cut[s], cut[s + 1]);
    if (e <= b) continue;
    if (P == 1) {
      for (int64_t i = b; i < e; i++) tile_of_row[i] = s;
      continue;
    }
    auto bfs = [&](int32_t src, int32_t base) -> int32_t {  // returns the last node reached
      q.clear();
      q.push_back(src);
      dist[src] = base;
      size_t h = 0;
      int32_t last = src;
      while (h < q.size()) {
        const int32_t v = q[h++];
        last = v;
        for (int64_t k = A.ptr[v]; k < A.ptr[v + 1]; k++) {
          const int32_t u = A.col[k];
          if (u >= b && u < e && dist[u] < 0) { dist[u] = dist[v] + 1; q.push_back(u); }
        }
      }
      return last;
    };
    // far end: BFS from the slab's first row, restart from the farthest node
    int32_t far = bfs((int32_t)b, 0);
    for (int64_t i = b; i < e; i++) dist[i] = -1;
    int32_t base = 0;
    bfs(far, 0);
    for (int64_t i = b; i < e; i++)  // other components of the slab continue the ordering
      if (dist[i] < 0) {
        int32_t mx = 0;
        for (int64_t j = b; j < e; j++) mx = std::max(mx, dist[j]);
        base = mx + 1;
        bfs((int32_t)i, base);
      }
    std::vector<int32_t> ord(e - b);
    std::iota(ord.begin(), ord.end(), (int32_t)b);
    std::stable_sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) { return dist[x] < dist[y]; });
    int64_t slab_nnz = A.ptr[e] - A.ptr[b], acc = 0;
    int piece = 0;
    for (int32_t r : ord) {
      while (piece < P - 1 && acc >= (int64_t)((double)slab_nnz * (piece + 1) / P)) piece++;
      tile_of_row[r] = s * P + piece;
      acc += A.ptr[r + 1] - A.ptr[r];
    }
    for (int64_t i = b; i < e; i++) dist[i] = -1;
  }
}

// fraction of nonzeros whose column is touched by one tile only
double private_fraction(const HostCSR& A, const std::vector<int32_t>& tile) {
  const int64_t m = A.m;
  std::vector<int32_t> ct(m, -1);
  std::vector<uint8_t> sh(m, 0);
  for (int64_t i = 0; i < m; i++)
    for (int64_t k = A.ptr[i]; k < A.ptr[i + 1]; k++) {
      const int32_t c = A.col[k];
      if (ct[c] < 0) ct[c] = tile[i];
      else if (ct[c] != tile[i]) sh[c] = 1;
    }
  int64_t priv = 0;
  for (int64_t k = 0; k < A.nnz(); k++) priv += !sh[A.col[k]];
  return A.nnz() ? (double)priv / (double)A.nnz() : 1.0;
}
}  // namespace

bool k2_build(Plan& p, const HostCSR& At, int tile_rows, std::string& why) {
  if (p.any_overlap) { why = "overlapping categories"; return false; }
  int sms = 148;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, p.device) == cudaSuccess) sms = prop.multiProcessorCount;
  const int64_t m = p.m;
  int T = sms * kCPS;
  if (tile_rows > 0) T = (int)std::max<int64_t>(1, std::min<int64_t>(T, (m + tile_rows - 1) / tile_rows));
  T = (int)std::min<int64_t>(T, std::max<int64_t>(1, p.nnz / 4096));
  // tiling: among T' in {T, T-4, T-8} (one tile per SM, a few SMs may idle) and the factorisations
  // T' = S x P, the one with the best (private fraction - load penalty); S = T' is the 1-D tiling
  std::vector<int32_t> tile;
  {
    double best = -1e9;
    int bestT = T;
    const char* force = getenv("POBK_K2_SLABS");  // development override of S
    for (int Tc : {T, T - 4, T - 8}) {
      if (Tc < 1) continue;
      for (int S = 1; S <= Tc; S++) {
        if (Tc % S) continue;
        if (force ? S != atoi(force) : (S != Tc && (S < 2 || Tc / S < 2))) continue;
        std::vector<int32_t> cand;
        tile_2d(At, S, Tc / S, cand);
        const double score = private_fraction(At, cand) - 1.5 * (1.0 - (double)Tc / T);
        if (score > best) { best = score; tile.swap(cand); bestT = Tc; }
      }
      if (force) break;
    }
    if (tile.empty()) tile_2d(At, T, 1, tile);
    T = bestT;
  }

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
  const size_t fixed = (size_t)kSlots * kChunkCap + sizeof(Ctl) + 256;
  const size_t meta_bytes = (size_t)20 * kMaxChunks + 16 * (size_t)p.nsteps;
  if (fixed + meta_bytes + 16 * 1024 > (size_t)kSmemLimit - 1024) {
    why = "too many schedule steps for K2's shared memory";
    return false;
  }
  const int np_cap = (int)((kSmemLimit - 1024 - fixed - meta_bytes) / 16);  // x~ and x~* per column
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
  // tasks and chunks, tile by tile (interior rows first within a task)
  std::vector<std::vector<std::vector<int32_t>>> rows_tk(T);
  for (int t = 0; t < T; t++) rows_tk[t].resize(p.nsteps);
  for (int k = 0; k < p.nsteps; k++) {
    for (int pass = 0; pass < 2; pass++)
      for (int q = p.sched.step_ptr[k]; q < p.sched.step_ptr[k + 1]; q++) {
        const int32_t r = p.sched.rows[q];
        if (boundary[r] == pass) rows_tk[tile[r]][k].push_back(r);
      }
  }
  std::vector<ChunkMeta> meta;
  std::vector<TaskMeta> tmeta;
  std::vector<int> tile_chunk(T + 1, 0), tile_task(T + 1, 0), k_first(T, p.nsteps);
  std::vector<std::vector<int32_t>> chunk_rows;
  for (int t = 0; t < T; t++) {
    std::vector<int> tasks;
    for (int k = 0; k < p.nsteps; k++)
      if (!rows_tk[t][k].empty()) tasks.push_back(k);
    if (!tasks.empty()) k_first[t] = tasks[0];
    for (size_t ti = 0; ti < tasks.size(); ti++) {
      const int k = tasks[ti];
      TaskMeta tm{};
      tm.step = k;
      tm.k_next = ti + 1 < tasks.size() ? tasks[ti + 1] : p.nsteps + tasks[0];
      tm.boundary = 0;
      const auto& rs = rows_tk[t][k];
      size_t a = 0;
      while (a < rs.size()) {
        const uint8_t kind = boundary[rs[a]];
        size_t b = a;
        int nnz = 0;
        while (b < rs.size() && boundary[rs[b]] == kind) {
          const int len = (int)(At.ptr[rs[b] + 1] - At.ptr[rs[b]]);
          if (ChunkLayout((int)(b - a + 1), nnz + len).bytes > kChunkCap || nnz + len > kEPT * kNCW * 32) break;
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
        mt.task = (int)ti;
        mt.flags = 0;
        if (kind == 1 && !tm.boundary) { mt.flags |= kFirstBoundary; tm.boundary = 1; }
        if (b == rs.size()) mt.flags |= kLastOfTask;
        meta.push_back(mt);
        chunk_rows.emplace_back(rs.begin() + a, rs.begin() + b);
        a = b;
      }
      tmeta.push_back(tm);
    }
    tile_chunk[t + 1] = (int)meta.size();
    tile_task[t + 1] = (int)tmeta.size();
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
  int nck_max = 1, ntask_max = 1;
  for (int t = 0; t < T; t++) {
    nck_max = std::max(nck_max, tile_chunk[t + 1] - tile_chunk[t]);
    ntask_max = std::max(ntask_max, tile_task[t + 1] - tile_task[t]);
  }
  k->nck_max = nck_max;
  k->ntask_max = ntask_max;
  k->np_max = std::max(1, *std::max_element(np_t.begin(), np_t.end()));
  k->smem = fixed + 16 * (size_t)nck_max + 4 * (size_t)((nck_max + 3) & ~3) + 16 * (size_t)ntask_max +
            16 * (size_t)k->np_max;
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
  K2_UP(&k->tmeta, tmeta.data(), tmeta.size());
  K2_UP(&k->tile_chunk, tile_chunk.data(), tile_chunk.size());
  K2_UP(&k->tile_task, tile_task.data(), tile_task.size());
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
  a.meta = k.meta;
  a.tile_chunk = k.tile_chunk;
  a.tmeta = k.tmeta;
  a.tile_task = k.tile_task;
  a.nbr = k.nbr;
  a.pmap_ptr = k.pmap_ptr;
  a.pmap = k.pmap;
  a.xg = p.d_xt;
  a.xst = p.d_xst;
  a.progress = k.progress;
  a.sync = k.sync;
  a.partials = k.partials;
  a.ctrl = p.d_ctrl;
  a.nsteps = p.nsteps;
  a.T = k.T;
  a.nck_max = k.nck_max;
  a.ntask_max = k.ntask_max;
  a.np_max = k.np_max;
  static const int dbg = getenv("POBK_K2_DEBUG") ? atoi(getenv("POBK_K2_DEBUG")) : 0;
  a.debug = dbg;
  a.prof = nullptr;
  static const bool prof_on = getenv("POBK_K2_PROFILE") != nullptr;
  if (prof_on) {
    if (!k.prof) cudaMalloc(&k.prof, (size_t)k.T * 16 * sizeof(unsigned long long));
    cudaMemsetAsync(k.prof, 0, (size_t)k.T * 16 * sizeof(unsigned long long), s);
    a.prof = k.prof;
  }
  void* args[] = {&a};
  const void* fn = (const void*)k2_sweeps;
  if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k.smem)) != cudaSuccess) return e;
  e = cudaLaunchCooperativeKernel(fn, dim3(k.T), dim3(kNT), args, k.smem, s);
  launches++;
  if (e == cudaSuccess && a.prof) {
    std::vector<unsigned long long> h((size_t)k.T * 16);
    cudaStreamSynchronize(s);
    cudaMemcpy(h.data(), a.prof, h.size() * 8, cudaMemcpyDeviceToHost);
    double sum[11] = {0}, mx[11] = {0};
    for (int t = 0; t < k.T; t++)
      for (int j = 0; j < 11; j++) { sum[j] += (double)h[t * 16 + j]; mx[j] = std::max(mx[j], (double)h[t * 16 + j]); }
    fprintf(stderr, "[k2 prof] phases (mean per tile): A %.3g barA %.3g B %.3g barB %.3g C %.3g\n", sum[6] / k.T,
            sum[7] / k.T, sum[8] / k.T, sum[9] / k.T, sum[10] / k.T);
    fprintf(stderr, "[k2 prof] warp0 cycles per tile (mean/max): go %.3g/%.3g full %.3g/%.3g taskbar %.3g/%.3g "
                    "epoch %.3g/%.3g total %.3g/%.3g chunks %.0f\n",
            sum[0] / k.T, mx[0], sum[1] / k.T, mx[1], sum[2] / k.T, mx[2], sum[3] / k.T, mx[3], sum[4] / k.T, mx[4],
            sum[5] / k.T);
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
