// K2: persistent tiled wavefront sweep.
//
// The rows of A~ are split into T tiles, one CTA per SM (cooperative launch; 256 threads = 7
// compute warps + 1 TMA producer warp, or 512 threads = 15 + 1 when tasks have many slices).  A
// schedule step (a category of pairwise-orthogonal rows) restricted to one tile is a
// "task".  The sequential semantics of a sweep (Alg 5 loop) only order rows that
// share a column.  Columns touched by one tile only are "private" (kept in that CTA's shared
// memory for the whole solve); the others are "shared".  A row is "interior" if all its columns
// are private, else "boundary".
//   * Inside a tile, task k runs after task k-1 (one named barrier per task).
//   * Across tiles, only shared columns carry dependencies.  Every row touching a shared column c
//     reads the value written by the previous row touching c (in schedule order, wrapping to the
//     previous sweep) and writes the value read by the next one: each written value has exactly
//     ONE consumer.  So the writer stores the new x~_c straight into that consumer's MAILBOX slot
//     (global memory; a consumer lane's slots are contiguous, entry j at lane*Wp + j with Wp = W
//     rounded up to 4, so it polls 4 entries per 256-bit load: a global load instruction costs
//     ~40 cycles of issue whatever its width or its active lanes, measured), and the consumer
//     polls its slots until they no longer hold the sentinel (a signalling-NaN bit pattern no
//     arithmetic produces), then re-arms them.  Aligned 8-byte relaxed accesses (also the
//     elements of a vector access) are single-copy atomic, so no flags, counters or fences are
//     on the critical path; slots are double-buffered by sweep parity and the per-sweep grid
//     barrier orders a slot's re-arm before its next write.
// Results are bitwise those of K1/K3 and of the oracle (the per-row contract of common.cuh).
//
//  * Rows are stored as SLICES of <= 32 rows, one lane per row, in ELL order inside the slice
//    (entry j of lane r at j*R + r; a task's rows are sorted by length before slicing so the
//    padding is small; padding entries are value +0 on a private "zero slot" column): coalesced,
//    conflict-free val/col loads; the row sum runs left to right in one thread (the oracle's
//    order).  An interior row recomputes ||a~_i||^2 in registers (the oracle's left-to-right sum)
//    and streams 12 B per stored entry + 10 B (f~, length); a boundary row also streams its
//    ||a~_i||^2 (8 B, the host's row_sqnorms in the same order) and 4 B per entry (the mailbox
//    slot its new value goes to), all loaded before the task barrier.
//  * A task's boundary slices come first; their warps note the shared entries, poll the
//    mailboxes, then read the private operands with the row sums; the interior slices run
//    meanwhile on the other warps.
//  * The tile's slices are packed, across task boundaries, into <= 24 KB chunks streamed by 1-D
//    TMA (cp.async.bulk, L2 evict-first) into a ring of NS slots by the PRODUCER warp (the last
//    warp), which never touches x~.
//  * Stop checks at the end of a due sweep.  RSE: each tile sums (x~ - x~*)^2
//    over the columns it owns (its private ones, x~ in shared memory, and the shared ones whose
//    last writer in the sweep it holds, read from the wrap mailbox slot), x~* from per-tile
//    contiguous arrays gathered once per solve.  RELRES: the owners publish the shared columns'
//    sweep-final values to global x~, a grid barrier, then a residual pass over each tile's own
//    stream.  Partials are combined in fixed orders; one grid-wide decision per sweep (every
//    tile forms the same total from the same partials).
//  * A task's slices, boundary first, go round-robin over the compute warps (the round-robin
//    continuing across tasks), so consecutive boundary slices run on different SM sub-partitions.
//  * One kernel instantiation per plan shape (threads, vector-slice width, interior mode): all
//    paths inlined into one kernel spilled registers and doubled the sweep time.
//  * Tensor memory as a per-thread parking area (DESIGN.md §5.2 (vii)): an interior slice's
//    pass 1 parks its columns, values and x~ in TMEM (tcgen05.st) and pass 2 reads them back
//    (tcgen05.ld) instead of re-reading them from shared memory, whose pipe the interior slices
//    saturate; interior slices store 16-bit column indices (tile-local).
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
// Threads per CTA (one CTA per SM) is a template parameter of k2_sweeps: 256 (7 compute warps,
// up to 255 registers: register-resident boundary slices, BSlice2) when a task has few slices,
// 512 (15 compute warps, 128 registers: BSlice) when tasks have many (k2_build decides).
#ifndef POBK_K2_SLOT_KB
#define POBK_K2_SLOT_KB 24  // (measured r02: 16 KB 102.6 / 24 KB 98.1 / 32 KB 98.2 us per config-4 sweep; 32 KB
                            //  starves the half-GPU config-5 tiles of private columns)
#endif
constexpr int kSlot = POBK_K2_SLOT_KB * 1024;  // ring slot (chunk) capacity, bytes
static_assert(kSlot <= 65536, "slice offsets are packed in 16 bits");
#ifndef POBK_K2_MAXSLOTS
#define POBK_K2_MAXSLOTS 8
#endif
constexpr int kMinSlots = 4, kMaxSlots = POBK_K2_MAXSLOTS;
constexpr int kSliceRows = 32;      // rows per slice (one lane each)
#ifndef POBK_K2_MAXJ
#define POBK_K2_MAXJ 24
#endif
constexpr int kMaxJ = POBK_K2_MAXJ; // entries per row whose x~ is kept in registers between passes (<= 32)
static_assert(POBK_K2_MAXJ % 8 == 0 && POBK_K2_MAXJ <= 32, "the register window is processed in batches of 8");
constexpr int kBatch = 8;           // loads issued together
#ifndef POBK_K2_CHAIN
#define POBK_K2_CHAIN 8
#endif
constexpr int kChainB = POBK_K2_CHAIN;
#ifndef POBK_K2_WB
#define POBK_K2_WB 8
#endif
constexpr int kWB = POBK_K2_WB;
#ifndef POBK_K2_RSEU
#define POBK_K2_RSEU 4
#endif
constexpr int kRU = POBK_K2_RSEU;  // end-of-sweep RSE scan: loads in flight per thread  // boundary write-back: entries issued per group  // boundary row sum: products of a group first, then its adds
#ifndef POBK_K2_TMEM
#define POBK_K2_TMEM 1  // interior pass-2 operands in tensor memory (measured r02f: config 4 96.8 -> 93.7 us/sweep)
#endif
// interior slices parked in TMEM: 8-entry batches for slices wider than 12 (fewer dependent
// load rounds: config 4 94.2 -> 92.6 us/sweep), 4-entry ones below (less clamped padding:
// config 5's 9-entry rows -- 8-entry batches cost it 6%)
constexpr int kTmWide = 12;
#ifndef POBK_K2_IBATCH
#define POBK_K2_IBATCH 4  // (measured r02: 4 vs 8 -- config 4 97.6 vs 98.1 us/sweep, config 5 200.6 vs 190.3 G)
#endif
constexpr int kIB = POBK_K2_IBATCH;    // interior slices: entries per batch
constexpr int kSmemTotal = 227 * 1024 - 256;  // (the opt-in budget less room for static shared memory)
constexpr int kMetaBudget = 16 * 1024;  // slice/chunk/task metadata in shared memory
constexpr unsigned kShared = 0x80000000u, kIdx = 0x7FFFFFFFu;
constexpr unsigned kWrap = 0x80000000u;  // mailbox target of a sweep's last writer: next sweep's slot
constexpr unsigned long long kSentinel = 0x7FF0DEADBEEFCAFEull;  // signalling NaN: "slot empty"
constexpr unsigned kFull = 0xffffffffu;

__host__ __device__ inline int a16(long long b) { return (int)((b + 15) & ~15LL); }

// slice block (bytes): val[W*R] f[R*nf] (fp64; nf right-hand sides, row-major) | [boundary slices] n2[R] (fp64: ||a~||^2)
//                      | col[W*R] (boundary slices: u32 shared flag | index; interior slices: u16 local index)
//                      | [boundary slices] mout[W*R] (u32: wrap flag | mailbox index) | len[R] (u16)
struct SliceLayout {
  int o_f, o_n2, o_col, o_mout, o_len, bytes;
  __host__ __device__ SliceLayout(int R, int W, bool bnd, int nf = 1) {
    o_f = 8 * W * R;
    o_n2 = o_f + 8 * R * nf;
    o_col = o_n2 + (bnd ? 8 * R : 0);
    o_mout = o_col + (bnd ? 4 : 2) * W * R;
    o_len = o_mout + (bnd ? 4 * W * R : 0);
    bytes = a16(o_len + 2 * R);
  }
};

struct SyncState {
  unsigned long long arrive;   // monotonic: T per completed sweep (64-bit: no wrap at any sweep count)
  unsigned long long arrive2;  // monotonic: T per RELRES publication (x~ of the shared columns)
  long long pad0[14];
};
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

struct K2Args {
  const unsigned char* stream;
  const long long* tile_off;  // [T] byte offset of each tile's first chunk
  const int4* smeta;          // slices: {chunk | R << 20, offset in chunk | (chunk mod 2NS) << 16, W, mailbox base (boundary)}
  const int* tile_slice;      // [T+1]
  const int4* cmeta;          // chunks: {offset from tile base, bytes, slices, 0}
  const int* tile_chunk;      // [T+1]
  const int4* tmeta;          // tasks: {first slice, n_boundary | n_interior << 16, step, 0}
  const int* tile_task;       // [T+1]
  const int* pmap_ptr;        // [T+1]
  const int* pmap;            // private columns (global ids), tile by tile
  const int* lastcol_ptr;     // [T+1]
  const int* lastcol;         // shared columns whose last writer in a sweep is in the tile, tile by tile
  const int* lastslot;        // ... and their wrap mailbox slot (the next sweep's first reader's)
  unsigned long long* mbox;   // [2*NB] mailboxes (fp64 bits or kSentinel), parity-major
  long long NB;
  double* xg;                 // x~ (RCM frame): x0 in, final out; shared columns' sweep-final values
  const double* xst;          // x~*
  const double* xsp;          // [pmap size] x~* of the private columns in tile-local order (RSE stop)
  const double* lcx;          // [lastcol size] x~* of the owned shared columns (RSE stop)
  SyncState* sync;
  double* partials;           // [2*kR*T]
  Ctrl* ctrl;
  // the second right-hand side of a two-RHS plan (kR = 2): its x~, x~* gathers and stop record
  double* xg1;
  const double* xsp1;
  const double* lcx1;
  Ctrl* ctrl1;
  int T, NS;
  int nsl_max, nck_max, ntask_max, np_max;  // shared-memory sizing
  unsigned long long* trace;  // optional [T*ntask_max*12] globaltimer stamps of one sweep (POBK_K2_TRACE=s)
  int trace_sweep;
};

// shared-memory control block
struct alignas(16) Ctl {  // (16-byte multiple: the int4 metadata follows it in shared memory)
  unsigned long long full[kMaxSlots];  // TMA completion mbarriers
  int released[kMaxSlots];             // slices consumed per slot (cumulative)
  unsigned long long issued;           // chunks issued (sequence number)
  int stop;
  long long done;                      // sweeps completed (all tiles stop at the same sweep)
  double part[64];                     // per-compute-warp RSE partials (right-hand side q at 32 q + warp)
  unsigned actm;                       // bit q: right-hand side q still iterating (two-RHS plans)
  int pad1[3];
};
static_assert(sizeof(Ctl) % 16 == 0, "int4 metadata follows Ctl in shared memory");

// ------------------------------------------------------------------ PTX helpers (TMA, mbarrier)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
// 1-D bulk copy global -> shared, completing on an mbarrier; the matrix stream is read once per
// sweep and must not evict x~ or the mailboxes from L2, so it carries an L2 evict-first policy.
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
// POBK_K2_DEV (development builds only, default 0): the per-task trace stamps of one sweep
// (POBK_K2_TRACE=<sweep>, tools/k2_trace.py and friends); production builds carry no trace code.
#ifndef POBK_K2_DEV
#if defined(POBK_K2_FT) || defined(POBK_K2_WT)
#define POBK_K2_DEV 1
#else
#define POBK_K2_DEV 0
#endif
#endif
// POBK_K2_FT (development): trace stamps in SM clock cycles instead of global nanoseconds, plus
// stamps inside the boundary post (tools/k2_ft.py)
#ifndef POBK_K2_FT
#define POBK_K2_FT 0
#endif
// POBK_K2_WT (development): per task, every compute warp's clock64 at its arrival at the barrier
// that closes the task (slots 0..6 of the task's record), slot 7: look-ahead warps of the next
// task (bit mask), slot 8: the barrier's release (tools/k2_wt.py; 256-thread instantiation; the
// other trace stamps share the record, so only slots 0..8 are meaningful in this mode)
#ifndef POBK_K2_WT
#define POBK_K2_WT 0
#endif
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long v;
  if (POBK_K2_FT)
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(v));
  else
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  return v;
}
__device__ __forceinline__ int ld_vol_shared(const int* p) { return *(const volatile int*)p; }
__device__ __forceinline__ unsigned long long ld_vol_shared64(const unsigned long long* p) {
  return *(const volatile unsigned long long*)p;
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
#ifndef POBK_K2_PSLEEP
#define POBK_K2_PSLEEP 64  // producer back-off while its next ring slot is still in use (ns)
#endif
#ifndef POBK_K2_CSLEEP
#define POBK_K2_CSLEEP 32  // consumer back-off while its chunk is not issued yet (ns)
#endif
#ifndef POBK_K2_POLLSLEEP
#define POBK_K2_POLLSLEEP 0  // back-off between mailbox poll rounds (ns)
#endif
#ifndef POBK_K2_PRIO
#define POBK_K2_PRIO 1  // boundary priority on the 256-thread path (measured 1-2% faster, configs 3-4)
#endif

// ------------------------------------------------------------------ slice arithmetic
// All shared-memory operands are addressed through 32-bit shared-window addresses held in
// registers ("opaque": the compiler may not rematerialise the window base inside predicated
// code, which serialised the loads), and predicated PTX stores replace branches.
__device__ __forceinline__ unsigned opaque(unsigned v) {
  asm volatile("mov.u32 %0, %0;" : "+r"(v));
  return v;
}
__device__ __forceinline__ double lds64(unsigned a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ unsigned lds32(unsigned a) {
  unsigned v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ unsigned lds16(unsigned a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
// eight shared-memory loads issued back to back (one asm block: the compiler cannot interleave
// their consumers, so all eight are in flight before the first use)
__device__ __forceinline__ void lds32x8(unsigned (&v)[8], const unsigned (&a)[8]) {
  asm volatile(
      "ld.shared.u32 %0, [%8];\n ld.shared.u32 %1, [%9];\n ld.shared.u32 %2, [%10];\n ld.shared.u32 %3, [%11];\n"
      " ld.shared.u32 %4, [%12];\n ld.shared.u32 %5, [%13];\n ld.shared.u32 %6, [%14];\n ld.shared.u32 %7, [%15];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
}
__device__ __forceinline__ void lds64x8(double (&v)[8], const unsigned (&a)[8]) {
  asm volatile(
      "ld.shared.f64 %0, [%8];\n ld.shared.f64 %1, [%9];\n ld.shared.f64 %2, [%10];\n ld.shared.f64 %3, [%11];\n"
      " ld.shared.f64 %4, [%12];\n ld.shared.f64 %5, [%13];\n ld.shared.f64 %6, [%14];\n ld.shared.f64 %7, [%15];"
      : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]), "=d"(v[4]), "=d"(v[5]), "=d"(v[6]), "=d"(v[7])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
}
__device__ __forceinline__ void sts64_if(unsigned p, unsigned a, double v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %0, 0;\n @q st.shared.f64 [%1], %2;\n}" ::"r"(p), "r"(a), "d"(v)
               : "memory");
}
// mailbox word: relaxed gpu-scope (single-copy atomic, observed at L2)
__device__ __forceinline__ unsigned long long ldm_if(unsigned p, const unsigned long long* a, unsigned long long dflt) {
  unsigned long long v = dflt;
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %1, 0;\n @q ld.relaxed.gpu.global.b64 %0, [%2];\n}"
               : "+l"(v)
               : "r"(p), "l"(a)
               : "memory");
  return v;
}
// four consecutive mailbox words of one lane (32-byte aligned), one 256-bit load: each word is
// still an aligned 8-byte single-copy-atomic access; unchanged registers when p == 0
__device__ __forceinline__ void ldm4_if(unsigned p, const unsigned long long* a, double& x0, double& x1, double& x2,
                                        double& x3) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %4, 0;\n @q ld.relaxed.gpu.global.v4.b64 {%0, %1, %2, %3}, [%5];\n}"
               : "+d"(x0), "+d"(x1), "+d"(x2), "+d"(x3)
               : "r"(p), "l"(a)
               : "memory");
}
__device__ __forceinline__ void stm4_if(unsigned p, unsigned long long* a, unsigned long long v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %0, 0;\n @q st.relaxed.gpu.global.v4.b64 [%1], {%2, %2, %2, %2};\n}" ::"r"(p),
               "l"(a), "l"(v)
               : "memory");
}
__device__ __forceinline__ void stm_if(unsigned p, unsigned long long* a, unsigned long long v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %0, 0;\n @q st.relaxed.gpu.global.b64 [%1], %2;\n}" ::"r"(p), "l"(a),
               "l"(v)
               : "memory");
}

// two consecutive fp64 (a column's two right-hand sides, 16-byte aligned)
__device__ __forceinline__ double2 lds128(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128_if(unsigned p, unsigned a, double v0, double v1) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %0, 0;\n @q st.shared.v2.f64 [%1], {%2, %3};\n}" ::"r"(p), "r"(a), "d"(v0),
               "d"(v1)
               : "memory");
}
// a mailbox slot of a two-RHS plan: two words, each single-copy atomic (the reader checks both)
__device__ __forceinline__ void stm2_if(unsigned p, unsigned long long* a, double v0, double v1) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %0, 0;\n @q st.relaxed.gpu.global.v2.b64 [%1], {%2, %3};\n}" ::"r"(p),
               "l"(a), "l"((unsigned long long)__double_as_longlong(v0)), "l"((unsigned long long)__double_as_longlong(v1))
               : "memory");
}

// four predicated shared-memory loads in one asm block (registers keep their value where the
// predicate is off)
__device__ __forceinline__ void lds64x4_if(double& v0, double& v1, double& v2, double& v3, unsigned p0, unsigned p1,
                                           unsigned p2, unsigned p3, unsigned a0, unsigned a1, unsigned a2, unsigned a3) {
  asm volatile(
      "{\n .reg .pred q0, q1, q2, q3;\n setp.ne.u32 q0, %4, 0;\n setp.ne.u32 q1, %5, 0;\n setp.ne.u32 q2, %6, 0;\n"
      " setp.ne.u32 q3, %7, 0;\n @q0 ld.shared.f64 %0, [%8];\n @q1 ld.shared.f64 %1, [%9];\n"
      " @q2 ld.shared.f64 %2, [%10];\n @q3 ld.shared.f64 %3, [%11];\n}"
      : "+d"(v0), "+d"(v1), "+d"(v2), "+d"(v3)
      : "r"(p0), "r"(p1), "r"(p2), "r"(p3), "r"(a0), "r"(a1), "r"(a2), "r"(a3));
}

// A slice in the ring (shared-window address blk): lane r < R holds row r.  Entries j >= len_r
// of a row are ELL padding: value +0 and the private "zero slot" column (x~ = +0, never written),
// so including them in the sums adds +0 * +0 = +0 and changes no bit (a row sum starting at +0
// is never -0); only the stores are predicated on j < len_r.  Rows are applied with the per-row
// contract of common.cuh (Eq 1.2).
struct SliceAddr {
  unsigned vb, cb, mb;  // this lane's val / col / mout entry 0; entry j at + j*vs / + j*cs (u32 col, boundary) or u16 col (interior)
  unsigned vs, cs;      // strides
  int myl;              // row length (0 for lanes >= R)
  double f, f1;         // f~_i (f1: the second right-hand side's, nf = 2)
  __device__ __forceinline__ SliceAddr(unsigned blk, int R, int W, bool bnd, int lane, int nf = 1) {
    const int ln = lane < R ? lane : 0;
    vs = 8u * R;
    cs = (bnd ? 4u : 2u) * R;
    const SliceLayout L(R, W, bnd, nf);
    vb = opaque(blk + 8u * ln);
    cb = opaque(blk + (unsigned)L.o_col + (bnd ? 4u : 2u) * ln);
    mb = blk + (unsigned)L.o_mout + 4u * ln;
    f = lds64(blk + (unsigned)L.o_f + 8u * nf * ln);
    f1 = nf > 1 ? lds64(blk + (unsigned)L.o_f + 8u * nf * ln + 8u) : 0.0;
    myl = lane < R ? (int)lds16(blk + (unsigned)L.o_len + 2u * ln) : 0;
  }
};

// interior slice: every column private (shared memory at xb); pass 2 re-reads x~ from shared
// memory (unchanged in between: no other row of the category touches these columns)
__device__ __forceinline__ void slice_interior(const SliceAddr& S, int W, unsigned xb) {
  double s = 0.0, n2 = 0.0;
  for (int jb = 0; jb < W; jb += kIB) {
    unsigned c[kIB];
    double av[kIB], xv[kIB];
#pragma unroll
    for (int u = 0; u < kIB; u++) c[u] = lds16(S.cb + min(jb + u, W - 1) * S.cs);
#pragma unroll
    for (int u = 0; u < kIB; u++) xv[u] = lds64(xb + 8u * c[u]);
#pragma unroll
    for (int u = 0; u < kIB; u++) av[u] = lds64(S.vb + min(jb + u, W - 1) * S.vs);
    // entries past the slice width contribute +0 * +0 (bit-exact no-ops): no per-entry branches,
    // so the next batch's loads can issue under this batch's arithmetic; the batch's products
    // first, then the two chains (common.cuh pin())
    double pp[kIB], qq[kIB];
#pragma unroll
    for (int u = 0; u < kIB; u++) {
      const bool in = jb + u < W;
      const double a = in ? av[u] : 0.0, x = in ? xv[u] : 0.0;
      pp[u] = pin(__dmul_rn(a, x));
      qq[u] = pin(__dmul_rn(a, a));
    }
#pragma unroll
    for (int u = 0; u < kIB; u++) {
      s = __dadd_rn(s, pp[u]);
      n2 = __dadd_rn(n2, qq[u]);
    }
  }
  const double alpha = __ddiv_rn(__dsub_rn(S.f, s), n2);
  for (int jb = 0; jb < W; jb += kIB) {
    unsigned c[kIB];
    double av[kIB], xv[kIB];
#pragma unroll
    for (int u = 0; u < kIB; u++) {
      c[u] = lds16(S.cb + min(jb + u, W - 1) * S.cs);
      av[u] = lds64(S.vb + min(jb + u, W - 1) * S.vs);
    }
#pragma unroll
    for (int u = 0; u < kIB; u++) xv[u] = lds64(xb + 8u * c[u]);
#pragma unroll
    for (int u = 0; u < kIB; u++) sts64_if(jb + u < S.myl, xb + 8u * c[u], __dadd_rn(xv[u], __dmul_rn(alpha, av[u])));
  }
}

// interior slice with pass 1's operands parked in tensor memory (TMEM) for pass 2: pass 2 reads
// them back with tcgen05.ld (own datapath) instead of re-reading col, value and x~ from shared
// memory -- the shared-memory pipe keeps only pass 1's loads and pass 2's x~ stores.
// taddr: this warp's TMEM region (its lane quarter, 20 columns per 4-entry batch); W <= kTmMaxW.
__device__ __forceinline__ void tm_st4(unsigned a, unsigned v0, unsigned v1, unsigned v2, unsigned v3) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v0), "r"(v1), "r"(v2), "r"(v3)
               : "memory");
}
__device__ __forceinline__ void tm_ld4(unsigned a, unsigned& v0, unsigned& v1, unsigned& v2, unsigned& v3) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3)
               : "r"(a)
               : "memory");
}
template <int IB>
__device__ __forceinline__ void slice_interior_tm(const SliceAddr& S, int W, unsigned xb, unsigned taddr) {
  static_assert(IB % 4 == 0, "batches park in 4-word TMEM stores");
  // per batch: columns [IB words] | values [2 IB] | x~ [2 IB]
  double s = 0.0, n2 = 0.0;
  for (int jb = 0; jb < W; jb += IB) {
    unsigned c[IB];
    double av[IB], xv[IB];
#pragma unroll
    for (int u = 0; u < IB; u++) c[u] = lds16(S.cb + min(jb + u, W - 1) * S.cs);
#pragma unroll
    for (int u = 0; u < IB; u++) xv[u] = lds64(xb + 8u * c[u]);
#pragma unroll
    for (int u = 0; u < IB; u++) av[u] = lds64(S.vb + min(jb + u, W - 1) * S.vs);
    const unsigned ta = taddr + (unsigned)(jb / IB) * (5u * IB);
#pragma unroll
    for (int g = 0; g < IB / 4; g++) tm_st4(ta + 4 * g, c[4 * g], c[4 * g + 1], c[4 * g + 2], c[4 * g + 3]);
#pragma unroll
    for (int g = 0; g < IB / 2; g++)
      tm_st4(ta + IB + 4 * g, __double2loint(av[2 * g]), __double2hiint(av[2 * g]), __double2loint(av[2 * g + 1]),
             __double2hiint(av[2 * g + 1]));
#pragma unroll
    for (int g = 0; g < IB / 2; g++)
      tm_st4(ta + 3 * IB + 4 * g, __double2loint(xv[2 * g]), __double2hiint(xv[2 * g]), __double2loint(xv[2 * g + 1]),
             __double2hiint(xv[2 * g + 1]));
    double pp[IB], qq[IB];
#pragma unroll
    for (int u = 0; u < IB; u++) {
      const bool in = jb + u < W;
      const double a = in ? av[u] : 0.0, x = in ? xv[u] : 0.0;
      pp[u] = pin(__dmul_rn(a, x));
      qq[u] = pin(__dmul_rn(a, a));
    }
#pragma unroll
    for (int u = 0; u < IB; u++) {
      s = __dadd_rn(s, pp[u]);
      n2 = __dadd_rn(n2, qq[u]);
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  const double alpha = __ddiv_rn(__dsub_rn(S.f, s), n2);
  for (int jb = 0; jb < W; jb += IB) {
    const unsigned ta = taddr + (unsigned)(jb / IB) * (5u * IB);
    unsigned c[IB], w[4 * IB];
#pragma unroll
    for (int g = 0; g < IB / 4; g++) tm_ld4(ta + 4 * g, c[4 * g], c[4 * g + 1], c[4 * g + 2], c[4 * g + 3]);
#pragma unroll
    for (int g = 0; g < IB; g++) tm_ld4(ta + IB + 4 * g, w[4 * g], w[4 * g + 1], w[4 * g + 2], w[4 * g + 3]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int u = 0; u < IB; u++) {
      const double av = __hiloint2double((int)w[2 * u + 1], (int)w[2 * u]);
      const double xv = __hiloint2double((int)w[2 * IB + 2 * u + 1], (int)w[2 * IB + 2 * u]);
      sts64_if(jb + u < S.myl, xb + 8u * c[u], __dadd_rn(xv, __dmul_rn(alpha, av)));
    }
  }
}

// boundary slice: pre() notes the shared entries; poll() loads the shared entries' mailboxes
// (this lane's slots are contiguous, entry j at mbox_in + j: one 256-bit load per 4 entries -- a
// global load instruction costs ~40 cycles of issue whatever its width or active lanes) until no
// sentinel is left, then re-arms them; post() reads the PRIVATE x~ (final for this step once the
// tile's previous task is done) while it forms the row sums, applies the rows, writes private
// results to shared memory and shared results to their consumers' mailboxes.  (A sweep's
// last writer of a column writes the next sweep's first reader's slot, which therefore holds the
// column's sweep-final value until that reader runs: the RSE and the final write-back read it.)
struct BSlice {
  double xr[kMaxJ];
  unsigned shm;  // bit j: entry j (< kMaxJ) is a shared column of this lane's row
  __device__ __forceinline__ void pre(const SliceAddr& S, int W, unsigned xb) {
    shm = 0u;
#pragma unroll
    for (int jb = 0; jb < kMaxJ; jb += kBatch) {
      if (jb < W) {
        unsigned cr[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; u++) cr[u] = lds32(S.cb + min(jb + u, W - 1) * S.cs);
#pragma unroll
        for (int u = 0; u < kBatch; u++) {
          const bool sh = (cr[u] & kShared) && jb + u < S.myl;
          shm |= sh ? (1u << (jb + u)) : 0u;
        }
      }
    }
  }
  // poll this lane's shared entries j < kMaxJ until every lane of the warp has all of them
  __device__ __forceinline__ void poll(const SliceAddr& S, int W, int R, unsigned long long* mbox_in,
                                       unsigned long long* trp = nullptr) {
    unsigned pend = shm;
    int it = 0;
    while (true) {
      it++;
#pragma unroll
      for (int j4 = 0; j4 < kMaxJ; j4 += 4)  // (the other entries of a group: overwritten in post)
        if (j4 < W) ldm4_if((pend >> j4) & 0xFu, mbox_in + j4, xr[j4], xr[j4 + 1], xr[j4 + 2], xr[j4 + 3]);
      unsigned np = 0u;
#pragma unroll
      for (int j = 0; j < kMaxJ; j++)
        if ((pend >> j) & 1u) np |= ((unsigned long long)__double_as_longlong(xr[j]) == kSentinel) ? (1u << j) : 0u;
      pend = np;
      if (!__any_sync(kFull, pend != 0u)) break;
    }
    if (trp && (threadIdx.x & 31) == 0) trp[11] = (unsigned long long)it;
    // re-arm the consumed slots for the sweep after next (ordered by the per-sweep grid barrier)
#pragma unroll
    for (int j4 = 0; j4 < kMaxJ; j4 += 4)
      if (j4 < W) stm4_if((shm >> j4) & 0xFu, mbox_in + j4, kSentinel);
  }
  // mbox: the mailbox array; off_p / off_q: index offsets of this sweep's / the next sweep's parity.
  // Entries are processed in groups of 4 (a 9-entry row -- config 5 -- touches 12 slots, not 16);
  // ||a~||^2 comes from the stream (the host's row_sqnorms, the oracle's O1 order).
  __device__ __forceinline__ void post(const SliceAddr& S, int W, unsigned xb, unsigned long long* mbox_in,
                                       unsigned long long* mbox, unsigned off_p, unsigned off_q, int R,
                                       unsigned long long* trp) {
    constexpr int kG = 4;
    const double n2 = lds64(S.vb + (unsigned)SliceLayout(R, W, true).o_n2);  // (vb = block + 8 * lane)
    const double y2 = rcp_ahead(n2);  // (independent of the row sum: overlaps it)
    double s = 0.0;
#pragma unroll
    for (int jb = 0; jb < kMaxJ; jb += kG) {
      if (jb < W) {
        // a group: columns, then the private x~ (always a valid address: branch-free), then the
        // values -- all loads in flight before the first use
        double av[kG], xp[kG];
        unsigned cr[kG];
#pragma unroll
        for (int u = 0; u < kG; u++) cr[u] = lds32(S.cb + min(jb + u, W - 1) * S.cs);
        lds64x4_if(xp[0], xp[1], xp[2], xp[3], 1u, 1u, 1u, 1u, xb + 8u * ((cr[0] & kShared) ? 0u : cr[0]),
                   xb + 8u * ((cr[1] & kShared) ? 0u : cr[1]), xb + 8u * ((cr[2] & kShared) ? 0u : cr[2]),
                   xb + 8u * ((cr[3] & kShared) ? 0u : cr[3]));
#pragma unroll
        for (int u = 0; u < kG; u++) av[u] = jb + u < W ? lds64(S.vb + min(jb + u, W - 1) * S.vs) : 0.0;
        double pp[kG];
#pragma unroll
        for (int u = 0; u < kG; u++) {  // past the width: +0 * +0 (xr, av are +0 there)
          const int j = jb + u;
          const bool priv = j < W && !(cr[u] & kShared);
          xr[j] = ((shm >> j) & 1u) ? xr[j] : (priv ? xp[u] : 0.0);
          pp[u] = pin(__dmul_rn(av[u], xr[jb + u]));
        }
#pragma unroll
        for (int u = 0; u < kG; u++) s = __dadd_rn(s, pp[u]);
      }
    }
    for (int j = kMaxJ; j < W; j++) {
      const unsigned cj = lds32(S.cb + j * S.cs);
      const double a = lds64(S.vb + j * S.vs);
      double x = 0.0;
      if ((cj & kShared) && j < S.myl) {
        unsigned long long w;
        do {
          w = ldm_if(1u, mbox_in + j, 0ull);
        } while (w == kSentinel);  // (re-armed in pass 2, after it is read again)
        x = __longlong_as_double((long long)w);
      } else if (!(cj & kShared)) {
        x = lds64(xb + 8u * (cj & kIdx));
      }
      s = __dadd_rn(s, __dmul_rn(a, x));
    }
    if (trp) {
      double s2 = s;
      asm volatile("mov.b64 %0, %0;" : "+d"(s2));
      __syncwarp();
      if ((threadIdx.x & 31) == 0) trp[2] = gtimer();
    }
    const double alpha = div_by_rcp(__dsub_rn(S.f, s), n2, y2);
    if (trp) {
      double a2 = alpha;
      asm volatile("mov.b64 %0, %0;" : "+d"(a2));
      __syncwarp();
      if ((threadIdx.x & 31) == 0) trp[9] = gtimer();
    }
#pragma unroll
    for (int jb = 0; jb < kMaxJ; jb += kG) {  // new x~ (in place), then the write-back of the group
      if (jb < W) {
        double av[kG];
        unsigned mo[kG], cr[kG];
#pragma unroll
        for (int u = 0; u < kG; u++) {
          av[u] = lds64(S.vb + min(jb + u, W - 1) * S.vs);
          cr[u] = lds32(S.cb + min(jb + u, W - 1) * S.cs);
          mo[u] = lds32(S.mb + min(jb + u, W - 1) * S.cs);
        }
#pragma unroll
        for (int u = 0; u < kG; u++) {
          const int j = jb + u;
          xr[j] = __dadd_rn(xr[j], __dmul_rn(alpha, av[u]));
          const unsigned act = j < S.myl, sh = (shm >> j) & 1u;
          sts64_if(act & (sh ^ 1u), xb + 8u * (cr[u] & kIdx), xr[j]);
          stm_if(act & sh, mbox + ((mo[u] & ~kWrap) + ((mo[u] & kWrap) ? off_q : off_p)),
                 (unsigned long long)__double_as_longlong(xr[j]));
        }
      }
    }
    for (int j = kMaxJ; j < W; j++) {  // tail: the slot still holds the consumed value (re-armed now)
      const unsigned cj = lds32(S.cb + j * S.cs), idx = cj & kIdx;
      const double a = lds64(S.vb + j * S.vs);
      if ((cj & kShared) && j < S.myl) {
        const unsigned long long w = ldm_if(1u, mbox_in + j, 0ull);
        stm_if(1u, mbox_in + j, kSentinel);
        {
          const double x1 = __dadd_rn(__longlong_as_double((long long)w), __dmul_rn(alpha, a));
          const unsigned mo = lds32(S.mb + j * S.cs);
          stm_if(1u, mbox + ((mo & ~kWrap) + ((mo & kWrap) ? off_q : off_p)), (unsigned long long)__double_as_longlong(x1));
        }
      } else if (!(cj & kShared) && j < S.myl) {
        const unsigned ca = xb + 8u * idx;
        sts64_if(1u, ca, __dadd_rn(lds64(ca), __dmul_rn(alpha, a)));
      }
    }
    if (POBK_K2_FT && trp && (threadIdx.x & 31) == 0) trp[7] = gtimer();
  }
};

// Register-resident boundary slice (the 256-thread instantiation): the row's values, one target
// word per entry (a private entry's x~ address in shared memory, a shared entry's mailbox target)
// and ||a~||^2 (from the stream: the host's left-to-right sum, the oracle's O1 order) are loaded
// from the ring BEFORE the barrier that closes the tile's previous task, together with the
// mailbox poll; after the barrier only the private x~ loads (all in flight at once), the row
// sum, the division and the stores remain on the critical path.  Same arithmetic in the same
// order as BSlice (the common.cuh contract).
struct BSlice2 {
  double xr[kMaxJ];
  double av[kMaxJ];
  unsigned tg[kMaxJ];
  unsigned shm, prv;  // bit j: entry j is a real shared entry / a private entry (incl. ELL padding)
  double n2, y2;  // ||a~||^2 and RN(1/||a~||^2) (the division's reciprocal, formed in the look-ahead)
  __device__ __forceinline__ void pre(const SliceAddr& S, int W, int R, int lane, unsigned blk, unsigned xb) {
    shm = 0u;
    prv = 0u;
    {
      const SliceLayout Ly(R, W, true);
      n2 = lds64(blk + (unsigned)Ly.o_n2 + 8u * (lane < R ? lane : 0));
    }
    y2 = rcp_ahead(n2);
#pragma unroll
    for (int jb = 0; jb < kMaxJ; jb += kBatch) {
      if (jb < W) {
        unsigned ad[kBatch], c8[kBatch], m8[kBatch];
        double a8[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; u++) ad[u] = S.cb + min(jb + u, W - 1) * S.cs;
        lds32x8(c8, ad);
#pragma unroll
        for (int u = 0; u < kBatch; u++) ad[u] = S.mb + min(jb + u, W - 1) * S.cs;
        lds32x8(m8, ad);
#pragma unroll
        for (int u = 0; u < kBatch; u++) ad[u] = S.vb + min(jb + u, W - 1) * S.vs;
        lds64x8(a8, ad);
#pragma unroll
        for (int u = 0; u < kBatch; u++) {
          const int j = jb + u;
          av[j] = j < W ? a8[u] : 0.0;
          const bool sh = (c8[u] & kShared) != 0u;
          shm |= (sh && j < S.myl) ? (1u << j) : 0u;
          prv |= (!sh && j < W) ? (1u << j) : 0u;
          tg[j] = sh ? m8[u] : xb + 8u * (c8[u] & kIdx);
        }
      }
    }
  }
  __device__ __forceinline__ void poll(int W, unsigned long long* mbox_in) {
    unsigned pend = shm;
    while (true) {
#pragma unroll
      for (int j4 = 0; j4 < kMaxJ; j4 += 4)
        if (j4 < W) ldm4_if((pend >> j4) & 0xFu, mbox_in + j4, xr[j4], xr[j4 + 1], xr[j4 + 2], xr[j4 + 3]);
      unsigned np = 0u;
#pragma unroll
      for (int j = 0; j < kMaxJ; j++)
        if ((pend >> j) & 1u) np |= ((unsigned long long)__double_as_longlong(xr[j]) == kSentinel) ? (1u << j) : 0u;
      pend = np;
      if (!__any_sync(kFull, pend != 0u)) break;
      if (POBK_K2_POLLSLEEP) __nanosleep(POBK_K2_POLLSLEEP);
    }
#pragma unroll
    for (int j4 = 0; j4 < kMaxJ; j4 += 4)
      if (j4 < W) stm4_if((shm >> j4) & 0xFu, mbox_in + j4, kSentinel);
  }
  __device__ __forceinline__ void post(const SliceAddr& S, int W, unsigned xb, unsigned long long* mbox_in,
                                       unsigned long long* mbox, unsigned off_p, unsigned off_q, unsigned long long* trp,
                                       int prio = 0) {
    // private x~ of entries j < W (final once the tile's previous task is done): all loads in
    // flight before the first use; shared entries keep the polled value; entries >= W are +0
#pragma unroll
    for (int j = 0; j < kMaxJ; j++)
      if ((j & ~(kBatch - 1)) < W) xr[j] = ((shm >> j) & 1u) ? xr[j] : 0.0;
#pragma unroll
    for (int j4 = 0; j4 < kMaxJ; j4 += 4) {
      if (j4 < W)
        lds64x4_if(xr[j4], xr[j4 + 1], xr[j4 + 2], xr[j4 + 3], (prv >> j4) & 1u, (prv >> (j4 + 1)) & 1u, (prv >> (j4 + 2)) & 1u,
                   (prv >> (j4 + 3)) & 1u, tg[j4], tg[j4 + 1], tg[j4 + 2], tg[j4 + 3]);
    }
#if POBK_K2_PRIO
    if (prio) {  // operands in registers: let the interior warps at the shared-memory pipe
#pragma unroll
      for (int j = 0; j < kMaxJ; j++) asm volatile("mov.b64 %0, %0;" : "+d"(xr[j]));
      named_arrive(3, prio);
    }
#endif
    if (POBK_K2_FT && trp) {  // all private x~ loads complete
#pragma unroll
      for (int j = 0; j < kMaxJ; j++) asm volatile("mov.b64 %0, %0;" : "+d"(xr[j]));
      if ((threadIdx.x & 31) == 0) trp[11] = gtimer();
    }
    double s = 0.0;
#pragma unroll
    for (int jb = 0; jb < kMaxJ; jb += kChainB) {  // per group: products first, then the chain
      if (jb < W) {
        double pp[kChainB];
#pragma unroll
        for (int u = 0; u < kChainB; u++) pp[u] = pin(__dmul_rn(av[jb + u], xr[jb + u]));
#pragma unroll
        for (int u = 0; u < kChainB; u++) s = __dadd_rn(s, pp[u]);
      }
    }
    for (int j = kMaxJ; j < W; j++) {  // long rows: entries past the register window
      const unsigned cj = lds32(S.cb + j * S.cs);
      const double a = lds64(S.vb + j * S.vs);
      double x = 0.0;
      if ((cj & kShared) && j < S.myl) {
        unsigned long long w;
        do {
          w = ldm_if(1u, mbox_in + j, 0ull);
        } while (w == kSentinel);  // (re-armed in the write-back, after it is read again)
        x = __longlong_as_double((long long)w);
      } else if (!(cj & kShared)) {
        x = lds64(xb + 8u * (cj & kIdx));
      }
      s = __dadd_rn(s, __dmul_rn(a, x));
    }
    if (trp) {
      double s2 = s;
      asm volatile("mov.b64 %0, %0;" : "+d"(s2));
      __syncwarp();
      if ((threadIdx.x & 31) == 0) trp[2] = gtimer();
    }
    const double alpha = div_by_rcp(__dsub_rn(S.f, s), n2, y2);
    if (trp) {
      double a2 = alpha;
      asm volatile("mov.b64 %0, %0;" : "+d"(a2));
      __syncwarp();
      if ((threadIdx.x & 31) == 0) trp[9] = gtimer();
    }
#pragma unroll
    for (int j = 0; j < kMaxJ; j++) xr[j] = __dadd_rn(xr[j], __dmul_rn(alpha, av[j]));
    if (POBK_K2_FT && trp) {
      double a2 = xr[0];
      asm volatile("mov.b64 %0, %0;" : "+d"(a2));
      if ((threadIdx.x & 31) == 0) trp[6] = gtimer();
    }
#pragma unroll
    for (int j = 0; j < kMaxJ; j++) {  // write back: the targets are in registers (pre)
      if ((j & ~(kWB - 1)) < W) {
        const unsigned act = j < S.myl, sh = (shm >> j) & 1u;
        sts64_if(act & (sh ^ 1u), tg[j], xr[j]);
        stm_if(act & sh, mbox + ((tg[j] & ~kWrap) + ((tg[j] & kWrap) ? off_q : off_p)),
               (unsigned long long)__double_as_longlong(xr[j]));
      }
    }
    for (int j = kMaxJ; j < W; j++) {  // tail: the slot still holds the consumed value (re-armed now)
      const unsigned cj = lds32(S.cb + j * S.cs), idx = cj & kIdx;
      const double a = lds64(S.vb + j * S.vs);
      if ((cj & kShared) && j < S.myl) {
        const unsigned long long w = ldm_if(1u, mbox_in + j, 0ull);
        stm_if(1u, mbox_in + j, kSentinel);
        const double x1 = __dadd_rn(__longlong_as_double((long long)w), __dmul_rn(alpha, a));
        const unsigned mo = lds32(S.mb + j * S.cs);
        stm_if(1u, mbox + ((mo & ~kWrap) + ((mo & kWrap) ? off_q : off_p)), (unsigned long long)__double_as_longlong(x1));
      } else if (!(cj & kShared) && j < S.myl) {
        const unsigned ca = xb + 8u * idx;
        sts64_if(1u, ca, __dadd_rn(lds64(ca), __dmul_rn(alpha, a)));
      }
    }
    if (POBK_K2_FT && trp && (threadIdx.x & 31) == 0) trp[7] = gtimer();
  }
};
// ------------------------------------------------------------------ two right-hand sides (kR = 2)
// A two-RHS plan (pobk_solve_multi) streams A~ once per sweep for both:
// x~ is pair-interleaved in shared memory (column c's two values in one 16-byte word pair), a
// mailbox slot holds the pair, f~ the pair per row.  Each right-hand side runs the per-row
// contract of common.cuh on its own (same operations, same order as its single solve), so its
// iterates are bitwise those of its own solve; a right-hand side that has met its stop rule is
// frozen (its new values are its old ones: act bit q clear) while the other one iterates.
__device__ __forceinline__ void slice_interior2(const SliceAddr& S, int W, unsigned xb, unsigned act) {
  double s0 = 0.0, s1 = 0.0, n2 = 0.0;
  for (int jb = 0; jb < W; jb += kIB) {
    unsigned c[kIB];
    double av[kIB];
    double2 xv[kIB];
#pragma unroll
    for (int u = 0; u < kIB; u++) c[u] = lds16(S.cb + min(jb + u, W - 1) * S.cs);
#pragma unroll
    for (int u = 0; u < kIB; u++) xv[u] = lds128(xb + 16u * c[u]);
#pragma unroll
    for (int u = 0; u < kIB; u++) av[u] = lds64(S.vb + min(jb + u, W - 1) * S.vs);
    double p0[kIB], p1[kIB], qq[kIB];
#pragma unroll
    for (int u = 0; u < kIB; u++) {
      const bool in = jb + u < W;
      const double a = in ? av[u] : 0.0, x0 = in ? xv[u].x : 0.0, x1 = in ? xv[u].y : 0.0;
      p0[u] = pin(__dmul_rn(a, x0));
      p1[u] = pin(__dmul_rn(a, x1));
      qq[u] = pin(__dmul_rn(a, a));
    }
#pragma unroll
    for (int u = 0; u < kIB; u++) {
      s0 = __dadd_rn(s0, p0[u]);
      s1 = __dadd_rn(s1, p1[u]);
      n2 = __dadd_rn(n2, qq[u]);
    }
  }
  const double y2 = rcp_ahead(n2);  // (one reciprocal for both quotients)
  const double al0 = div_by_rcp(__dsub_rn(S.f, s0), n2, y2), al1 = div_by_rcp(__dsub_rn(S.f1, s1), n2, y2);
  for (int jb = 0; jb < W; jb += kIB) {
    unsigned c[kIB];
    double av[kIB];
    double2 xv[kIB];
#pragma unroll
    for (int u = 0; u < kIB; u++) {
      c[u] = lds16(S.cb + min(jb + u, W - 1) * S.cs);
      av[u] = lds64(S.vb + min(jb + u, W - 1) * S.vs);
    }
#pragma unroll
    for (int u = 0; u < kIB; u++) xv[u] = lds128(xb + 16u * c[u]);
#pragma unroll
    for (int u = 0; u < kIB; u++) {
      const double y0 = (act & 1u) ? __dadd_rn(xv[u].x, __dmul_rn(al0, av[u])) : xv[u].x;
      const double y1 = (act & 2u) ? __dadd_rn(xv[u].y, __dmul_rn(al1, av[u])) : xv[u].y;
      sts128_if(jb + u < S.myl, xb + 16u * c[u], y0, y1);
    }
  }
}

// slice_interior2 with pass 1's operands parked in TMEM (slice_interior_tm's scheme; 28 columns
// per 4-entry batch: the columns, the values and both right-hand sides' x~)
__device__ __forceinline__ void slice_interior2_tm(const SliceAddr& S, int W, unsigned xb, unsigned act, unsigned taddr) {
  static_assert(kIB == 4, "slice_interior2_tm parks 4-entry batches (28 TMEM columns each)");
  double s0 = 0.0, s1 = 0.0, n2 = 0.0;
  for (int jb = 0; jb < W; jb += kIB) {
    unsigned c[kIB];
    double av[kIB];
    double2 xv[kIB];
#pragma unroll
    for (int u = 0; u < kIB; u++) c[u] = lds16(S.cb + min(jb + u, W - 1) * S.cs);
#pragma unroll
    for (int u = 0; u < kIB; u++) xv[u] = lds128(xb + 16u * c[u]);
#pragma unroll
    for (int u = 0; u < kIB; u++) av[u] = lds64(S.vb + min(jb + u, W - 1) * S.vs);
    const unsigned ta = taddr + (unsigned)(jb / kIB) * 28u;
    tm_st4(ta, c[0], c[1], c[2], c[3]);
    tm_st4(ta + 4, __double2loint(av[0]), __double2hiint(av[0]), __double2loint(av[1]), __double2hiint(av[1]));
    tm_st4(ta + 8, __double2loint(av[2]), __double2hiint(av[2]), __double2loint(av[3]), __double2hiint(av[3]));
#pragma unroll
    for (int u = 0; u < kIB; u++)
      tm_st4(ta + 12 + 4 * u, __double2loint(xv[u].x), __double2hiint(xv[u].x), __double2loint(xv[u].y), __double2hiint(xv[u].y));
    double p0[kIB], p1[kIB], qq[kIB];
#pragma unroll
    for (int u = 0; u < kIB; u++) {
      const bool in = jb + u < W;
      const double a = in ? av[u] : 0.0, x0 = in ? xv[u].x : 0.0, x1 = in ? xv[u].y : 0.0;
      p0[u] = pin(__dmul_rn(a, x0));
      p1[u] = pin(__dmul_rn(a, x1));
      qq[u] = pin(__dmul_rn(a, a));
    }
#pragma unroll
    for (int u = 0; u < kIB; u++) {
      s0 = __dadd_rn(s0, p0[u]);
      s1 = __dadd_rn(s1, p1[u]);
      n2 = __dadd_rn(n2, qq[u]);
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  const double y2 = rcp_ahead(n2);  // (one reciprocal for both quotients)
  const double al0 = div_by_rcp(__dsub_rn(S.f, s0), n2, y2), al1 = div_by_rcp(__dsub_rn(S.f1, s1), n2, y2);
  for (int jb = 0; jb < W; jb += kIB) {
    const unsigned ta = taddr + (unsigned)(jb / kIB) * 28u;
    unsigned c[kIB], w[24];
    tm_ld4(ta, c[0], c[1], c[2], c[3]);
#pragma unroll
    for (int q = 0; q < 6; q++) tm_ld4(ta + 4 + 4 * q, w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int u = 0; u < kIB; u++) {
      const double av = __hiloint2double((int)w[2 * u + 1], (int)w[2 * u]);
      const double x0 = __hiloint2double((int)w[8 + 4 * u + 1], (int)w[8 + 4 * u]);
      const double x1 = __hiloint2double((int)w[8 + 4 * u + 3], (int)w[8 + 4 * u + 2]);
      const double y0 = (act & 1u) ? __dadd_rn(x0, __dmul_rn(al0, av)) : x0;
      const double y1 = (act & 2u) ? __dadd_rn(x1, __dmul_rn(al1, av)) : x1;
      sts128_if(jb + u < S.myl, xb + 16u * c[u], y0, y1);
    }
  }
}

// boundary slice of a two-RHS plan (BSlice's structure; a lane's mailbox words: entry j's pair at
// mbox_in + 2j, so one 256-bit load polls two entries)
struct BSliceR2 {
  double xr[kMaxJ][2];
  unsigned shm;
  __device__ __forceinline__ void pre(const SliceAddr& S, int W) {
    shm = 0u;
#pragma unroll
    for (int jb = 0; jb < kMaxJ; jb += kBatch) {
      if (jb < W) {
        unsigned cr[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; u++) cr[u] = lds32(S.cb + min(jb + u, W - 1) * S.cs);
#pragma unroll
        for (int u = 0; u < kBatch; u++) {
          const bool sh = (cr[u] & kShared) && jb + u < S.myl;
          shm |= sh ? (1u << (jb + u)) : 0u;
        }
      }
    }
  }
  __device__ __forceinline__ void poll(int W, unsigned long long* mbox_in) {
    unsigned pend = shm;
    while (true) {
#pragma unroll
      for (int j = 0; j < kMaxJ; j += 2)
        if (j < W) ldm4_if((pend >> j) & 3u, mbox_in + 2 * j, xr[j][0], xr[j][1], xr[j + 1][0], xr[j + 1][1]);
      unsigned np = 0u;
#pragma unroll
      for (int j = 0; j < kMaxJ; j++)
        if ((pend >> j) & 1u)
          np |= ((unsigned long long)__double_as_longlong(xr[j][0]) == kSentinel ||
                 (unsigned long long)__double_as_longlong(xr[j][1]) == kSentinel)
                    ? (1u << j)
                    : 0u;
      pend = np;
      if (!__any_sync(kFull, pend != 0u)) break;
    }
#pragma unroll
    for (int j = 0; j < kMaxJ; j += 2)
      if (j < W) stm4_if((shm >> j) & 3u, mbox_in + 2 * j, kSentinel);
  }
  __device__ __forceinline__ void post(const SliceAddr& S, int W, int R, unsigned xb, unsigned long long* mbox_in,
                                       unsigned long long* mbox, unsigned off_p, unsigned off_q, unsigned act) {
    constexpr int kG = 4;
    const double n2 = lds64(S.vb + (unsigned)SliceLayout(R, W, true, 2).o_n2);  // (vb = block + 8 * lane)
    const double y2 = rcp_ahead(n2);  // (independent of the row sums: overlaps them)
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int jb = 0; jb < kMaxJ; jb += kG) {
      if (jb < W) {
        double av[kG];
        double2 xp[kG];
        unsigned cr[kG];
#pragma unroll
        for (int u = 0; u < kG; u++) cr[u] = lds32(S.cb + min(jb + u, W - 1) * S.cs);
#pragma unroll
        for (int u = 0; u < kG; u++) xp[u] = lds128(xb + 16u * ((cr[u] & kShared) ? 0u : cr[u]));
#pragma unroll
        for (int u = 0; u < kG; u++) av[u] = jb + u < W ? lds64(S.vb + min(jb + u, W - 1) * S.vs) : 0.0;
        double p0[kG], p1[kG];
#pragma unroll
        for (int u = 0; u < kG; u++) {
          const int j = jb + u;
          const bool priv = j < W && !(cr[u] & kShared), sh = (shm >> j) & 1u;
          xr[j][0] = sh ? xr[j][0] : (priv ? xp[u].x : 0.0);
          xr[j][1] = sh ? xr[j][1] : (priv ? xp[u].y : 0.0);
          p0[u] = pin(__dmul_rn(av[u], xr[j][0]));
          p1[u] = pin(__dmul_rn(av[u], xr[j][1]));
        }
#pragma unroll
        for (int u = 0; u < kG; u++) {
          s0 = __dadd_rn(s0, p0[u]);
          s1 = __dadd_rn(s1, p1[u]);
        }
      }
    }
    for (int j = kMaxJ; j < W; j++) {  // long rows: entries past the register window
      const unsigned cj = lds32(S.cb + j * S.cs);
      const double a = lds64(S.vb + j * S.vs);
      double x0 = 0.0, x1 = 0.0;
      if ((cj & kShared) && j < S.myl) {
        unsigned long long w0, w1;
        do {
          w0 = ldm_if(1u, mbox_in + 2 * j, 0ull);
          w1 = ldm_if(1u, mbox_in + 2 * j + 1, 0ull);
        } while (w0 == kSentinel || w1 == kSentinel);
        x0 = __longlong_as_double((long long)w0);
        x1 = __longlong_as_double((long long)w1);
      } else if (!(cj & kShared)) {
        const double2 v = lds128(xb + 16u * (cj & kIdx));
        x0 = v.x;
        x1 = v.y;
      }
      s0 = __dadd_rn(s0, __dmul_rn(a, x0));
      s1 = __dadd_rn(s1, __dmul_rn(a, x1));
    }
    const double al0 = div_by_rcp(__dsub_rn(S.f, s0), n2, y2), al1 = div_by_rcp(__dsub_rn(S.f1, s1), n2, y2);
#pragma unroll
    for (int jb = 0; jb < kMaxJ; jb += kG) {
      if (jb < W) {
        double av[kG];
        unsigned mo[kG], cr[kG];
#pragma unroll
        for (int u = 0; u < kG; u++) {
          av[u] = lds64(S.vb + min(jb + u, W - 1) * S.vs);
          cr[u] = lds32(S.cb + min(jb + u, W - 1) * S.cs);
          mo[u] = lds32(S.mb + min(jb + u, W - 1) * S.cs);
        }
#pragma unroll
        for (int u = 0; u < kG; u++) {
          const int j = jb + u;
          const double y0 = (act & 1u) ? __dadd_rn(xr[j][0], __dmul_rn(al0, av[u])) : xr[j][0];
          const double y1 = (act & 2u) ? __dadd_rn(xr[j][1], __dmul_rn(al1, av[u])) : xr[j][1];
          const unsigned on = j < S.myl, sh = (shm >> j) & 1u;
          sts128_if(on & (sh ^ 1u), xb + 16u * (cr[u] & kIdx), y0, y1);
          stm2_if(on & sh, mbox + (2u * (mo[u] & ~kWrap) + ((mo[u] & kWrap) ? off_q : off_p)), y0, y1);
        }
      }
    }
    for (int j = kMaxJ; j < W; j++) {  // tail: the slot still holds the consumed pair (re-armed now)
      const unsigned cj = lds32(S.cb + j * S.cs), idx = cj & kIdx;
      const double a = lds64(S.vb + j * S.vs);
      if ((cj & kShared) && j < S.myl) {
        const double x0 = __longlong_as_double((long long)ldm_if(1u, mbox_in + 2 * j, 0ull));
        const double x1 = __longlong_as_double((long long)ldm_if(1u, mbox_in + 2 * j + 1, 0ull));
        stm_if(1u, mbox_in + 2 * j, kSentinel);
        stm_if(1u, mbox_in + 2 * j + 1, kSentinel);
        const double y0 = (act & 1u) ? __dadd_rn(x0, __dmul_rn(al0, a)) : x0;
        const double y1 = (act & 2u) ? __dadd_rn(x1, __dmul_rn(al1, a)) : x1;
        const unsigned mo = lds32(S.mb + j * S.cs);
        stm2_if(1u, mbox + (2u * (mo & ~kWrap) + ((mo & kWrap) ? off_q : off_p)), y0, y1);
      } else if (!(cj & kShared) && j < S.myl) {
        const unsigned ca = xb + 16u * idx;
        const double2 v = lds128(ca);
        const double y0 = (act & 1u) ? __dadd_rn(v.x, __dmul_rn(al0, a)) : v.x;
        const double y1 = (act & 2u) ? __dadd_rn(v.y, __dmul_rn(al1, a)) : v.y;
        sts128_if(1u, ca, y0, y1);
      }
    }
  }
};

// One instantiation per CTA shape: 256 threads (register-resident boundary slices, BSlice2) or
// 512 threads (BSlice).  (Round-2 experiments -- vector boundary slices, register-resident
// interior slices, dynamic slice claiming, strict boundary priority, tile placement by die --
// were measured and removed; with every path inlined into one kernel ptxas
// spilled and the sweep ran 2x slower.)
template <int kNT, bool kBReg, int kR>
__global__ void __launch_bounds__(kNT, 1) k2_sweeps(K2Args a) {
  static_assert(kR == 1 || (kR == 2 && !kBReg), "two-RHS plans use the BSliceR2 boundary path");
  constexpr int kNCW = kNT / 32 - 1;  // compute warps; warp kNCW is the TMA producer
  constexpr int kNC = kNCW * 32;      // compute threads
  constexpr int kPub = kNCW - 1;      // compute warp that runs the per-sweep grid decision
  // interior slices park pass 1's operands in TMEM for pass 2 (slice_interior_tm): each warp owns
  // a TMEM region of its lane quarter (warp % 4), 512 / (warps per quarter) columns wide
  constexpr bool kTM = POBK_K2_TMEM;
  constexpr int kTmCols = 512 / ((kNT / 32 + 3) / 4);        // columns per warp region (256 / 128)
  constexpr int kTmMaxW = kR == 1 ? (kTmCols / 20) * 4 : (kTmCols / 28) * kIB;  // widest slice whose operands fit
  constexpr int kTmMaxW8 = (kTmCols / 40) * 8;                                    // (8-entry batches)
  extern __shared__ __align__(128) unsigned char smem[];
  const int NS = a.NS;
  unsigned char* ring = smem;                                // NS * kSlot
  Ctl* ctl = (Ctl*)(smem + NS * kSlot);
  int4* smeta = (int4*)(ctl + 1);                            // [nsl_max]
  int4* cmeta = smeta + a.nsl_max;                           // [nck_max]
  int4* tmeta = cmeta + a.nck_max;                           // [ntask_max]
  double* xloc = (double*)(tmeta + a.ntask_max);             // [np_max + 1] private x~ + the zero slot

  const int t = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int s0 = a.tile_slice[t], nsl = a.tile_slice[t + 1] - s0;
  const int c0 = a.tile_chunk[t], nck = a.tile_chunk[t + 1] - c0;
  const int j0 = a.tile_task[t], ntask = a.tile_task[t + 1] - j0;
  const int q0 = a.pmap_ptr[t], np = a.pmap_ptr[t + 1] - q0;
  const long long maxs = a.ctrl->max_sweeps;
  const int mode = a.ctrl->stop_mode, every = a.ctrl->check_every;
  const bool rse = mode == POBK_STOP_RSE;
  // (constant during the solve: read once, not on the end-of-sweep decision path)
  const long long offset = a.ctrl->offset;
  const double tol = a.ctrl->tol, sden = sqrt(a.ctrl->den);
  const double sden1 = kR > 1 && rse ? sqrt(a.ctrl1->den) : 0.0;
  unsigned actm = kR > 1 ? 3u : 1u;  // right-hand sides still iterating

  if (tid == 0) {
    for (int i = 0; i < kMaxSlots; i++) {
      mbar_init(&ctl->full[i], 1);
      ctl->released[i] = 0;
    }
    ctl->issued = 0;
    ctl->stop = 0;
    ctl->done = 0;
    ctl->actm = actm;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int j = tid; j < nsl; j += kNT) smeta[j] = a.smeta[s0 + j];
  for (int j = tid; j < nck; j += kNT) cmeta[j] = a.cmeta[c0 + j];
  for (int j = tid; j < ntask; j += kNT) tmeta[j] = a.tmeta[j0 + j];
  if (tid < kR) xloc[kR * a.np_max + tid] = 0.0;  // the zero slot of the ELL padding (never written)
  for (int j = tid; j < np; j += kNT) {
    const int gcol = a.pmap[q0 + j];  // -1: a hole of the bank-aware placement
    xloc[kR * j] = gcol >= 0 ? a.xg[gcol] : 0.0;
    if (kR > 1) xloc[kR * j + 1] = gcol >= 0 ? a.xg1[gcol] : 0.0;
  }
  __shared__ unsigned s_tmem;
  if (kTM && warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (kTM) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (kTM) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem_w = kTM ? s_tmem + ((32u * (unsigned)(warp & 3)) << 16) + (unsigned)((warp >> 2) * kTmCols) : 0u;

  if (warp == kNCW) {
    // ================================================================ producer warp (TMA only)
    if (lane == 0 && nck > 0 && maxs > 0) {
      const unsigned long long pol = policy_evict_first();
      const unsigned char* tbase = a.stream + a.tile_off[t];
      int cum[kMaxSlots];
      for (int i = 0; i < kMaxSlots; i++) cum[i] = 0;
      // (RELRES: every checked sweep streams the tile's chunks once more for the residual)
      const unsigned long long gmax = (mode == POBK_STOP_RELRES ? 2ull : 1ull) * (unsigned long long)maxs * (unsigned long long)nck;
      unsigned long long g = 0;
      int slot = 0, c = 0;
      while (!ld_vol_shared(&ctl->stop)) {
        if (g >= gmax || (g >= (unsigned long long)NS && ld_vol_shared(&ctl->released[slot]) < cum[slot])) {
          if (POBK_K2_PSLEEP) __nanosleep(POBK_K2_PSLEEP);
          continue;
        }
        const int4 cm = cmeta[c];
        mbar_expect_tx(&ctl->full[slot], (unsigned)cm.y);
        tma_load_1d(ring + slot * kSlot, tbase + cm.x, (unsigned)cm.y, &ctl->full[slot], pol);
        cum[slot] += cm.z;
        g++;
        if (++slot == NS) slot = 0;
        if (++c == nck) c = 0;
        *(volatile unsigned long long*)&ctl->issued = g;
      }
      // drain: every issued copy must land before the CTA exits
      const unsigned long long h0 = g > (unsigned long long)NS ? g - NS : 0;
      for (unsigned long long h = h0; h < g; h++)
        mbar_wait(&ctl->full[(int)(h % (unsigned)NS)], (unsigned)((h / (unsigned)NS) & 1));
    }
  } else {
    // ================================================================ compute warps
    const unsigned xb = opaque(smem_u32(xloc));
    const unsigned ring_s = opaque(smem_u32(ring));
    long long sweep = 0;
    long long pass = 0;  // passes over the tile's stream: sweeps + RELRES residual passes
    long long nres = 0;  // RELRES residual passes done
    const int nck2 = nck % (2 * NS);
    int hbase = 0;  // (pass * nck) mod 2NS
    while (sweep < maxs) {
      const unsigned off_p = (unsigned)((sweep & 1) * a.NB * kR), off_q = (unsigned)(((sweep + 1) & 1) * a.NB * kR);
      unsigned long long* const mbox_p = a.mbox + off_p;  // this sweep's slots
      const bool tr = POBK_K2_DEV && a.trace != nullptr && sweep == a.trace_sweep;
      int rot = 0;  // round-robin offset (continues across tasks)
      for (int ti = 0; ti < ntask; ti++) {
        const int4 tm = tmeta[ti];
        const int nbnd = tm.y & 0xffff, ntot = nbnd + (tm.y >> 16);
        unsigned long long* trp = tr ? a.trace + ((size_t)t * a.ntask_max + ti) * 12 : nullptr;
        // this warp's slices of the task: q = qs, qs + qstep, ... < qe
        int qs, qe, qstep;
        {
          // continuous round-robin over all compute warps
          qs = warp >= rot ? warp - rot : warp - rot + kNCW;
          qe = ntot;
          qstep = kNCW;
          rot += ntot % kNCW;
          rot = rot >= kNCW ? rot - kNCW : rot;
        }
        if (tr && qs == 0 && lane == 0) trp[0] = gtimer();
        if (ti == ntask - 1 && warp == kPub && lane == 0 && rse && np > 0) {
          // the end-of-sweep RSE scan reads this tile's x~* next: bring it into L2 now
          const unsigned bytes = (unsigned)np * 8u;  // multiple of 128 (np: multiple of 16)
          for (int q = 0; q < kR; q++) {
            const char* xs0 = (const char*)((q == 0 ? a.xsp : a.xsp1) + q0);
            for (unsigned o = 0; o < bytes; o += 32768u) {
              const unsigned n = bytes - o < 32768u ? bytes - o : 32768u;
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(xs0 + o), "r"(n) : "memory");
            }
          }
        }
        // LOOK-AHEAD: this warp's first boundary slice of task ti (q = qs).  Its operands and the
        // neighbours' values (mailboxes) do not depend on the tile's task ti-1, so they are fetched
        // and awaited BEFORE the barrier that closes task ti-1; only the private x~ reads (post)
        // come after it.  (No deadlock: every slice of task ti-1 this warp owns is done, and the
        // producers of task ti's inputs are rows of earlier steps.)  The slice's chunk must not wait
        // for a ring slot that a slice of task ti frees: chunk g is issued once chunk g - NS is
        // consumed, so it has to lie within NS chunks of the task's first one.
        const int4 sl0 = smeta[tm.x + (qs < nbnd && qs < qe ? qs : 0)];
        const bool la = qs < nbnd && qs < qe && (sl0.x & 0xfffff) - (smeta[tm.x].x & 0xfffff) < NS;
        unsigned long long* const wtp = (POBK_K2_WT && tr && ti > 0) ? a.trace + ((size_t)t * a.ntask_max + ti - 1) * 12 : nullptr;
        if (POBK_K2_WT && wtp && lane == 0 && warp < 8) {
          wtp[warp] = clock64();
          if (la) atomicOr(&wtp[7], 1ull << warp);
        }
        if (!la && ti > 0) named_bar(1, kNC);  // the tile's task ti-1 is complete
        if (POBK_K2_WT && wtp && lane == 0 && warp == 0 && !la) wtp[8] = clock64();
#if POBK_K2_PRIO
        // boundary priority: the interior warps start the task once the look-ahead warps hold
        // their private operands (barrier 3: look-ahead warps arrive, the others sync)
        if (kBReg && !la) named_bar(3, kNC);
#endif
        for (int q = qs; q < qe; q += qstep) {
          const bool bnd = q < nbnd;
          const int4 sl = smeta[tm.x + q];
          const int chunk = sl.x & 0xfffff, R = sl.x >> 20, W = sl.z;
          const unsigned long long g = (unsigned long long)pass * nck + chunk;
          // ring position of chunk g without 64-bit division: h = g mod 2NS from the sweep's base
          // and the chunk's residue (precomputed); slot = h mod NS, phase parity = h >= NS
          int h = hbase + (sl.y >> 16);
          h = h >= 2 * NS ? h - 2 * NS : h;
          const int slot = h >= NS ? h - NS : h;
          while (ld_vol_shared64(&ctl->issued) <= g)  // ring full: let the others use the smem pipe
            if (POBK_K2_CSLEEP) __nanosleep(POBK_K2_CSLEEP);
          mbar_wait(&ctl->full[slot], h >= NS ? 1u : 0u);
          const unsigned blk = ring_s + (unsigned)(slot * kSlot + (sl.y & 0xffff));
          if (tr && lane == 0 && (q == 0 || (!POBK_K2_FT && q == nbnd))) trp[q == 0 ? 4 : 6] = gtimer();
          const SliceAddr S(blk, R, W, bnd, lane, kR);
          if (bnd) {
            unsigned long long* const mbox_in = mbox_p + (size_t)kR * (sl.w + (size_t)(lane < R ? lane : 0) * ((W + 3) & ~3));
            const bool bar = la && q == qs && ti > 0;  // look-ahead slice: barrier after the poll
            if constexpr (kR == 2) {
              BSliceR2 B;
              B.pre(S, W);
              B.poll(W, mbox_in);
              if (bar) named_bar(1, kNC);
              B.post(S, W, R, xb, mbox_in, a.mbox, off_p, off_q, actm);
            } else if constexpr (kBReg) {
              BSlice2 B;
              B.pre(S, W, R, lane, blk, xb);
              if (tr && q == 0 && lane == 0) trp[8] = gtimer();
              B.poll(W, mbox_in);
              if (tr && q == 0 && lane == 0) trp[1] = gtimer();
              if (POBK_K2_WT && bar && wtp && lane == 0 && warp < 8) wtp[warp] = clock64();
              if (bar) named_bar(1, kNC);
              if (POBK_K2_WT && bar && wtp && lane == 0 && warp == 0) wtp[8] = clock64();
              if (tr && q == 0 && lane == 0) trp[3] = gtimer();
              B.post(S, W, xb, mbox_in, a.mbox, off_p, off_q, (tr && q == 0) ? trp : nullptr, (la && q == qs) ? kNC : 0);
            } else {
              BSlice B;
              B.pre(S, W, xb);
              if (tr && q == 0 && lane == 0) trp[8] = gtimer();
              B.poll(S, W, R, mbox_in, (tr && q == 0) ? trp : nullptr);
              if (tr && q == 0 && lane == 0) trp[1] = gtimer();
              if (POBK_K2_WT && bar && wtp && lane == 0 && warp < 8) wtp[warp] = clock64();
              if (bar) named_bar(1, kNC);
              if (POBK_K2_WT && bar && wtp && lane == 0 && warp == 0) wtp[8] = clock64();
              if (tr && q == 0 && lane == 0) trp[3] = gtimer();
              B.post(S, W, xb, mbox_in, a.mbox, off_p, off_q, R, (tr && q == 0) ? trp : nullptr);
            }
            if (tr && q == 0) {
              __syncwarp();
              if (lane == 0) trp[10] = gtimer();
            }
          } else if constexpr (kR == 2) {
            if (kTM && W <= kTmMaxW) slice_interior2_tm(S, W, xb, actm, tmem_w);
            else slice_interior2(S, W, xb, actm);
          } else {
            if (kTM && kNT == 256 && W > kTmWide && W <= kTmMaxW8) slice_interior_tm<8>(S, W, xb, tmem_w);
            else if (kTM && W <= kTmMaxW) slice_interior_tm<4>(S, W, xb, tmem_w);
            else slice_interior(S, W, xb);
          }
          __syncwarp();
          if (lane == 0) atomicAdd(&ctl->released[slot], 1);
          if (tr && lane == 0 && (q == 0 || (!POBK_K2_FT && q == nbnd))) trp[q == 0 ? 5 : 7] = gtimer();
        }
      }
      named_bar(1, kNC);  // the sweep's last task is complete
      sweep++;
      pass++;
      hbase += nck2;
      hbase = hbase >= 2 * NS ? hbase - 2 * NS : hbase;
      // ---- end of sweep: a grid barrier every sweep (it also orders the mailbox re-arms of this
      //      sweep before the writes of the next ones); the stop test when due
      const bool due_check = ((sweep + offset) % every) == 0 || sweep >= maxs;
      const bool due = mode != POBK_STOP_NONE && due_check;
      if (kR == 1 && mode == POBK_STOP_RELRES && due_check) {  // (two-RHS plans: RSE / none only)
        // RELRES = ||f~ - A~ x~||_2 / ||f~||_2 at the end of the sweep (the fused
        // SpMV + norm of the north star): (1) the last-writer tile of every shared column
        // publishes the column's sweep-final value (its wrap slot) to x~ in global memory; (2) a
        // grid barrier; (3) a residual pass over the tile's own stream (the producer streams the
        // tile's chunks once more), private x~ from shared memory, shared x~ from global memory;
        // per-row residuals in fixed order per lane, then the fixed-order reductions below.
        const unsigned long long* wrap = a.mbox + (size_t)(sweep & 1) * a.NB;
        for (int j = a.lastcol_ptr[t] + tid; j < a.lastcol_ptr[t + 1]; j += kNC)
          a.xg[a.lastcol[j]] = __longlong_as_double((long long)ldm_if(1u, wrap + a.lastslot[j], 0ull));
        __threadfence();
        named_bar(1, kNC);
        nres++;
        if (tid == 0) {
          atomicAdd(&a.sync->arrive2, 1ull);
          const unsigned long long target = (unsigned long long)nres * (unsigned long long)a.T;
          while (ld_acquire_u64(&a.sync->arrive2) < target) {
          }
          __threadfence();
        }
        named_bar(1, kNC);
        double acc = 0.0;
        int rr = 0;  // running slice index: slice rr goes to compute warp rr mod kNCW
        for (int ti = 0; ti < ntask; ti++) {
          const int4 tm = tmeta[ti];
          const int nbnd = tm.y & 0xffff, ntot = nbnd + (tm.y >> 16);
          for (int q = 0; q < ntot; q++, rr = rr + 1 == kNCW ? 0 : rr + 1) {
            if (rr != warp) continue;
            const int4 sl = smeta[tm.x + q];
            const int chunk = sl.x & 0xfffff, R = sl.x >> 20, W = sl.z;
            const unsigned long long g = (unsigned long long)pass * nck + chunk;
            int h = hbase + (sl.y >> 16);
            h = h >= 2 * NS ? h - 2 * NS : h;
            const int slot = h >= NS ? h - NS : h;
            while (ld_vol_shared64(&ctl->issued) <= g)
              if (POBK_K2_CSLEEP) __nanosleep(POBK_K2_CSLEEP);
            mbar_wait(&ctl->full[slot], h >= NS ? 1u : 0u);
            const unsigned blk = ring_s + (unsigned)(slot * kSlot + (sl.y & 0xffff));
            const SliceAddr S(blk, R, W, q < nbnd, lane);
            if (lane < R) {
              double sr = 0.0;
              for (int j = 0; j < W; j++) {
                const unsigned c = q < nbnd ? lds32(S.cb + j * S.cs) : lds16(S.cb + j * S.cs);
                const double av = lds64(S.vb + j * S.vs);
                const double xv = (c & kShared) ? ld_cg(a.xg + (c & kIdx)) : lds64(xb + 8u * c);
                sr = __dadd_rn(sr, __dmul_rn(av, xv));
              }
              const double r = __dsub_rn(S.f, sr);
              acc = fma(r, r, acc);
            }
            __syncwarp();
            if (lane == 0) atomicAdd(&ctl->released[slot], 1);
          }
        }
        pass++;
        hbase += nck2;
        hbase = hbase >= 2 * NS ? hbase - 2 * NS : hbase;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);  // fixed lane order
        if (lane == 0) ctl->part[warp] = acc;
      }
      if (kR == 2 && mode == POBK_STOP_RSE && due) {
        // the scan below for both right-hand sides (x~ pairs in shared memory and the mailboxes),
        // each in the single scan's order (so each RSE is bitwise its single solve's)
        double acc0 = 0.0, acc1 = 0.0;
        const double2* xl2 = (const double2*)xloc;  // column c: (rhs 0, rhs 1)
        const double2* xs0p = (const double2*)(a.xsp + q0);
        const double2* xs1p = (const double2*)(a.xsp1 + q0);
        const int np2 = np >> 1;
        for (int j0 = tid; j0 < np2; j0 += kRU * kNC) {
          double2 s0[kRU], s1[kRU];
#pragma unroll
          for (int u = 0; u < kRU; u++) {
            const bool in = j0 + u * kNC < np2;
            s0[u] = in ? __ldg(xs0p + j0 + u * kNC) : make_double2(0.0, 0.0);
            s1[u] = in ? __ldg(xs1p + j0 + u * kNC) : make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int u = 0; u < kRU; u++)
            if (j0 + u * kNC < np2) {
              const double2 xa = xl2[2 * (j0 + u * kNC)], xb2 = xl2[2 * (j0 + u * kNC) + 1];
              double d = xa.x - s0[u].x;
              acc0 = fma(d, d, acc0);
              d = xb2.x - s0[u].y;
              acc0 = fma(d, d, acc0);
              d = xa.y - s1[u].x;
              acc1 = fma(d, d, acc1);
              d = xb2.y - s1[u].y;
              acc1 = fma(d, d, acc1);
            }
        }
        const unsigned long long* wrap = a.mbox + (size_t)(sweep & 1) * a.NB * 2;
        const int lc1 = a.lastcol_ptr[t + 1];
        for (int j0 = a.lastcol_ptr[t] + tid; j0 < lc1; j0 += kRU * kNC) {
          int sl4[kRU];
          double xs0[kRU], xs1[kRU];
#pragma unroll
          for (int u = 0; u < kRU; u++) {
            const bool in = j0 + u * kNC < lc1;
            sl4[u] = in ? __ldg(a.lastslot + j0 + u * kNC) : 0;
            xs0[u] = in ? __ldg(a.lcx + j0 + u * kNC) : 0.0;
            xs1[u] = in ? __ldg(a.lcx1 + j0 + u * kNC) : 0.0;
          }
          unsigned long long w0[kRU], w1[kRU];
#pragma unroll
          for (int u = 0; u < kRU; u++) {
            const unsigned in = j0 + u * kNC < lc1 ? 1u : 0u;
            w0[u] = ldm_if(in, wrap + 2 * (size_t)sl4[u], 0ull);
            w1[u] = ldm_if(in, wrap + 2 * (size_t)sl4[u] + 1, 0ull);
          }
#pragma unroll
          for (int u = 0; u < kRU; u++)
            if (j0 + u * kNC < lc1) {
              const double d0 = __longlong_as_double((long long)w0[u]) - xs0[u];
              const double d1 = __longlong_as_double((long long)w1[u]) - xs1[u];
              acc0 = fma(d0, d0, acc0);
              acc1 = fma(d1, d1, acc1);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          acc0 += __shfl_xor_sync(kFull, acc0, o);
          acc1 += __shfl_xor_sync(kFull, acc1, o);
        }
        if (lane == 0) {
          ctl->part[warp] = acc0;
          ctl->part[32 + warp] = acc1;
        }
      } else if (mode == POBK_STOP_RSE && due) {
        // columns final for this sweep once the tile's last task is done: the private ones, and
        // the shared ones whose last writer (row of the highest step) is in this tile.  x~* of the
        // private columns is contiguous per tile (16-B loads, prefetched into L2 during the
        // sweep's last task); 4 x 16 B in flight per thread
        double acc = 0.0;
        const double2* xsp2 = (const double2*)(a.xsp + q0);  // (q0, np: multiples of 16)
        const int np2 = np >> 1;
        const double2* xl2 = (const double2*)xloc;
        for (int j0 = tid; j0 < np2; j0 += kRU * kNC) {
          double2 xs[kRU];
#pragma unroll
          for (int u = 0; u < kRU; u++) xs[u] = j0 + u * kNC < np2 ? __ldg(xsp2 + j0 + u * kNC) : make_double2(0.0, 0.0);
#pragma unroll
          for (int u = 0; u < kRU; u++)
            if (j0 + u * kNC < np2) {
              const double2 xv = xl2[j0 + u * kNC];
              const double d0 = xv.x - xs[u].x, d1 = xv.y - xs[u].y;
              acc = fma(d0, d0, acc);
              acc = fma(d1, d1, acc);
            }
        }
        // owned shared columns: slot indices and x~* first (independent), then the wrap slots --
        // two dependent global round trips per thread instead of two per element
        const unsigned long long* wrap = a.mbox + (size_t)(sweep & 1) * a.NB;  // sweep = sweeps done
        const int lc1 = a.lastcol_ptr[t + 1];
        for (int j0 = a.lastcol_ptr[t] + tid; j0 < lc1; j0 += kRU * kNC) {
          int sl4[kRU];
          double xs4[kRU];
#pragma unroll
          for (int u = 0; u < kRU; u++) {
            const bool in = j0 + u * kNC < lc1;
            sl4[u] = in ? __ldg(a.lastslot + j0 + u * kNC) : 0;
            xs4[u] = in ? __ldg(a.lcx + j0 + u * kNC) : 0.0;
          }
          unsigned long long w4[kRU];
#pragma unroll
          for (int u = 0; u < kRU; u++) w4[u] = ldm_if(j0 + u * kNC < lc1 ? 1u : 0u, wrap + sl4[u], 0ull);
#pragma unroll
          for (int u = 0; u < kRU; u++)
            if (j0 + u * kNC < lc1) {
              const double d = __longlong_as_double((long long)w4[u]) - xs4[u];
              acc = fma(d, d, acc);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);  // fixed lane order
        if (lane == 0) ctl->part[warp] = acc;
      }
      named_bar(1, kNC);
      if (warp == kPub) {
        // grid barrier, one hop: publish the tile's partial, arrive on a monotonic counter, wait
        // until all T tiles of this sweep have arrived; then EVERY tile forms the same total (fixed
        // order) and takes the same decision -- no second, releasing hop
        const int par = (int)(sweep & 1);
        if (lane == 0) {
          for (int q = 0; q < kR; q++) {
            double part = 0.0;
            if (due)
              for (int w2 = 0; w2 < kNCW; w2++) part += ((volatile double*)ctl->part)[32 * q + w2];
            a.partials[(par * kR + q) * a.T + t] = part;
          }
          __threadfence();
          atomicAdd(&a.sync->arrive, 1ull);
          const unsigned long long target = (unsigned long long)sweep * (unsigned long long)a.T;
          while (ld_acquire_u64(&a.sync->arrive) < target) {
          }
        }
        __syncwarp();
        (void)ld_acquire_u64(&a.sync->arrive);  // (each lane: acquire before reading partials)
        int st = sweep >= maxs, term = POBK_TERM_MAX_SWEEPS;
        double v = 0.0;
        if constexpr (kR == 2) {
          // each right-hand side still iterating takes its own decision; a
          // stopped one is frozen and keeps its record; the kernel ends when none is left
          unsigned nact = actm;
          for (int q = 0; q < 2; q++) {
            if (!due || !((actm >> q) & 1u)) continue;
            const double* pq = a.partials + (par * 2 + q) * a.T;
            double tot = 0.0;
            for (int b0 = 0; b0 < a.T; b0 += 32) tot += b0 + lane < a.T ? ld_cg(pq + b0 + lane) : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(kFull, tot, o);
            const double vq = sqrt(tot) / (q ? sden1 : sden);
            const int tq = !isfinite(vq) ? POBK_TERM_NONFINITE : (vq < tol ? POBK_TERM_CONVERGED : -1);
            Ctrl* cq = q ? a.ctrl1 : a.ctrl;
            if (lane == 0 && t == 0) {
              cq->value = vq;
              if (tq >= 0) {
                cq->sweeps = sweep;
                cq->term = tq;
              }
            }
            if (tq >= 0) nact &= ~(1u << q);
          }
          if (sweep >= maxs && lane == 0 && t == 0)
            for (int q = 0; q < 2; q++)
              if ((nact >> q) & 1u) {
                Ctrl* cq = q ? a.ctrl1 : a.ctrl;
                cq->sweeps = sweep;
                cq->term = POBK_TERM_MAX_SWEEPS;
              }
          st = nact == 0u || sweep >= maxs;
          if (lane == 0) *(volatile unsigned*)&ctl->actm = nact;
        } else if (due) {
          double tot = 0.0;  // fixed order: lane l sums tiles l, l+32, ..., then a fixed butterfly
          {  // (loads first, then the adds in the same order; T <= 160 in one round trip)
            double pv[5];
#pragma unroll
            for (int u = 0; u < 5; u++) pv[u] = u * 32 + lane < a.T ? ld_cg(a.partials + par * a.T + u * 32 + lane) : 0.0;
#pragma unroll
            for (int u = 0; u < 5; u++) tot += pv[u];
          }
          for (int b0 = 160; b0 < a.T; b0 += 32)
            tot += b0 + lane < a.T ? ld_cg(a.partials + par * a.T + b0 + lane) : 0.0;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(kFull, tot, o);
          v = sqrt(tot) / sden;
          if (!isfinite(v)) { st = 1; term = POBK_TERM_NONFINITE; }
          else if (v < tol) { st = 1; term = POBK_TERM_CONVERGED; }
        }
        if (lane == 0) {
          if (kR == 1 && st && t == 0) {  // (every tile holds the same values)
            if (due) a.ctrl->value = v;
            a.ctrl->sweeps = sweep;
            a.ctrl->term = term;
          }
          *(volatile int*)&ctl->stop = st;
        }
      }
      named_bar(2, kNC);
      if (kR > 1) actm = *(volatile unsigned*)&ctl->actm;
      if (ld_vol_shared(&ctl->stop)) {
        if (tid == 0) ctl->done = sweep;
        break;
      }
    }
  }
  if (kTM) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (kTM && warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem) : "memory");
  }
  for (int j = tid; j < np; j += kNT) {
    const int gcol = a.pmap[q0 + j];
    if (gcol >= 0) {
      a.xg[gcol] = xloc[kR * j];
      if (kR > 1) a.xg1[gcol] = xloc[kR * j + 1];
    }
  }
  {  // shared columns owned by this tile: their final value sits in the last sweep's wrap slot
    const long long done = min(maxs, (long long)ctl->done);
    const unsigned long long* wrap = a.mbox + (size_t)(done & 1) * a.NB * kR;
    for (int j = a.lastcol_ptr[t] + tid; j < a.lastcol_ptr[t + 1]; j += kNT) {
      a.xg[a.lastcol[j]] = __longlong_as_double((long long)ldm_if(1u, wrap + (size_t)kR * a.lastslot[j], 0ull));
      if (kR > 1) a.xg1[a.lastcol[j]] = __longlong_as_double((long long)ldm_if(1u, wrap + (size_t)kR * a.lastslot[j] + 1, 0ull));
    }
  }
}

// x~* of the private columns in tile-local order (holes: 0) and of the owned shared columns, for
// the end-of-sweep RSE scan (contiguous per tile: no dependent gathers at the end of a sweep)
__global__ void k2_gather_xs(int n, const int* __restrict__ pmap, int nl, const int* __restrict__ lastcol,
                             const double* __restrict__ xst, double* __restrict__ xsp, double* __restrict__ lcx) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n + nl; i += gridDim.x * blockDim.x) {
    if (i < n) {
      const int c = pmap[i];
      xsp[i] = c >= 0 ? xst[c] : 0.0;
    } else {
      lcx[i - n] = xst[lastcol[i - n]];
    }
  }
}

__global__ void k2_reset(SyncState* sync) {
  sync->arrive = 0;
  sync->arrive2 = 0;
}

// every mailbox slot empty, then each shared column's first reader of sweep 0 gets x~0
__global__ void k2_mbox_fill(unsigned long long* mbox, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    mbox[i] = kSentinel;
}
// (kR right-hand sides: slot s's words at kR s + q; this call seeds right-hand side q)
__global__ void k2_mbox_seed(unsigned long long* mbox, int n, const int* __restrict__ idx, const int* __restrict__ col,
                             const double* __restrict__ xt, int kR, int q) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double v = xt[col[i]];
    if (v != v) v = __longlong_as_double(0x7FF8000000000000ll);  // a NaN x0 never reads as the sentinel
    mbox[(size_t)kR * idx[i] + q] = (unsigned long long)__double_as_longlong(v);
  }
}

// f (user frame) into the f~ slots of the slice stream
__global__ void k2_scatter_f(int64_t m, const int32_t* __restrict__ orig, const int64_t* __restrict__ fslot,
                             const double* __restrict__ f, double* __restrict__ stream_d) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x)
    stream_d[fslot[q]] = f[orig[q]];
}
}  // namespace

struct K2Plan {
  int T = 0, NS = 0;
  int nt = 256;                // threads per CTA: 256 (BSlice2) or 512 (BSlice), see k2_build
  int kR = 1;                  // right-hand sides per sweep (2: the two-RHS plan of pobk_solve_multi)
  size_t smem = 0;
  int nsl_max = 1, nck_max = 1, ntask_max = 1, np_max = 1;
  unsigned char* stream = nullptr;
  long long* tile_off = nullptr;
  unsigned long long* trace = nullptr;
  int4 *smeta = nullptr, *cmeta = nullptr, *tmeta = nullptr;
  int *tile_slice = nullptr, *tile_chunk = nullptr, *tile_task = nullptr, *pmap_ptr = nullptr, *pmap = nullptr,
      *lastcol_ptr = nullptr, *lastcol = nullptr, *lastslot = nullptr, *seed_idx = nullptr, *seed_col = nullptr;
  unsigned long long* mbox = nullptr;
  double* xsp = nullptr;       // [npmap] private x~* in tile-local order
  double* lcx = nullptr;       // [nlast] owned shared columns' x~*
  double *xsp1 = nullptr, *lcx1 = nullptr;  // (kR = 2) the second right-hand side's
  double *xt2[2] = {nullptr, nullptr}, *xst2[2] = {nullptr, nullptr};  // (kR = 2) x~, x~* per right-hand side
  Ctrl* ctrl2 = nullptr;       // (kR = 2) [2] device stop records
  Ctrl* h_ctrl2 = nullptr;     // pinned mirror
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  int npmap = 0, nlast = 0;
  long long NB = 0;
  int nseed = 0;
  SyncState* sync = nullptr;
  double* partials = nullptr;
  int32_t* orig_q = nullptr;   // stream-order row -> user-frame row
  int64_t* fslot = nullptr;    // stream-order row -> double index of its f~ slot in the stream
  std::vector<void*> allocs;
  // stats (bench)
  double private_frac = 0.0;   // fraction of nnz whose column is private
  double interior_frac = 0.0;  // fraction of rows that are interior
  long long stream_bytes = 0;
  long long pad_entries = 0;   // ELL padding entries in the stream
  int nchunks = 0;
  int ntask_total = 0;
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

bool k2_build(Plan& p, const HostCSR& At, const std::vector<double>& nrm2, int tile_rows, std::string& why, int kR) {
  if (p.any_overlap) { why = "overlapping categories"; return false; }
  int sms = 148;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, p.device) == cudaSuccess) sms = prop.multiProcessorCount;
  const int64_t m = p.m;
  int T = sms;
  if (tile_rows > 0) T = (int)std::max<int64_t>(1, std::min<int64_t>(T, (m + tile_rows - 1) / tile_rows));
  // at least ~1k nonzeros per tile (config 2: 43 -> 148 tiles, 72.5 -> 63.2 us/sweep, measured)
  const int64_t tile_nnz_min = getenv("POBK_K2_TILE_NNZ") ? atoll(getenv("POBK_K2_TILE_NNZ")) : 1024;
  T = (int)std::min<int64_t>(T, std::max<int64_t>(1, p.nnz / std::max<int64_t>(1, tile_nnz_min)));
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

  // columns: owner tile / shared; a column no row touches stays constant and is kept private to
  // tile 0 (it still counts in the RSE)
  std::vector<int32_t> col_tile(m, -1);
  std::vector<uint8_t> shared(m, 0);
  for (int64_t i = 0; i < m; i++)
    for (int64_t q = At.ptr[i]; q < At.ptr[i + 1]; q++) {
      const int32_t c = At.col[q];
      if (col_tile[c] < 0) col_tile[c] = tile[i];
      else if (col_tile[c] != tile[i]) shared[c] = 1;
    }
  for (int64_t c = 0; c < m; c++)
    if (col_tile[c] < 0) col_tile[c] = 0;
  // private columns per tile (ascending), capped so that kMinSlots ring slots still fit
  const size_t fixed = sizeof(Ctl) + 128;
  // (16 B per column: conservative -- x~ takes 8 -- so that tiles keep a deep TMA ring)
  // bytes of shared memory budgeted per private column: 8 (x~ only; the ring takes what remains,
  // at least kMinSlots slots), so that half-GPU tilings (batched solves on two lanes) stay private
  const int pcb = getenv("POBK_K2_PCB") ? std::max(8, atoi(getenv("POBK_K2_PCB"))) : 8;
  const int np_cap = (int)((kSmemTotal - fixed - kMetaBudget - (size_t)kMinSlots * kSlot) / (pcb * kR) / 1.04) - 48;
  std::vector<int32_t> local(m, -1);
  std::vector<int> pmap_ptr(T + 1, 0);
  std::vector<int> pmap;
  std::vector<int> np_t(T, 0);
  {
    std::vector<std::vector<int32_t>> per(T);
    for (int64_t c = 0; c < m; c++)
      if (!shared[c]) per[col_tile[c]].push_back((int32_t)c);
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
  // rows: interior (all columns private) or boundary
  std::vector<uint8_t> boundary(m, 0);
  int64_t n_private_nnz = 0, n_interior = 0;
  for (int64_t i = 0; i < m; i++) {
    const int64_t len = At.ptr[i + 1] - At.ptr[i];
    if (len > 65535 || SliceLayout(1, (int)len, true, kR).bytes > kSlot) {
      why = "row " + std::to_string(i) + " (" + std::to_string(len) + " nonzeros) is too long for one " +
            std::to_string(kSlot) + "-byte slice";
      return false;
    }
    for (int64_t q = At.ptr[i]; q < At.ptr[i + 1]; q++) {
      if (shared[At.col[q]]) boundary[i] = 1;
      else n_private_nnz++;
    }
    n_interior += !boundary[i];
  }
  // tasks (tile, step): boundary slices first, then interior slices; each group is sorted by
  // decreasing row length (then row id) and cut into slices of <= 32 rows (ELL inside a slice)
  std::vector<std::vector<std::vector<int32_t>>> rows_tk(T);
  for (int t = 0; t < T; t++) rows_tk[t].resize(p.nsteps);
  for (int k = 0; k < p.nsteps; k++)
    for (int q = p.sched.step_ptr[k]; q < p.sched.step_ptr[k + 1]; q++) {
      const int32_t r = p.sched.rows[q];
      rows_tk[tile[r]][k].push_back(r);
    }
  auto rlen = [&](int32_t r) { return (int)(At.ptr[r + 1] - At.ptr[r]); };
  // CTA size (see the upload below): from the one-lane slicing's slices per task
  int nt_choice = 256;
  {
    long long ns = 0, ntk = 0;
    for (int t = 0; t < T; t++)
      for (int k = 0; k < p.nsteps; k++) {
        if (rows_tk[t][k].empty()) continue;
        int nb = 0;
        for (int32_t r : rows_tk[t][k]) nb += boundary[r];
        const int ni = (int)rows_tk[t][k].size() - nb;
        ns += (nb + kSliceRows - 1) / kSliceRows + (ni + kSliceRows - 1) / kSliceRows;
        ntk++;
      }
    nt_choice = (double)ns / std::max<long long>(ntk, 1) > 10.0 ? 512 : 256;
    if (const char* e = getenv("POBK_K2_THREADS")) nt_choice = atoi(e) == 512 ? 512 : 256;  // development override
  }
  std::vector<int4> smeta, cmeta, tmeta;
  std::vector<int> tile_slice(T + 1, 0), tile_chunk(T + 1, 0), tile_task(T + 1, 0);
  std::vector<std::vector<int32_t>> slice_rows;  // global slice order
  std::vector<int64_t> slice_pos;                // byte offset of each slice in the stream
  std::vector<uint8_t> slice_bnd;
  std::vector<int64_t> mb_of_row(m, -1);         // boundary rows: mailbox index of entry 0
  long long off = 0, pad = 0, NB = 0;
  int nsl_max = 1, nck_max = 1, ntask_max = 1;
  for (int t = 0; t < T; t++) {
    const int sl0 = (int)smeta.size();
    int chunk_local = -1, chunk_bytes = kSlot;  // force a new chunk for the tile's first slice
    const long long tile_base = off;
    for (int k = 0; k < p.nsteps; k++) {
      if (rows_tk[t][k].empty()) continue;
      int cnt[2] = {0, 0};
      const int first = (int)smeta.size() - sl0;
      for (int kind = 0; kind < 2; kind++) {  // 0: boundary, 1: interior
        const bool bnd = kind == 0;
        std::vector<int32_t> g;
        for (int32_t r : rows_tk[t][k])
          if (boundary[r] == (uint8_t)bnd) g.push_back(r);
        std::stable_sort(g.begin(), g.end(), [&](int32_t x, int32_t y) { return rlen(x) > rlen(y); });
        size_t a = 0;
        while (a < g.size()) {
          const int W = rlen(g[a]);
          size_t b = a;
          while (b < g.size() && (int)(b - a) < kSliceRows && SliceLayout((int)(b - a + 1), W, bnd, kR).bytes <= kSlot) b++;
          const int R = (int)(b - a), bytes = SliceLayout(R, W, bnd, kR).bytes;
          for (size_t r = a; r < b; r++) pad += W - rlen(g[r]);
          if (chunk_bytes + bytes > kSlot) {  // open a new chunk
            chunk_local++;
            chunk_bytes = 0;
            cmeta.push_back(make_int4((int)(off - tile_base), 0, 0, 0));
          }
          if (chunk_local >= (1 << 20)) { why = "too many chunks in tile " + std::to_string(t); return false; }
          int mbase = 0;
          if (bnd) {
            const int Wp = (W + 3) & ~3;  // a lane's slots: contiguous, 32-byte aligned groups of 4
            if (2 * kR * (NB + (long long)Wp * R) >= (1LL << 31)) { why = "too many boundary entries for the mailboxes"; return false; }
            mbase = (int)NB;
            for (int r = 0; r < R; r++) mb_of_row[g[a + r]] = NB + (long long)r * Wp;
            NB += (long long)Wp * R;
          }
          smeta.push_back(make_int4(chunk_local | (R << 20), chunk_bytes, W, mbase));
          slice_rows.emplace_back(g.begin() + a, g.begin() + b);
          slice_pos.push_back(off);
          slice_bnd.push_back(bnd);
          cmeta.back().y += bytes;
          cmeta.back().z += 1;
          chunk_bytes += bytes;
          off += bytes;
          cnt[kind]++;
          a = b;
        }
      }
      if (cnt[0] > 0xffff || cnt[1] > 0x7fff) { why = "too many slices in one task"; return false; }
      tmeta.push_back(make_int4(first, cnt[0] | (cnt[1] << 16), k, 0));
    }
    tile_slice[t + 1] = (int)smeta.size();
    tile_chunk[t + 1] = (int)cmeta.size();
    tile_task[t + 1] = (int)tmeta.size();
    nsl_max = std::max(nsl_max, tile_slice[t + 1] - tile_slice[t]);
    nck_max = std::max(nck_max, tile_chunk[t + 1] - tile_chunk[t]);
    ntask_max = std::max(ntask_max, tile_task[t + 1] - tile_task[t]);
  }
  const size_t meta_bytes = 16 * ((size_t)nsl_max + nck_max + ntask_max);
  if (meta_bytes > (size_t)kMetaBudget) {
    why = "K2 metadata (" + std::to_string(meta_bytes) + " B per tile) exceeds its shared-memory budget";
    return false;
  }
  // Bank-aware placement of the private x~ in shared memory.  A warp's access to entry j of its
  // slice touches one 8-byte word per lane, served per half warp (16 words = one 128-B wavefront);
  // words w and w' of one half conflict when w = w' (mod 16) (same bank pair), and each half takes
  // max over residues of the number of distinct words, >= 1 (ncu: 4.5 wavefronts per access with
  // the former whole-warp model vs an ideal 2).
  // Random placement costs ~5; here each tile's private columns get residues greedily (most
  // accessed first), each residue chosen to minimise the column's collisions with the residues
  // already in its access groups, under a per-residue capacity; local index = residue + 16 * rank.
  double bank_stats[3] = {0, 0, 0};
  {
    pmap.clear();
    for (int t = 0; t < T; t++) {
      const int b = pmap_ptr[t], e = pmap_ptr[t + 1], n = e - b;
      pmap_ptr[t] = (int)pmap.size();
      if (n == 0) { np_t[t] = 0; continue; }
      // access groups of this tile: (slice, j); member lists per private column (by old local index)
      std::vector<int32_t> cols(n);
      std::vector<std::vector<int32_t>> groups_of(n);
      int ng = 0;
      // an 8-byte warp access is served per HALF warp (lanes 0-15, 16-31: 16 words = 128 B per
      // wavefront), so an access group is (slice, entry j, half)
      for (int si = tile_slice[t]; si < tile_slice[t + 1]; si++) {
        const auto& rows = slice_rows[si];
        const int W = smeta[si].z;
        for (int j = 0; j < W; j++, ng += 2)
          for (size_t r = 0; r < rows.size(); r++) {
            const int32_t i = rows[r];
            if (j < rlen(i)) {
              const int32_t cg = At.col[At.ptr[i] + j];
              if (!shared[cg]) groups_of[local[cg]].push_back(ng + (r >= 16 ? 1 : 0));
            }
          }
      }
      std::vector<int32_t> gl;  // old local -> global column
      gl.resize(n);
      for (int64_t c = 0; c < m; c++)
        if (!shared[c] && col_tile[c] == t && local[c] >= 0) gl[local[c]] = (int32_t)c;
      std::vector<int> order(n);
      std::iota(order.begin(), order.end(), 0);
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return groups_of[x].size() > groups_of[y].size(); });
      const int cap = (int)((n + 15) / 16 * 1.03) + 1;
      std::vector<uint8_t> cnt((size_t)ng * 16, 0);
      std::vector<int> csize(16, 0);
      std::vector<int> res(n, 0);
      for (int x : order) {
        int best = -1;
        long cost_best = 1L << 60;
        for (int k = 0; k < 16; k++) {
          if (csize[k] >= cap) continue;
          long cost = 0;
          for (int g : groups_of[x]) cost += cnt[(size_t)g * 16 + k];
          cost = cost * 64 + csize[k] * 64 / cap;  // tie-break towards emptier residues
          if (cost < cost_best) { cost_best = cost; best = k; }
        }
        res[x] = best;
        csize[best]++;
        for (int g : groups_of[x]) cnt[(size_t)g * 16 + best]++;
      }
      // local search on the modelled cost itself: an access group (slice, entry, half warp) takes
      // max(1, max_k members with residue k) wavefronts; move a column to the residue that lowers
      // the sum over its groups the most (capacity permitting), a few passes
      auto col_ls = [&](int passes) {
        std::vector<uint8_t> gmax(ng, 0);
        for (int g = 0; g < ng; g++) {
          uint8_t mx = 0;
          for (int k = 0; k < 16; k++) mx = std::max(mx, cnt[(size_t)g * 16 + k]);
          gmax[g] = mx;
        }
        std::vector<int> mr;  // per group of x: max over residues with x removed
        for (int pass = 0; pass < passes; pass++) {
          long moved = 0;
          for (int x : order) {
            const int r = res[x];
            const auto& G = groups_of[x];
            if (G.empty()) continue;
            mr.resize(G.size());
            long cur = 0;
            for (size_t q = 0; q < G.size(); q++) {
              const uint8_t* c = &cnt[(size_t)G[q] * 16];
              int mx = 0;
              for (int k = 0; k < 16; k++) mx = std::max(mx, (int)c[k] - (k == r ? 1 : 0));
              mr[q] = mx;
              cur += std::max(1, (int)gmax[G[q]]);
            }
            int best = r;
            long best_cost = cur;
            for (int k = 0; k < 16; k++) {
              if (k == r || csize[k] >= cap) continue;
              long cost = 0;
              for (size_t q = 0; q < G.size(); q++) cost += std::max(1, std::max(mr[q], (int)cnt[(size_t)G[q] * 16 + k] + 1));
              if (cost < best_cost) { best_cost = cost; best = k; }
            }
            if (best == r) continue;
            for (size_t q = 0; q < G.size(); q++) {
              uint8_t* c = &cnt[(size_t)G[q] * 16];
              c[r]--;
              c[best]++;
              gmax[G[q]] = (uint8_t)std::max(mr[q], (int)c[best]);
            }
            csize[r]--;
            csize[best]++;
            res[x] = best;
            moved++;
          }
          if (moved == 0) break;
        }
      };
      const int cpasses = getenv("POBK_K2_BANKPASS") ? atoi(getenv("POBK_K2_BANKPASS")) : 4;
      col_ls(cpasses);
      if (getenv("POBK_K2_BANKSTATS")) {  // development aid: modelled wavefronts per x~ access
        double& acc_new = bank_stats[0]; double& acc_old = bank_stats[1]; double& acc_n = bank_stats[2];
        std::vector<std::vector<int>> members(ng);
        for (int x = 0; x < n; x++)
          for (int g : groups_of[x]) members[g].push_back(x);
        for (int g = 0; g < ng; g++) {
          if (members[g].empty()) continue;
          int a1[16] = {0}, a0[16] = {0}, m1 = 0, m0 = 0;
          for (int x : members[g]) { m1 = std::max(m1, ++a1[res[x]]); m0 = std::max(m0, ++a0[x & 15]); }
          acc_new += std::max(m1, 1); acc_old += std::max(m0, 1); acc_n += 0.5;  // per half warp
        }
      }
      int mx = 0;
      for (int k = 0; k < 16; k++) mx = std::max(mx, csize[k]);
      np_t[t] = 16 * mx;
      std::vector<int> rank(16, 0);
      std::vector<int> slot_col((size_t)16 * mx, -1);
      for (int x = 0; x < n; x++) {
        const int li = res[x] + 16 * rank[res[x]]++;
        slot_col[li] = gl[x];
      }
      for (int li = 0; li < 16 * mx; li++) {
        if (slot_col[li] >= 0) local[slot_col[li]] = li;
        pmap.push_back(slot_col[li]);  // -1: a hole (x~ = x~* = 0, never accessed)
      }
    }
    pmap_ptr[T] = (int)pmap.size();
    if (bank_stats[2] > 0)
      fprintf(stderr, "[k2 banks] modelled wavefronts per private x~ access: placed %.2f, unplaced %.2f\n",
              bank_stats[0] / bank_stats[2], bank_stats[1] / bank_stats[2]);
  }
  const int np_max = std::max(1, *std::max_element(np_t.begin(), np_t.end()));
  if (np_max > 65535) { why = "private columns per tile exceed the 16-bit interior column index"; return false; }
  const size_t base_smem = fixed + meta_bytes + 8 * (size_t)kR * ((size_t)np_max + 1);  // private x~ + the zero slot
  int NS = (int)std::min<size_t>(kMaxSlots, (kSmemTotal - base_smem) / kSlot);
  if (getenv("POBK_K2_NS_CAP")) NS = std::min(NS, atoi(getenv("POBK_K2_NS_CAP")));  // development experiments
  if (NS < kMinSlots) { why = "shared memory too small for the TMA ring"; return false; }
  // slice meta .y = offset in chunk (< 2^16) | (tile-local chunk index mod 2NS) << 16
  for (auto& sm : smeta) sm.y |= ((sm.x & 0xfffff) % (2 * NS)) << 16;

  // the version chain of every shared column c: the rows touching c in schedule (step) order; the
  // value written by the p-th goes to the (p+1)-th's mailbox slot, the last one's (kWrap) to the
  // first one's slot of the next sweep and to x~.  mout[row entry] = target slot.
  std::vector<unsigned> mout_of_entry(At.nnz(), 0u);
  std::vector<int> seed_idx, seed_col;
  std::vector<int> lastcol_ptr(T + 1, 0), lastcol, lastslot;
  {
    std::vector<int64_t> cptr(m + 1, 0);
    for (int64_t q = 0; q < At.nnz(); q++) cptr[At.col[q] + 1]++;
    for (int64_t c = 0; c < m; c++) cptr[c + 1] += cptr[c];
    std::vector<int64_t> ent(At.nnz());  // entries (CSR positions) of each column
    {
      std::vector<int64_t> fill(cptr.begin(), cptr.end() - 1);
      for (int64_t i = 0; i < m; i++)
        for (int64_t q = At.ptr[i]; q < At.ptr[i + 1]; q++) ent[fill[At.col[q]]++] = q;
    }
    std::vector<int32_t> row_of_entry(At.nnz());
    for (int64_t i = 0; i < m; i++)
      for (int64_t q = At.ptr[i]; q < At.ptr[i + 1]; q++) row_of_entry[q] = (int32_t)i;
    auto slot_of = [&](int64_t q) -> int64_t {  // mailbox slot of CSR entry q (its row is a boundary row)
      const int32_t i = row_of_entry[q];
      const int64_t j = q - At.ptr[i];
      return mb_of_row[i] + j;
    };
    std::vector<std::vector<std::pair<int, int>>> per(T);
    std::vector<int64_t> ch;
    for (int64_t c = 0; c < m; c++) {
      if (!shared[c]) continue;
      ch.assign(ent.begin() + cptr[c], ent.begin() + cptr[c + 1]);
      std::sort(ch.begin(), ch.end(), [&](int64_t x, int64_t y) { return step_of[row_of_entry[x]] < step_of[row_of_entry[y]]; });
      for (size_t pidx = 0; pidx < ch.size(); pidx++) {
        const bool last = pidx + 1 == ch.size();
        const int64_t tgt = slot_of(ch[last ? 0 : pidx + 1]);
        mout_of_entry[ch[pidx]] = (unsigned)tgt | (last ? kWrap : 0u);
      }
      seed_idx.push_back((int)slot_of(ch[0]));
      seed_col.push_back((int)c);
      per[tile[row_of_entry[ch.back()]]].push_back({(int)c, (int)slot_of(ch[0])});
    }
    for (int t = 0; t < T; t++) {
      lastcol_ptr[t + 1] = lastcol_ptr[t] + (int)per[t].size();
      for (auto& pr : per[t]) { lastcol.push_back(pr.first); lastslot.push_back(pr.second); }
    }
  }

  // the stream: slices in tile, task, kind order; ELL inside a slice
  std::vector<unsigned char> stream(off, 0);
  std::vector<int32_t> orig_q;
  std::vector<int64_t> fslot;
  orig_q.reserve(m);
  fslot.reserve(m);
  for (size_t si = 0; si < slice_rows.size(); si++) {
    const auto& rows = slice_rows[si];
    const int R = (int)rows.size(), W = smeta[si].z;
    const bool bnd = slice_bnd[si];
    unsigned char* blk = stream.data() + slice_pos[si];
    const SliceLayout L(R, W, bnd, kR);
    double* val = (double*)blk;
    double* fv = (double*)(blk + L.o_f);
    unsigned* col = (unsigned*)(blk + L.o_col);             // boundary slices
    unsigned short* col16 = (unsigned short*)(blk + L.o_col);  // interior slices
    unsigned* mout = (unsigned*)(blk + L.o_mout);
    unsigned short* len = (unsigned short*)(blk + L.o_len);
    for (int r = 0; r < R; r++) {
      const int32_t i = rows[r];
      for (int j = 0; j < rlen(i); j++) {
        const int64_t q = At.ptr[i] + j;
        const int32_t cg = At.col[q];
        if (bnd) col[j * R + r] = shared[cg] ? (kShared | (unsigned)cg) : (unsigned)local[cg];
        else col16[j * R + r] = (unsigned short)local[cg];
        val[j * R + r] = At.val[q];
        if (bnd) mout[j * R + r] = shared[cg] ? mout_of_entry[q] : 0u;
      }
      for (int j = rlen(i); j < W; j++) {  // ELL padding: zero slot, value +0
        if (bnd) col[j * R + r] = (unsigned)np_max;
        else col16[j * R + r] = (unsigned short)np_max;
      }
      if (bnd) ((double*)(blk + L.o_n2))[r] = nrm2[i];  // ||a~_i||^2 (row_sqnorms: the oracle's O1 order)
      len[r] = (unsigned short)rlen(i);
      for (int q = 0; q < kR; q++) fv[kR * r + q] = 0.0;  // f~ is scattered in per solve (k2_scatter_f)
      orig_q.push_back(p.perm[i]);
      fslot.push_back((slice_pos[si] + L.o_f) / 8 + (int64_t)kR * r);
    }
  }
  // Bounds check of the finished layout (every index the kernel will dereference), before upload:
  // slices inside their chunk, chunks inside a ring slot, private columns inside the tile's x~
  // window (or the zero slot), shared columns < m, mailbox targets (both parities) < NB, row
  // lengths <= slice width, every row streamed exactly once.  (compute-sanitizer is closed on the
  // GPU pool: DESIGN.md §9.)
  {
    auto bad = [&](const std::string& w) { why = "K2 layout check failed: " + w; return false; };
    std::vector<uint8_t> seen(m, 0);
    for (int t = 0; t < T; t++) {
      for (int ci = tile_chunk[t]; ci < tile_chunk[t + 1]; ci++)
        if (cmeta[ci].y > kSlot || cmeta[ci].y <= 0) return bad("chunk size " + std::to_string(cmeta[ci].y));
      for (int si = tile_slice[t]; si < tile_slice[t + 1]; si++) {
        const int4 sm = smeta[si];
        const int chunk = sm.x & 0xfffff, R = sm.x >> 20, W = sm.z;
        const int off_in = sm.y & 0xffff;
        if (tile_chunk[t] + chunk >= tile_chunk[t + 1]) return bad("slice chunk index");
        const int bytes = SliceLayout(R, W, slice_bnd[si], kR).bytes;
        if (off_in + bytes > cmeta[tile_chunk[t] + chunk].y) return bad("slice outside its chunk");
        if (R < 1 || R > kSliceRows) return bad("slice rows");
        const unsigned char* blk = stream.data() + slice_pos[si];
        const SliceLayout L(R, W, slice_bnd[si], kR);
        const unsigned* col = (const unsigned*)(blk + L.o_col);
        const unsigned short* col16 = (const unsigned short*)(blk + L.o_col);
        const unsigned* mout = (const unsigned*)(blk + L.o_mout);
        const unsigned short* len = (const unsigned short*)(blk + L.o_len);
        for (int r = 0; r < R; r++) {
          const int32_t i = slice_rows[si][r];
          if (seen[i]++) return bad("row " + std::to_string(i) + " streamed twice");
          if (len[r] > W) return bad("row length > slice width");
          for (int j = 0; j < W; j++) {
            const unsigned c = slice_bnd[si] ? col[j * R + r] : (unsigned)col16[j * R + r];
            if (c & kShared) {
              if ((c & kIdx) >= (unsigned)m || !slice_bnd[si]) return bad("shared column");
              const unsigned mo = mout[j * R + r] & ~kWrap;
              if ((long long)mo >= NB) return bad("mailbox target >= NB");
            } else if (c > (unsigned)np_max || (c < (unsigned)np_max && (int)c >= np_t[t])) {
              return bad("private column outside the tile's window");
            }
          }
        }
      }
    }
    for (int64_t i = 0; i < m; i++)
      if (!seen[i]) return bad("row " + std::to_string(i) + " never streamed");
  }
  if (kR == 1) p.tile_of_row.assign(tile.begin(), tile.end());

  // upload
  K2Plan* k = new K2Plan();
  (kR == 1 ? p.k2 : p.k2r) = k;
  k->kR = kR;
  k->T = T;
  k->NS = NS;
  // CTA size: each compute warp takes about one slice per task with 7 warps when tasks are small
  // (register-resident boundary slices, 256 threads); tasks of many slices (config 5: ~16) need
  // the 15 compute warps of the 512-thread instantiation (measured: 84.6 vs 70.5 us/sweep)
  k->nt = kR == 1 ? nt_choice : 256;  // (two-RHS plans: 256 threads, BSliceR2)
  k->nsl_max = nsl_max;
  k->nck_max = nck_max;
  k->ntask_max = ntask_max;
  k->np_max = np_max;
  k->smem = (size_t)NS * kSlot + base_smem;
  k->NB = NB;
  k->npmap = (int)pmap.size();
  k->nlast = (int)lastcol.size();
  k->nseed = (int)seed_idx.size();
  std::vector<long long> tile_off(T, 0);
  {
    int ci = 0;
    long long pos = 0;
    for (int t = 0; t < T; t++) {
      tile_off[t] = pos;
      for (; ci < tile_chunk[t + 1]; ci++) pos += cmeta[ci].y;
    }
  }
  k->private_frac = p.nnz ? (double)n_private_nnz / (double)p.nnz : 0.0;
  k->interior_frac = (double)n_interior / (double)m;
  k->stream_bytes = off;
  k->pad_entries = pad;
  k->nchunks = (int)cmeta.size();
  k->ntask_total = (int)tmeta.size();
  cudaError_t e = cudaSuccess;
#define K2_UP(dst, src, n) \
  if (e == cudaSuccess) e = k2_upload(*k, dst, src, n)
  K2_UP(&k->stream, stream.data(), stream.size());
  K2_UP(&k->tile_off, tile_off.data(), tile_off.size());
  K2_UP(&k->smeta, smeta.data(), smeta.size());
  K2_UP(&k->cmeta, cmeta.data(), cmeta.size());
  K2_UP(&k->tmeta, tmeta.data(), tmeta.size());
  K2_UP(&k->tile_slice, tile_slice.data(), tile_slice.size());
  K2_UP(&k->tile_chunk, tile_chunk.data(), tile_chunk.size());
  K2_UP(&k->tile_task, tile_task.data(), tile_task.size());
  K2_UP(&k->pmap_ptr, pmap_ptr.data(), pmap_ptr.size());
  K2_UP(&k->pmap, pmap.data(), pmap.size());
  K2_UP(&k->lastcol_ptr, lastcol_ptr.data(), lastcol_ptr.size());
  K2_UP(&k->lastcol, lastcol.data(), lastcol.size());
  K2_UP(&k->lastslot, lastslot.data(), lastslot.size());
  K2_UP(&k->seed_idx, seed_idx.data(), seed_idx.size());
  K2_UP(&k->seed_col, seed_col.data(), seed_col.size());
  K2_UP(&k->mbox, (unsigned long long*)nullptr, 2 * (size_t)kR * std::max<long long>(NB, 1));
  K2_UP(&k->xsp, (double*)nullptr, pmap.size());
  K2_UP(&k->lcx, (double*)nullptr, lastcol.size());
  if (kR == 2) {
    K2_UP(&k->xsp1, (double*)nullptr, pmap.size());
    K2_UP(&k->lcx1, (double*)nullptr, lastcol.size());
    for (int q = 0; q < 2; q++) {
      K2_UP(&k->xt2[q], (double*)nullptr, (size_t)m);
      K2_UP(&k->xst2[q], (double*)nullptr, (size_t)m);
    }
    K2_UP(&k->ctrl2, (Ctrl*)nullptr, 2);
    if (e == cudaSuccess) e = cudaMallocHost(&k->h_ctrl2, 2 * sizeof(Ctrl));
    for (auto& ev : k->ev)
      if (e == cudaSuccess) e = cudaEventCreate(&ev);
  }
  K2_UP(&k->orig_q, orig_q.data(), orig_q.size());
  K2_UP(&k->fslot, fslot.data(), fslot.size());
  K2_UP(&k->sync, (SyncState*)nullptr, 1);
  K2_UP(&k->partials, (double*)nullptr, 2 * (size_t)kR * T);
#undef K2_UP
  if (e != cudaSuccess) {
    why = std::string("device upload failed: ") + cudaGetErrorString(e);
    if (kR == 1) k2_free(p);
    else k2r_free(p);
    return false;
  }
  if (kR == 1) p.ntiles = T;
  return true;
}

namespace {
// the sweep kernel for a plan shape: threads per CTA, vector-slice width, interior mode
const void* k2_kernel(int nt, int kR) {
  if (kR == 2) return (const void*)k2_sweeps<256, false, 2>;
  return nt == 512 ? (const void*)k2_sweeps<512, false, 1> : (const void*)k2_sweeps<256, true, 1>;
}
}  // namespace

cudaError_t k2_solve(Plan& p, const double* f_user, cudaStream_t s, long long& launches) {
  K2Plan& k = *p.k2;
  cudaError_t e;
  k2_scatter_f<<<(int)std::min<int64_t>((p.m + 255) / 256, 148 * 8), 256, 0, s>>>(p.m, k.orig_q, k.fslot, f_user,
                                                                                  (double*)k.stream);
  k2_reset<<<1, 1, 0, s>>>(k.sync);
  k2_mbox_fill<<<148 * 4, 256, 0, s>>>(k.mbox, 2 * std::max<long long>(k.NB, 1));
  k2_mbox_seed<<<std::max(1, std::min(148 * 4, (k.nseed + 255) / 256)), 256, 0, s>>>(k.mbox, k.nseed, k.seed_idx, k.seed_col,
                                                                                      p.d_xt, 1, 0);
  launches += 4;
  if (p.d_xst && k.npmap + k.nlast > 0) {
    k2_gather_xs<<<std::max(1, std::min(148 * 4, (k.npmap + k.nlast + 255) / 256)), 256, 0, s>>>(
        k.npmap, k.pmap, k.nlast, k.lastcol, p.d_xst, k.xsp, k.lcx);
    launches++;
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  K2Args a;
  a.stream = k.stream;
  a.tile_off = k.tile_off;
  a.smeta = k.smeta;
  a.tile_slice = k.tile_slice;
  a.cmeta = k.cmeta;
  a.tile_chunk = k.tile_chunk;
  a.tmeta = k.tmeta;
  a.tile_task = k.tile_task;
  a.pmap_ptr = k.pmap_ptr;
  a.pmap = k.pmap;
  a.lastcol_ptr = k.lastcol_ptr;
  a.lastcol = k.lastcol;
  a.lastslot = k.lastslot;
  a.mbox = k.mbox;
  a.NB = k.NB;
  a.xg = p.d_xt;
  a.xst = p.d_xst;
  a.xsp = k.xsp;
  a.lcx = k.lcx;
  a.xg1 = nullptr;
  a.xsp1 = nullptr;
  a.lcx1 = nullptr;
  a.ctrl1 = nullptr;
  a.sync = k.sync;
  a.partials = k.partials;
  a.ctrl = p.d_ctrl;
  a.T = k.T;
  a.NS = k.NS;
  a.nsl_max = k.nsl_max;
  a.nck_max = k.nck_max;
  a.ntask_max = k.ntask_max;
  a.np_max = k.np_max;
  a.trace = nullptr;
  a.trace_sweep = -1;
  static const char* trace_env = POBK_K2_DEV ? getenv("POBK_K2_TRACE") : nullptr;  // (development builds)
  if (trace_env) {
    const size_t n = (size_t)k.T * k.ntask_max * 12;
    if (!k.trace) cudaMalloc(&k.trace, n * sizeof(unsigned long long));
    cudaMemsetAsync(k.trace, 0, n * sizeof(unsigned long long), s);
    a.trace = k.trace;
    a.trace_sweep = atoi(trace_env);
  }
  void* args[] = {&a};
  const void* fn = k2_kernel(k.nt, 1);
  if ((e = raise_smem_limit(fn)) != cudaSuccess) return e;
  e = cudaLaunchCooperativeKernel(fn, dim3(k.T), dim3(k.nt), args, k.smem, s);
  launches++;
  if (e == cudaSuccess && a.trace) {  // development aid: raw stamps + the task table for tools/k2_trace.py
    const size_t n = (size_t)k.T * k.ntask_max * 12;
    std::vector<unsigned long long> h(n);
    cudaStreamSynchronize(s);
    cudaMemcpy(h.data(), a.trace, n * 8, cudaMemcpyDeviceToHost);
    std::vector<int4> tm(k.ntask_total);
    std::vector<int> tt(k.T + 1);
    cudaMemcpy(tm.data(), k.tmeta, tm.size() * sizeof(int4), cudaMemcpyDeviceToHost);
    cudaMemcpy(tt.data(), k.tile_task, tt.size() * sizeof(int), cudaMemcpyDeviceToHost);
    const char* path = getenv("POBK_K2_TRACE_OUT") ? getenv("POBK_K2_TRACE_OUT") : "k2_trace.bin";
    FILE* fp = fopen(path, "wb");
    if (fp) {
      int hdr[4] = {k.T, k.ntask_max, 12, k.ntask_total};
      fwrite(hdr, sizeof(hdr), 1, fp);
      fwrite(h.data(), 8, n, fp);
      fwrite(tm.data(), sizeof(int4), tm.size(), fp);
      fwrite(tt.data(), sizeof(int), tt.size(), fp);
      fclose(fp);
    }
  }
  return e;
}

void k2_free(Plan& p) {
  if (!p.k2) return;
  for (void* v : p.k2->allocs) cudaFree(v);
  if (p.k2->trace) cudaFree(p.k2->trace);
  delete p.k2;
  p.k2 = nullptr;
}

void k2r_free(Plan& p) {
  if (!p.k2r) return;
  for (void* v : p.k2r->allocs) cudaFree(v);
  if (p.k2r->h_ctrl2) cudaFreeHost(p.k2r->h_ctrl2);
  for (auto& ev : p.k2r->ev)
    if (ev) cudaEventDestroy(ev);
  delete p.k2r;
  p.k2r = nullptr;
}

// The two-RHS plan (built on the first pobk_solve_multi call with R = 2 on a K2 plan): A~ in RCM
// row order, rebuilt from the plan's device copy (storage row q is RCM row sched.rows[q]), then
// the K2 layout with pair-interleaved x~, mailboxes and f~.
bool k2r_build(Plan& p, std::string& why) {
  const int64_t m = p.m, nnz = p.nnz;
  std::vector<int32_t> rp(m + 1), col(nnz);
  std::vector<double> val(nnz), n2s(m);
  cudaError_t e = cudaMemcpy(rp.data(), p.A.rp, (m + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(col.data(), p.A.col, nnz * sizeof(int32_t), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(val.data(), p.A.val, nnz * sizeof(double), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(n2s.data(), p.A.nrm2, m * sizeof(double), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    why = std::string("device copy failed: ") + cudaGetErrorString(e);
    return false;
  }
  std::vector<int64_t> pos(m);
  for (int64_t q = 0; q < m; q++) pos[p.sched.rows[q]] = q;
  HostCSR At;
  At.m = m;
  At.ptr.assign(m + 1, 0);
  At.col.resize(nnz);
  At.val.resize(nnz);
  std::vector<double> nrm2(m);
  for (int64_t i = 0; i < m; i++) {
    const int64_t q = pos[i], b = rp[q], len = rp[q + 1] - rp[q];
    At.ptr[i + 1] = At.ptr[i] + len;
    std::copy(col.begin() + b, col.begin() + b + len, At.col.begin() + At.ptr[i]);
    std::copy(val.begin() + b, val.begin() + b + len, At.val.begin() + At.ptr[i]);
    nrm2[i] = n2s[q];
  }
  return k2_build(p, At, nrm2, p.k2_tile_rows, why, 2);
}

// Two right-hand sides in one K2 launch: A~ streamed once per sweep for both; each stops on its
// own rule and is then frozen; iterates bitwise those of the single solves.
cudaError_t k2r_solve(Plan& p, const double* const* f, double* const* x, const double* const* xstar,
                      const pobk_solve_opts& o, cudaStream_t s, pobk_report* reps) {
  K2Plan& k = *p.k2r;
  cudaError_t e;
  long long launches = 0;
  const bool rse = o.stop == POBK_STOP_RSE;
  const long long ncall = o.max_sweeps - o.sweep_offset;
  for (int q = 0; q < 2; q++) {
    Ctrl& c = k.h_ctrl2[q];
    c.sweeps = 0;
    c.max_sweeps = ncall;
    c.offset = o.sweep_offset;
    c.tol = o.tol;
    c.value = NAN;
    c.den = 0.0;
    c.stop_mode = o.stop;
    c.check_every = o.check_every;
    c.stopped = ncall <= 0 ? 1 : 0;
    c.term = POBK_TERM_MAX_SWEEPS;
    c.arrive = 0;
    c.pad = 0;
  }
  if ((e = cudaEventRecord(k.ev[0], s)) != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(k.ctrl2, k.h_ctrl2, 2 * sizeof(Ctrl), cudaMemcpyHostToDevice, s)) != cudaSuccess) return e;
  for (int q = 0; q < 2; q++) {
    if ((e = launch_permute_in(p, nullptr, x[q], rse ? xstar[q] : nullptr, nullptr, k.xt2[q], k.xst2[q], s, launches)) !=
        cudaSuccess)
      return e;
    if (rse && (e = launch_den(p, k.ctrl2 + q, k.xst2[q], s, launches)) != cudaSuccess) return e;
  }
  const int gf = (int)std::min<int64_t>((p.m + 255) / 256, 148 * 8);
  for (int q = 0; q < 2; q++) k2_scatter_f<<<gf, 256, 0, s>>>(p.m, k.orig_q, k.fslot, f[q], (double*)k.stream + q);
  k2_reset<<<1, 1, 0, s>>>(k.sync);
  k2_mbox_fill<<<148 * 4, 256, 0, s>>>(k.mbox, 4 * std::max<long long>(k.NB, 1));
  for (int q = 0; q < 2; q++)
    k2_mbox_seed<<<std::max(1, std::min(148 * 4, (k.nseed + 255) / 256)), 256, 0, s>>>(k.mbox, k.nseed, k.seed_idx,
                                                                                        k.seed_col, k.xt2[q], 2, q);
  launches += 6;
  if (rse && k.npmap + k.nlast > 0) {
    const int gb = std::max(1, std::min(148 * 4, (k.npmap + k.nlast + 255) / 256));
    k2_gather_xs<<<gb, 256, 0, s>>>(k.npmap, k.pmap, k.nlast, k.lastcol, k.xst2[0], k.xsp, k.lcx);
    k2_gather_xs<<<gb, 256, 0, s>>>(k.npmap, k.pmap, k.nlast, k.lastcol, k.xst2[1], k.xsp1, k.lcx1);
    launches += 2;
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = cudaEventRecord(k.ev[1], s)) != cudaSuccess) return e;
  if (ncall > 0) {
    K2Args a;
    a.stream = k.stream;
    a.tile_off = k.tile_off;
    a.smeta = k.smeta;
    a.tile_slice = k.tile_slice;
    a.cmeta = k.cmeta;
    a.tile_chunk = k.tile_chunk;
    a.tmeta = k.tmeta;
    a.tile_task = k.tile_task;
    a.pmap_ptr = k.pmap_ptr;
    a.pmap = k.pmap;
    a.lastcol_ptr = k.lastcol_ptr;
    a.lastcol = k.lastcol;
    a.lastslot = k.lastslot;
    a.mbox = k.mbox;
    a.NB = k.NB;
    a.xg = k.xt2[0];
    a.xst = k.xst2[0];
    a.xsp = k.xsp;
    a.lcx = k.lcx;
    a.xg1 = k.xt2[1];
    a.xsp1 = k.xsp1;
    a.lcx1 = k.lcx1;
    a.ctrl1 = k.ctrl2 + 1;
    a.sync = k.sync;
    a.partials = k.partials;
    a.ctrl = k.ctrl2;
    a.T = k.T;
    a.NS = k.NS;
    a.nsl_max = k.nsl_max;
    a.nck_max = k.nck_max;
    a.ntask_max = k.ntask_max;
    a.np_max = k.np_max;
    a.trace = nullptr;
    a.trace_sweep = -1;
    void* args[] = {&a};
    const void* fn = k2_kernel(k.nt, 2);
    if ((e = raise_smem_limit(fn)) != cudaSuccess) return e;
    if ((e = cudaLaunchCooperativeKernel(fn, dim3(k.T), dim3(k.nt), args, k.smem, s)) != cudaSuccess) return e;
    launches++;
  }
  if ((e = cudaEventRecord(k.ev[2], s)) != cudaSuccess) return e;
  for (int q = 0; q < 2; q++)
    if ((e = launch_permute_out_from(p, k.xt2[q], x[q], s, launches)) != cudaSuccess) return e;
  if ((e = cudaEventRecord(k.ev[3], s)) != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(k.h_ctrl2, k.ctrl2, 2 * sizeof(Ctrl), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  float t_all = 0.f, t_sw = 0.f;
  cudaEventElapsedTime(&t_all, k.ev[0], k.ev[3]);
  cudaEventElapsedTime(&t_sw, k.ev[1], k.ev[2]);
  for (int q = 0; q < 2 && reps; q++) {
    const Ctrl& c = k.h_ctrl2[q];
    pobk_report& rp = reps[q];
    rp.sweeps = c.sweeps;
    rp.termination = c.term;
    rp.kernel = POBK_KERNEL_WAVEFRONT;
    rp.final_value = o.stop == POBK_STOP_NONE ? NAN : c.value;
    rp.solve_seconds = t_all * 1e-3;
    rp.sweep_seconds = t_sw * 1e-3;
    rp.launches = launches;
    rp.sweeps_total = o.sweep_offset + c.sweeps;
    rp.final_rse = rse ? c.value : NAN;
    rp.final_relres = NAN;
  }
  return cudaSuccess;
}

// RELRES runs inside K2 on one-lane layouts (the residual pass reads slices in that layout)
bool k2_relres_ok(const Plan& p) { return p.k2 != nullptr; }

bool k2_stats(const Plan& p, K2Stats& st) {
  if (!p.k2) return false;
  st.T = p.k2->T;
  st.private_frac = p.k2->private_frac;
  st.interior_frac = p.k2->interior_frac;
  st.stream_bytes = p.k2->stream_bytes;
  st.nchunks = p.k2->nchunks;
  st.threads = p.k2->nt;
  return true;
}

}  // namespace pobk
