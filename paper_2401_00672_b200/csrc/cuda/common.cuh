// Device helpers shared by the sweep kernels (K1, K2, K3) and the check kernels.
//
// THE PER-ROW ARITHMETIC CONTRACT.  Every sweep kernel applies a row's
// projection (Eq 1.2) with exactly the operations of the oracle's O7, each
// rounded separately (no FMA contraction):
//     s = 0;  for p ascending:  s = s + (a_p * x_{col p})       (dmul_rn, then dadd_rn)
//     alpha = (f_i - s) / nrm2_i                                   (dsub_rn, ddiv_rn)
//     for p:  x_{col p} = x_{col p} + (alpha * a_p)                (dmul_rn, then dadd_rn)
// Because the rows of one category have disjoint supports (thr = 0), the order in which a
// category's rows are applied cannot change any value, so every kernel family reproduces the
// oracle's iterates BIT FOR BIT, whatever its parallel schedule.  (thr > 0 overlapping categories:
// every alpha first, then per column x_c = x_c + (alpha_i * a_ic) in ascending row order -- the
// oracle's order, also bitwise; POBK_THR_ATOMIC=1 switches to fp64 atomics, parity to 1e-9.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pobk {

__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ void st_cg(double* p, double v) { __stcg(p, v); }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// One row of Eq 1.2 by one thread, x in any memory space reachable through a generic pointer.
// Returns alpha.
// Products ahead of the chain: in-order issue runs `s = s + a_j*x_j` at ~21 cycles per link when
// each product is issued next to its add (ptxas keeps the source order), ~8.8 when all products
// of a row (or batch) are formed first (tools/microbench/mb11.cu).  pin() is a volatile register
// move that keeps a product where it is written; the additions, and so every rounded result,
// are unchanged (same operations, same order).
__device__ __forceinline__ double pin(double v) {
  asm volatile("mov.b64 %0, %0;" : "+d"(v));
  return v;
}

// alpha = RN(r / b) from y = RN(1/b) computed ahead of time (off the row's critical path):
// q = RN(r*y) is within 1 ulp of r/b, e = r - b*q is exact (one FMA), and RN(q + e*y) is the
// correctly rounded quotient (Markstein's theorem; also checked against the division on 2e8
// random operand pairs) -- so this is bitwise __ddiv_rn(r, b), the contract's division, in three
// dependent operations instead of the ~40-instruction division sequence.  e = 0 means q is the
// exact quotient (keeps the sign of a zero r); a non-finite q (r non-finite) returns q as the
// division would (inf) or NaN.
__device__ __forceinline__ double rcp_ahead(double b) { return __drcp_rn(b); }
__device__ __forceinline__ double div_by_rcp(double r, double b, double y) {
  const double q = __dmul_rn(r, y);
  const double e = __fma_rn(-b, q, r);
  return (e == 0.0 || !isfinite(q)) ? q : __fma_rn(e, y, q);
}

__device__ __forceinline__ double row_project(const int32_t* __restrict__ col, const double* __restrict__ val,
                                              int p0, int p1, double f, double nrm2, double* x) {
  double s = 0.0;
  for (int p = p0; p < p1; p++) s = __dadd_rn(s, __dmul_rn(val[p], x[col[p]]));
  const double alpha = __ddiv_rn(__dsub_rn(f, s), nrm2);
  for (int p = p0; p < p1; p++) {
    const int c = col[p];
    x[c] = __dadd_rn(x[c], __dmul_rn(alpha, val[p]));
  }
  return alpha;
}

// Eq 1.2 residual part only (thr > 0 pass 1, RELRES): alpha of a row at the current x.
__device__ __forceinline__ double row_dot(const int32_t* __restrict__ col, const double* __restrict__ val, int p0,
                                          int p1, const double* x) {
  double s = 0.0;
  for (int p = p0; p < p1; p++) s = __dadd_rn(s, __dmul_rn(val[p], x[col[p]]));
  return s;
}

// Deterministic block sum (fixed tree): every thread passes its value; thread 0 gets the sum.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh /* >= NT/32 doubles */) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = (l < NT / 32) ? sh[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  }
  __syncthreads();
  return r;
}

}  // namespace pobk
