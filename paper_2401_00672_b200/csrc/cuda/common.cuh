// Device helpers shared by the sweep kernels (K1, K2, K3) and the check kernels.
//
// THE PER-ROW ARITHMETIC CONTRACT.  Every sweep kernel computes a row's
// projection (Eq 1.2) with exactly these operations, so all kernel families
// produce bitwise-identical iterates for thr = 0:
//   lane l (0 <= l < V) of the row's V-lane vector:  acc_l = 0; for p = p0+l, p0+l+V, ... < p1:
//                                                     acc_l = fma(a_p, x_{col p}, acc_l)
//   xor-butterfly over the V lanes (offsets V/2, ..., 1): acc += shfl_xor(acc, o)
//   alpha = (f_i - acc) / nrm2_i                       (division, as in Eq 1.2)
//   x_{col p} = fma(alpha, a_p, x_{col p})            (for the lane's own entries)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pobk {

template <int V>
__device__ __forceinline__ double vec_sum(double v) {
#pragma unroll
  for (int o = V / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, V);
  return v;
}

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
