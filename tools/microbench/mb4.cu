// L2-hit latency of a batch of 8 independent fp64 gathers (ld.global.cg) from an 8 MB vector,
// alone and while the other SMs stream HBM (development aid for K2's boundary path).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void k(const double* x, int n, const double2* big, size_t nbig, int stream, long long* out, volatile int* done) {
  if (blockIdx.x == 0) {
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    unsigned h = 12345u + lane * 7919u;
    long long best = 1LL << 60, sum = 0;
    double acc = 0;
    for (int it = 0; it < 2000; it++) {
      int idx[8];
      for (int u = 0; u < 8; u++) { h = h * 1664525u + 1013904223u; idx[u] = (h >> 8) % n; }
      __syncwarp();
      long long t0 = clock64();
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; u++) v[u] = __ldcg(x + idx[u]);
      double s = 0;
#pragma unroll
      for (int u = 0; u < 8; u++) s += v[u];
      acc += s;
      __syncwarp();
      long long t1 = clock64() - t0;
      if (t1 < best) best = t1;
      sum += t1;
    }
    if (lane == 0) { out[0] = best; out[1] = sum / 2000; out[2] = (long long)acc; *done = 1; }
    return;
  }
  if (!stream) return;
  double s = 0;
  size_t i = (blockIdx.x - 1) * (size_t)blockDim.x + threadIdx.x;
  while (!*done) {
    double2 v = __ldcs(big + i);
    s += v.x;
    i += (size_t)(gridDim.x - 1) * blockDim.x;
    if (i >= nbig) i -= nbig;
  }
  if (s == 1.2345) out[3] = 1;
}

int main() {
  const int n = 1 << 20;
  double* x; double2* big; long long* out; int* done;
  const size_t nbig = (size_t)1 << 27;  // 4 GB
  CK(cudaMalloc(&x, n * 8)); CK(cudaMalloc(&big, nbig * 16)); CK(cudaMalloc(&out, 64)); CK(cudaMalloc(&done, 4));
  CK(cudaMemset(x, 0, n * 8)); CK(cudaMemset(big, 0, nbig * 16));
  for (int stream = 0; stream < 2; stream++) {
    CK(cudaMemset(done, 0, 4));
    k<<<148, 512>>>(x, n, big, nbig, stream, out, done);
    CK(cudaDeviceSynchronize());
    long long h[3]; CK(cudaMemcpy(h, out, 24, cudaMemcpyDeviceToHost));
    printf("%s: 8 gathers + sum: best %lld cycles, mean %lld cycles\n", stream ? "with HBM streaming" : "idle", h[0], h[1]);
  }
  return 0;
}
