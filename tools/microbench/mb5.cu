// Issue cost of 24 scattered fp64 stores per lane by one warp: st.relaxed.gpu vs st.global.cg vs
// st.global (weak), and the latency of a batch of 24 relaxed.gpu loads (development aid).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int MODE>
__global__ void k(unsigned long long* buf, int n, long long* out) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  long long best = 1LL << 60;
  unsigned h = 777u + lane * 131u;
  for (int it = 0; it < 200; it++) {
    unsigned idx[24];
    for (int j = 0; j < 24; j++) { h = h * 1664525u + 1013904223u; idx[j] = (h >> 6) % n; }
    __syncwarp();
    long long t0 = clock64();
    unsigned long long acc = 0;
#pragma unroll
    for (int j = 0; j < 24; j++) {
      unsigned long long* p = buf + idx[j];
      unsigned long long v = (unsigned long long)it * 31 + j;
      if (MODE == 0) asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
      if (MODE == 1) asm volatile("st.global.cg.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
      if (MODE == 2) asm volatile("st.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
      if (MODE == 3) { unsigned long long w; asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory"); acc += w; }
      if (MODE == 4) { unsigned long long w; asm volatile("ld.global.cg.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory"); acc += w; }
    }
    if (MODE >= 3 && acc == 12345) buf[0] = acc;
    __syncwarp();
    long long t1 = clock64() - t0;
    if (t1 < best) best = t1;
  }
  if (lane == 0) out[MODE] = best;
}

int main() {
  unsigned long long* buf; long long* out;
  const int n = 1 << 20;
  CK(cudaMalloc(&buf, n * 8)); CK(cudaMalloc(&out, 64)); CK(cudaMemset(buf, 0, n * 8));
  k<0><<<1, 32>>>(buf, n, out); k<1><<<1, 32>>>(buf, n, out); k<2><<<1, 32>>>(buf, n, out);
  k<3><<<1, 32>>>(buf, n, out); k<4><<<1, 32>>>(buf, n, out);
  CK(cudaDeviceSynchronize());
  long long h[5]; CK(cudaMemcpy(h, out, 40, cudaMemcpyDeviceToHost));
  printf("24 scattered stores/lane: relaxed.gpu %lld cyc, .cg %lld cyc, weak %lld cyc\n", h[0], h[1], h[2]);
  printf("24 scattered loads/lane (+sum): relaxed.gpu %lld cyc, .cg %lld cyc\n", h[3], h[4]);
  return 0;
}
