// Dependent fp64 chains on sm_100a (development aid): cycles per link of s = s + a_j * x_j
// (__dadd_rn(__dmul_rn)), of a plain __dadd_rn chain, and of __ddiv_rn, one warp alone.
#include <cstdio>
__global__ void mb10(const double* in, double* out, long long* cyc) {
  double a[24], x[24];
  for (int j = 0; j < 24; j++) { a[j] = in[j + threadIdx.x]; x[j] = in[j + 24 + threadIdx.x]; }
  double s = 0.0;
  long long t0 = clock64();
#pragma unroll
  for (int j = 0; j < 24; j++) s = __dadd_rn(s, __dmul_rn(a[j], x[j]));
  asm volatile("mov.b64 %0, %0;" : "+d"(s));
  long long t1 = clock64();
  double u = s;
#pragma unroll
  for (int j = 0; j < 24; j++) u = __dadd_rn(u, a[j]);
  asm volatile("mov.b64 %0, %0;" : "+d"(u));
  long long t2 = clock64();
  double d = __ddiv_rn(u, s + 3.0);
  asm volatile("mov.b64 %0, %0;" : "+d"(d));
  long long t3 = clock64();
  double v = d;
#pragma unroll
  for (int j = 0; j < 24; j++) v = fma(a[j], x[j], v);
  asm volatile("mov.b64 %0, %0;" : "+d"(v));
  long long t4 = clock64();
  out[threadIdx.x] = s + u + d + v;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double *in, *out; long long* cyc;
  cudaMallocManaged(&in, 128 * 8); cudaMallocManaged(&out, 128 * 8); cudaMallocManaged(&cyc, 64);
  for (int i = 0; i < 128; i++) in[i] = 1.0 + 1e-3 * i;
  for (int r = 0; r < 3; r++) { mb10<<<1, 32>>>(in, out, cyc); cudaDeviceSynchronize(); }
  printf("24-link dmul+dadd chain: %lld cycles (%.1f/link); 24 dadd: %lld (%.1f/link); ddiv: %lld; 24 dfma chain: %lld (%.1f/link)\n",
         cyc[0], cyc[0] / 24.0, cyc[1], cyc[1] / 24.0, cyc[2], cyc[3], cyc[3] / 24.0);
  return 0;
}
