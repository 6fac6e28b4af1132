// Row-sum chain orderings on sm_100a (development aid): s = s + a_j*x_j left to right with the
// products (a) interleaved (as written), (b) computed in a separate loop first, (c) pinned ahead of
// the chain with volatile register moves.  Same operations, same order of additions.
#include <cstdio>
__global__ void mb11(const double* in, double* out, long long* cyc) {
  double a[24], x[24];
  for (int j = 0; j < 24; j++) { a[j] = in[j + threadIdx.x]; x[j] = in[j + 24 + threadIdx.x]; }
  long long t0 = clock64();
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 24; j++) s = __dadd_rn(s, __dmul_rn(a[j], x[j]));
  asm volatile("mov.b64 %0, %0;" : "+d"(s));
  long long t1 = clock64();
  double p[24];
#pragma unroll
  for (int j = 0; j < 24; j++) p[j] = __dmul_rn(a[j], x[j] + s);
  double u = 0.0;
#pragma unroll
  for (int j = 0; j < 24; j++) u = __dadd_rn(u, p[j]);
  asm volatile("mov.b64 %0, %0;" : "+d"(u));
  long long t2 = clock64();
  double q[24];
#pragma unroll
  for (int j = 0; j < 24; j++) q[j] = __dmul_rn(a[j], x[j] + u);
#pragma unroll
  for (int j = 0; j < 24; j++) asm volatile("mov.b64 %0, %0;" : "+d"(q[j]));
  double v = 0.0;
#pragma unroll
  for (int j = 0; j < 24; j++) v = __dadd_rn(v, q[j]);
  asm volatile("mov.b64 %0, %0;" : "+d"(v));
  long long t3 = clock64();
  out[threadIdx.x] = s + u + v;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
  double *in, *out; long long* cyc;
  cudaMallocManaged(&in, 128 * 8); cudaMallocManaged(&out, 128 * 8); cudaMallocManaged(&cyc, 64);
  for (int i = 0; i < 128; i++) in[i] = 1.0 + 1e-3 * i;
  for (int r = 0; r < 3; r++) { mb11<<<1, 32>>>(in, out, cyc); cudaDeviceSynchronize(); }
  printf("interleaved %lld (%.1f/link); products first %lld (%.1f/link); pinned products %lld (%.1f/link)\n",
         cyc[0], cyc[0] / 24.0, cyc[1], cyc[1] / 24.0, cyc[2], cyc[2] / 24.0);
  return 0;
}
