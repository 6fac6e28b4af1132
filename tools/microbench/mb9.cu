// Latency of one poll round (development aid): one warp issues NJ independent 8-byte loads per lane
// (lanes coalesced, entries R*8 bytes apart, L2-resident) and waits for all of them, for several
// load flavours: relaxed.gpu (K2's mailbox polls), volatile, .cg, .cv, default (.ca).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__device__ __forceinline__ unsigned long long ld(const unsigned long long* p) {
  unsigned long long v;
  if (MODE == 0) asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  if (MODE == 1) asm volatile("ld.volatile.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  if (MODE == 2) asm volatile("ld.global.cg.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  if (MODE == 3) asm volatile("ld.global.cv.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  if (MODE == 4) asm volatile("ld.global.b64 %0, [%1];" : "=l"(v) : "l"(p));
  if (MODE == 5) asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
template <int MODE, int NJ>
__global__ void k(const unsigned long long* mb, int R, long long* out) {
  const int lane = threadIdx.x;
  long long best = 1LL << 60;
  unsigned long long acc = 0;
  for (int rep = 0; rep < 64; rep++) {
    const unsigned long long* b = mb + (size_t)(rep & 7) * NJ * R + lane;
    __syncwarp();
    long long t0 = clock64();
    unsigned long long v[NJ];
#pragma unroll
    for (int j = 0; j < NJ; j++) v[j] = ld<MODE>(b + (size_t)j * R);
    unsigned long long x = 0;
#pragma unroll
    for (int j = 0; j < NJ; j++) x ^= v[j];
    acc += __any_sync(~0u, x == 12345) ? 1 : 0;
    long long t1 = clock64();
    best = min(best, t1 - t0);
  }
  if (lane == 0) { out[0] = best; out[1] = acc; }
}
// ACT active lanes; VEC: 1 = 8 B per lane, 2 = 16 B per lane (ld.v2.b64), 4 = 32 B per lane (ld.v4.b64)
template <int NJ, int ACT, int VEC>
__global__ void kv(const unsigned long long* mb, int R, long long* out) {
  const int lane = threadIdx.x;
  long long best = 1LL << 60;
  unsigned long long acc = 0;
  for (int rep = 0; rep < 64; rep++) {
    const unsigned long long* b = mb + (size_t)(rep & 7) * NJ * R * VEC + lane * VEC;
    __syncwarp();
    long long t0 = clock64();
    unsigned long long v[NJ][VEC];
#pragma unroll
    for (int j = 0; j < NJ; j++) {
      const unsigned long long* p = b + (size_t)j * R * VEC;
      if (VEC == 1) asm volatile("{\n .reg .pred q;\n setp.lt.s32 q, %2, %3;\n mov.b64 %0, 0;\n @q ld.relaxed.gpu.global.b64 %0, [%1];\n}" : "=l"(v[j][0]) : "l"(p), "r"(lane), "n"(ACT) : "memory");
      if (VEC == 2) asm volatile("{\n .reg .pred q;\n setp.lt.s32 q, %3, %4;\n mov.b64 %0, 0;\n mov.b64 %1, 0;\n @q ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];\n}" : "=l"(v[j][0]), "=l"(v[j][VEC > 1 ? 1 : 0]) : "l"(p), "r"(lane), "n"(ACT) : "memory");
      if (VEC == 4) asm volatile("{\n .reg .pred q;\n setp.lt.s32 q, %5, %6;\n @q ld.relaxed.gpu.global.v4.b64 {%0, %1, %2, %3}, [%4];\n}" : "=l"(v[j][0]), "=l"(v[j][VEC > 1 ? 1 : 0]), "=l"(v[j][VEC > 2 ? 2 : 0]), "=l"(v[j][VEC > 3 ? 3 : 0]) : "l"(p), "r"(lane), "n"(ACT) : "memory");
    }
    unsigned long long x = 0;
#pragma unroll
    for (int j = 0; j < NJ; j++)
#pragma unroll
      for (int w = 0; w < VEC; w++) x ^= v[j][w];
    acc += __any_sync(~0u, x == 12345) ? 1 : 0;
    long long t1 = clock64();
    best = min(best, t1 - t0);
  }
  if (lane == 0) { out[0] = best; out[1] = acc; }
}
template <int NJ, int ACT, int VEC>
void runv(const unsigned long long* mb, long long* out) {
  kv<NJ, ACT, VEC><<<1, 32>>>(mb, 32, out);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2]; cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
  printf("relaxed NJ=%2d active=%2d bytes/lane=%2d: %lld cycles per round (%s)\n", NJ, ACT, 8 * VEC, h[0], cudaGetErrorString(e));
}
template <int MODE, int NJ>
void run(const unsigned long long* mb, long long* out, const char* nm) {
  k<MODE, NJ><<<1, 32>>>(mb, 32, out);
  cudaDeviceSynchronize();
  long long h[2]; cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
  printf("%-22s NJ=%2d: %lld cycles per round\n", nm, NJ, h[0]);
}
int main() {
  unsigned long long* mb; long long* out;
  cudaMalloc(&mb, 8 * 24 * 32 * 8 * 4); cudaMalloc(&out, 16);
  cudaMemset(mb, 1, 8 * 24 * 32 * 8 * 4);
  run<0, 1>(mb, out, "relaxed.gpu");
  run<0, 8>(mb, out, "relaxed.gpu");
  run<0, 24>(mb, out, "relaxed.gpu");
  run<5, 24>(mb, out, "relaxed.gpu no-clobber");
  run<1, 24>(mb, out, "volatile");
  run<2, 24>(mb, out, "cg");
  run<3, 24>(mb, out, "cv");
  run<4, 1>(mb, out, "default");
  run<4, 24>(mb, out, "default");
  runv<24, 32, 1>(mb, out);
  runv<24, 16, 1>(mb, out);
  runv<24, 4, 1>(mb, out);
  runv<24, 1, 1>(mb, out);
  runv<24, 0, 1>(mb, out);
  runv<12, 32, 2>(mb, out);
  runv<6, 32, 4>(mb, out);
  runv<8, 32, 1>(mb, out);
  runv<4, 32, 2>(mb, out);
  return 0;
}
