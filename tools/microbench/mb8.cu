// Hand-off latency map (development aid): CTA 0 ping-pongs one 8-byte word with every other CTA,
// with the word pair placed at 8 different 2 KB-grain addresses (L2 home varies with address).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned long long* slot, int partner, int iters, long long* out, unsigned* smid) {
  if (threadIdx.x != 0) return;
  const int me = blockIdx.x;
  unsigned id; asm volatile("mov.u32 %0, %%smid;" : "=r"(id)); smid[me] = id;
  if (me != 0 && me != partner) return;
  unsigned long long* mine = slot + (me == 0 ? 0 : 16);
  unsigned long long* theirs = slot + (me == 0 ? 16 : 0);
  long long t0 = clock64();
  for (int i = 1; i <= iters; i++) {
    if (me == 0) {
      asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(theirs), "l"((unsigned long long)i) : "memory");
      unsigned long long v;
      do { asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory"); } while (v != (unsigned long long)i);
    } else {
      unsigned long long v;
      do { asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory"); } while (v != (unsigned long long)i);
      asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(theirs), "l"((unsigned long long)i) : "memory");
    }
  }
  if (me == 0) out[0] = clock64() - t0;
}
int main() {
  unsigned long long* slot; long long* out; unsigned* smid;
  const int NO = 8;
  cudaMalloc(&slot, 2048 * NO * 8); cudaMalloc(&out, 8); cudaMalloc(&smid, 148 * 4);
  const int iters = 1000;
  printf("partner smid0 smidp | one-way cycles at %d addresses\n", NO);
  for (int partner = 1; partner < 148; partner++) {
    unsigned s[148];
    double c[NO];
    for (int o = 0; o < NO; o++) {
      unsigned long long* sl = slot + (size_t)o * 2048;  // 16 KB apart
      cudaMemset(sl, 0, 256);
      k<<<148, 32>>>(sl, partner, iters, out, smid);
      cudaDeviceSynchronize();
      long long cc; cudaMemcpy(&cc, out, 8, cudaMemcpyDeviceToHost);
      c[o] = cc / (2.0 * iters);
      cudaMemcpy(s, smid, 148 * 4, cudaMemcpyDeviceToHost);
    }
    printf("%3d %3u %3u |", partner, s[0], s[partner]);
    for (int o = 0; o < NO; o++) printf(" %4.0f", c[o]);
    printf("\n");
  }
  return 0;
}
