// One-way cross-SM hand-off latency (development aid): CTA 0 and CTA p ping-pong one 8-byte word
// with relaxed gpu-scope stores / polling loads (K2's mailbox protocol), for several partners p.
#include <cstdio>
#include <cstdlib>
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
  cudaMalloc(&slot, 4096); cudaMalloc(&out, 8); cudaMalloc(&smid, 148 * 4);
  const int iters = 2000;
  for (int partner : {1, 2, 10, 37, 74, 75, 100, 147}) {
    cudaMemset(slot, 0, 4096);
    k<<<148, 32>>>(slot, partner, iters, out, smid);
    cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
    unsigned s[148]; cudaMemcpy(s, smid, 148 * 4, cudaMemcpyDeviceToHost);
    printf("CTA 0 (SM %u) <-> CTA %d (SM %u): one-way %.0f cycles\n", s[0], partner, s[partner], c / (2.0 * iters));
  }
  return 0;
}
