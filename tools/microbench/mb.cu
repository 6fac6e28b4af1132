// Day-one B200 microbenchmarks for the POBK sweep design.
// Not part of the product; numbers feed DESIGN.md.
//   1. HBM streaming read bandwidth (16-B vector loads)
//   2. x-gather / gather+scatter throughput on an L2-resident 8 MB vector,
//      banded random columns (config-4-like |i-j| <= 3000), L2 (.cg) vs L1 (.ca)
//   3. flag ping-pong latency between two CTAs (release/acquire at gpu scope)
//   4. grid-barrier latency over 148 CTAs
//   5. per-kernel cost of back-to-back tiny kernels inside a CUDA graph
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void k_stream(const double2* __restrict__ a, size_t n2, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldg(a + i); s += v.x + v.y;
  }
  if (s == 12345.678) out[0] = s;
}

template <int MODE>  // 0: gather .cg, 1: gather .ca, 2: gather+scatter .cg, 3: gather+scatter .ca
__global__ void k_gather(const int* __restrict__ col, const double* __restrict__ val, double* x, size_t nnz, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nnz; i += (size_t)gridDim.x * blockDim.x) {
    int c = __ldg(col + i); double v = __ldg(val + i);
    double xv;
    if (MODE == 0 || MODE == 2) xv = __ldcg(x + c); else xv = __ldca(x + c);
    s += v * xv;
    if (MODE >= 2) { if (MODE == 2) __stcg(x + c, xv + 1e-30 * v); else x[c] = xv + 1e-30 * v; }
  }
  if (s == 12345.678) out[0] = s;
}

__global__ void k_pingpong(volatile int* flag, int iters, long long* cyc) {
  if (threadIdx.x != 0) return;
  int me = blockIdx.x;
  if (me > 1) return;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
    if (me == 0) {
      int v; do { asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory"); } while (v != 2 * i);
      asm volatile("st.release.gpu.global.b32 [%0], %1;" :: "l"(flag), "r"(2 * i + 1) : "memory");
    } else {
      int v; do { asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory"); } while (v != 2 * i + 1);
      asm volatile("st.release.gpu.global.b32 [%0], %1;" :: "l"(flag), "r"(2 * i + 2) : "memory");
    }
  }
  if (me == 0) cyc[0] = clock64() - t0;
}

__global__ void k_gridbar(unsigned* count, volatile unsigned* gen, int iters) {
  for (int i = 0; i < iters; i++) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned g; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
      unsigned arrived = atomicAdd(count, 1u);
      if (arrived == gridDim.x - 1) {
        *count = 0; __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(gen), "r"(g + 1) : "memory");
      } else {
        unsigned v; do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gen) : "memory"); } while (v == g);
      }
    }
    __syncthreads();
  }
}

__global__ void k_tiny(double* x, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] += 1.0;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s SMs %d L2 %d MB persistL2max %d MB smemOptin %zu\n", p.name, p.multiProcessorCount, p.l2CacheSize >> 20,
         p.persistingL2CacheMaxSize >> 20, p.sharedMemPerBlockOptin);
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  float ms;
  double* out; CK(cudaMalloc(&out, 8));
  const int SMS = p.multiProcessorCount;
  // 1. stream
  {
    size_t n = (size_t)1 << 27;  // 1 GiB of doubles
    double* a; CK(cudaMalloc(&a, n * 8)); CK(cudaMemset(a, 0, n * 8));
    for (int bs : {256, 512, 1024}) for (int per : {2, 4, 8}) {
      k_stream<<<SMS * per, bs>>>((double2*)a, n / 2, out);
      CK(cudaEventRecord(e0));
      for (int r = 0; r < 5; r++) k_stream<<<SMS * per, bs>>>((double2*)a, n / 2, out);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
      printf("stream bs=%d ctas/sm=%d: %.1f GB/s\n", bs, per, 5.0 * n * 8 / (ms * 1e-3) / 1e9);
    }
    CK(cudaFree(a));
  }
  // 2. gather
  {
    const int m = 1 << 20; const size_t nnz = (size_t)m * 16;
    std::vector<int> hc(nnz); std::mt19937 rng(1);
    for (size_t k = 0; k < nnz; k++) { long r = (long)(k / 16); long c = r + (long)(rng() % 3001) - 1500; if (c < 0) c = -c; if (c >= m) c = 2 * m - 2 - c; hc[k] = (int)c; }
    // sort columns within row (as CSR)
    for (int r = 0; r < m; r++) std::sort(hc.begin() + (size_t)r * 16, hc.begin() + (size_t)r * 16 + 16);
    int* col; double* val; double* x;
    CK(cudaMalloc(&col, nnz * 4)); CK(cudaMalloc(&val, nnz * 8)); CK(cudaMalloc(&x, m * 8));
    CK(cudaMemcpy(col, hc.data(), nnz * 4, cudaMemcpyHostToDevice)); CK(cudaMemset(val, 0, nnz * 8)); CK(cudaMemset(x, 0, m * 8));
    auto run = [&](int mode, const char* name) {
      for (int per : {4, 8}) {
        auto launch = [&]() {
          if (mode == 0) k_gather<0><<<SMS * per, 256>>>(col, val, x, nnz, out);
          if (mode == 1) k_gather<1><<<SMS * per, 256>>>(col, val, x, nnz, out);
          if (mode == 2) k_gather<2><<<SMS * per, 256>>>(col, val, x, nnz, out);
          if (mode == 3) k_gather<3><<<SMS * per, 256>>>(col, val, x, nnz, out);
        };
        launch(); CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0)); for (int r = 0; r < 10; r++) launch(); CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
        double t = ms / 10 * 1e-3;
        printf("%s ctas/sm=%d: %.1f us per 16.8M nnz; A-stream %.1f GB/s; %.2f Gnnz/s\n", name, per, t * 1e6, nnz * 12.0 / t / 1e9, nnz / t / 1e9);
      }
    };
    run(0, "gather .cg        "); run(1, "gather .ca        "); run(2, "gather+scatter .cg"); run(3, "gather+scatter .ca");
    CK(cudaFree(col)); CK(cudaFree(val)); CK(cudaFree(x));
  }
  // 3. ping-pong
  {
    int* flag; long long* cyc; CK(cudaMalloc(&flag, 4)); CK(cudaMalloc(&cyc, 8)); CK(cudaMemset(flag, 0, 4));
    for (int nb : {2, 74, 148}) {
      CK(cudaMemset(flag, 0, 4));
      int iters = 10000;
      CK(cudaEventRecord(e0)); k_pingpong<<<nb, 32>>>(flag, iters, cyc); CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
      long long c; CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
      printf("pingpong (grid %d): %.3f us per one-way hop (%.0f cycles)\n", nb, ms * 1e3 / (2.0 * iters), c / (2.0 * iters));
    }
  }
  // 4. grid barrier
  {
    unsigned *cnt, *gen; CK(cudaMalloc(&cnt, 4)); CK(cudaMalloc(&gen, 4)); CK(cudaMemset(cnt, 0, 4)); CK(cudaMemset(gen, 0, 4));
    for (int bs : {256, 1024}) {
      int iters = 2000;
      k_gridbar<<<SMS, bs>>>(cnt, gen, 10); CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0)); k_gridbar<<<SMS, bs>>>(cnt, gen, iters); CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
      printf("grid barrier (%d CTAs x %d thr): %.3f us each\n", SMS, bs, ms * 1e3 / iters);
    }
  }
  // 5. graph of tiny kernels
  {
    double* x; CK(cudaMalloc(&x, 1 << 20)); cudaStream_t s; CK(cudaStreamCreate(&s));
    for (int blocks : {1, 148, 1184}) {
      cudaGraph_t g; cudaGraphExec_t ge;
      CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
      for (int i = 0; i < 100; i++) k_tiny<<<blocks, 128, 0, s>>>(x, blocks * 128 < 131072 ? blocks * 128 : 131072);
      CK(cudaStreamEndCapture(s, &g)); CK(cudaGraphInstantiate(&ge, g, 0));
      CK(cudaGraphLaunch(ge, s)); CK(cudaStreamSynchronize(s));
      CK(cudaEventRecord(e0, s)); for (int r = 0; r < 10; r++) CK(cudaGraphLaunch(ge, s)); CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
      printf("graph of tiny kernels (grid %d): %.3f us per kernel\n", blocks, ms * 1e3 / 1000);
      // plain stream launches
      CK(cudaEventRecord(e0, s)); for (int r = 0; r < 1000; r++) k_tiny<<<blocks, 128, 0, s>>>(x, 1024); CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
      printf("stream of tiny kernels (grid %d): %.3f us per kernel\n", blocks, ms * 1e3 / 1000);
    }
  }
  printf("done\n");
  return 0;
}
