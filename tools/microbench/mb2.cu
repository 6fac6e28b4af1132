// Microbench 2: one emulated category step (disjoint supports, RMW of x), vector-per-row,
// and flag-latency variants.  Not part of the product.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int V, bool CG>
__global__ void k_step(const int* __restrict__ rp, const int* __restrict__ col, const double* __restrict__ val,
                       const double* __restrict__ f, const double* __restrict__ nrm2, double* x, int r0, int r1) {
  int lane = threadIdx.x % V;
  int row = r0 + (blockIdx.x * blockDim.x + threadIdx.x) / V;
  if (row >= r1) return;   // whole vector exits together (V divides 32)
  int p0 = rp[row], p1 = rp[row + 1];
  double s = 0; double xv[4]; int cc[4]; double vv[4]; int n = 0;
  for (int p = p0 + lane; p < p1; p += V) {
    int c = __ldg(col + p); double a = __ldg(val + p);
    double xx = CG ? __ldcg(x + c) : x[c];
    s += a * xx;
    if (n < 4) { xv[n] = xx; cc[n] = c; vv[n] = a; } n++;
  }
#pragma unroll
  for (int o = V / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, V);
  double alpha = (f[row] - s) / nrm2[row];
  for (int k = 0; k < n && k < 4; k++) { if (CG) __stcg(x + cc[k], xv[k] + alpha * vv[k]); else x[cc[k]] = xv[k] + alpha * vv[k]; }
}

__global__ void k_pp(int* flag, int iters, int mode) {
  if (threadIdx.x != 0 || blockIdx.x > 1) return;
  int me = blockIdx.x;
  for (int i = 0; i < iters; i++) {
    int want = 2 * i + me, next = 2 * i + me + 1; int v;
    if (mode == 0) {  // acquire poll, release store
      do { asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory"); } while (v != want);
      asm volatile("st.release.gpu.global.b32 [%0], %1;" :: "l"(flag), "r"(next) : "memory");
    } else if (mode == 1) {  // relaxed poll + fence; fence + relaxed store
      do { asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory"); } while (v != want);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" :: "l"(flag), "r"(next) : "memory");
    } else if (mode == 2) {  // volatile poll, no fences (latency floor)
      do { v = *(volatile int*)flag; } while (v != want);
      *(volatile int*)flag = next;
    } else {  // atomic exch store
      do { asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory"); } while (v != want);
      atomicExch(flag, next);
    }
  }
}

int main() {
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1)); float ms;
  // emulated config-4 sweep: m = 1M rows, 16 nnz/row, 33 categories; category c holds rows r with
  // (r / 21) % 33 == c ... simpler: rows of category c are r = c + 33*k; row r touches 16 of the 21
  // columns in [r*... ] -- use disjoint column blocks per row inside a category: block = r (own index)
  const int m = 1 << 20, ncat = 33, npr = 16;
  std::vector<int> rp(m + 1), col((size_t)m * npr), order(m);
  std::mt19937 rng(7);
  // sweep order: category-major
  int pos = 0;
  std::vector<int> cat_ptr(ncat + 1);
  for (int c = 0; c < ncat; c++) { cat_ptr[c] = pos; for (int r = c; r < m; r += ncat) order[pos++] = r; }
  cat_ptr[ncat] = pos;
  for (int s = 0; s < m; s++) {
    int r = order[s]; rp[s] = s * npr;
    // columns: 16 distinct from r-16..r+16 (conflicting rows share columns; within a category rows are 33 apart -> overlap!)
    // to keep disjointness within a category, use columns in [r - 16, r + 16] step pattern that stays inside r's 33-window
    int base = (r / ncat) * ncat;  // window [base, base+33) owned by the 33 rows of this window (one per category)
    std::vector<int> cand(ncat); for (int k = 0; k < ncat; k++) cand[k] = base + k;
    std::shuffle(cand.begin(), cand.end(), rng);
    std::sort(cand.begin(), cand.begin() + npr);
    for (int k = 0; k < npr; k++) col[(size_t)s * npr + k] = std::min(cand[k], m - 1);
  }
  rp[m] = m * npr;
  // NOTE: rows in the same category touch columns in disjoint windows -> disjoint supports.
  int *d_rp, *d_col; double *d_val, *d_f, *d_n, *d_x;
  CK(cudaMalloc(&d_rp, (m + 1) * 4)); CK(cudaMalloc(&d_col, (size_t)m * npr * 4)); CK(cudaMalloc(&d_val, (size_t)m * npr * 8));
  CK(cudaMalloc(&d_f, m * 8)); CK(cudaMalloc(&d_n, m * 8)); CK(cudaMalloc(&d_x, m * 8));
  CK(cudaMemcpy(d_rp, rp.data(), (m + 1) * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_col, col.data(), (size_t)m * npr * 4, cudaMemcpyHostToDevice));
  std::vector<double> ones((size_t)m * npr, 0.01); CK(cudaMemcpy(d_val, ones.data(), (size_t)m * npr * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_f, ones.data(), m * 8, cudaMemcpyHostToDevice)); std::vector<double> n2(m, 1.0);
  CK(cudaMemcpy(d_n, n2.data(), m * 8, cudaMemcpyHostToDevice)); CK(cudaMemset(d_x, 0, m * 8));
  cudaStream_t st; CK(cudaStreamCreate(&st));
  auto sweep = [&](int v, bool cg) {
    for (int c = 0; c < ncat; c++) {
      int r0 = cat_ptr[c], r1 = cat_ptr[c + 1]; int rows = r1 - r0; int thr = 256; int blocks = (rows * v + thr - 1) / thr;
      if (v == 4 && cg) k_step<4, true><<<blocks, thr, 0, st>>>(d_rp, d_col, d_val, d_f, d_n, d_x, r0, r1);
      if (v == 8 && cg) k_step<8, true><<<blocks, thr, 0, st>>>(d_rp, d_col, d_val, d_f, d_n, d_x, r0, r1);
      if (v == 16 && cg) k_step<16, true><<<blocks, thr, 0, st>>>(d_rp, d_col, d_val, d_f, d_n, d_x, r0, r1);
      if (v == 8 && !cg) k_step<8, false><<<blocks, thr, 0, st>>>(d_rp, d_col, d_val, d_f, d_n, d_x, r0, r1);
    }
  };
  for (int v : {4, 8, 16}) for (int cg : {1, 0}) {
    if (!cg && v != 8) continue;
    cudaGraph_t g; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal)); for (int k = 0; k < 10; k++) sweep(v, cg); CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0)); CK(cudaGraphLaunch(ge, st)); CK(cudaStreamSynchronize(st));
    CK(cudaEventRecord(e0, st)); for (int r = 0; r < 5; r++) CK(cudaGraphLaunch(ge, st)); CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    double t = ms / 50 * 1e-3; double B = 12.0 * m * npr + 12.0 * m;
    printf("per-category graph sweep V=%d %s: %.1f us/sweep, alg %.0f GB/s (%.0f%% of 6556)\n", v, cg ? ".cg" : "default", t * 1e6, B / t / 1e9, 100 * B / t / 1e9 / 6556.5);
  }
  // single huge step (all rows, emulating ideal no-sync): treat the whole matrix as one launch
  {
    int thr = 256, blocks = (m * 8 + thr - 1) / thr;
    k_step<8, true><<<blocks, thr, 0, st>>>(d_rp, d_col, d_val, d_f, d_n, d_x, 0, m); CK(cudaStreamSynchronize(st));
    CK(cudaEventRecord(e0, st)); for (int r = 0; r < 20; r++) k_step<8, true><<<blocks, thr, 0, st>>>(d_rp, d_col, d_val, d_f, d_n, d_x, 0, m);
    CK(cudaEventRecord(e1, st)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    double t = ms / 20 * 1e-3; double B = 12.0 * m * npr + 12.0 * m;
    printf("single launch over all rows (racy, throughput only) V=8: %.1f us, alg %.0f GB/s\n", t * 1e6, B / t / 1e9);
  }
  int* flag; CK(cudaMalloc(&flag, 4));
  for (int mode = 0; mode < 4; mode++) {
    CK(cudaMemset(flag, 0, 4)); int iters = 10000;
    CK(cudaEventRecord(e0)); k_pp<<<2, 32>>>(flag, iters, mode); CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("pingpong mode %d: %.3f us per hop\n", mode, ms * 1e3 / (2.0 * iters));
  }
  printf("done\n");
}
