// Latency microbenchmarks for the K2 slice code (development aid, not the product).
//   1. dependent DADD / DMUL / DFMA chains, __ddiv_rn chain
//   2. dependent LDS chain (pointer chase in shared memory)
//   3. one warp running an interior slice (R=32 rows, W entries, private x~ in smem): variants
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void k_chain(double* out, long long* cyc, double a, double b) {
  double x = a, y = b;
  long long t0 = clock64();
  for (int i = 0; i < 1024; i++) x = __dadd_rn(x, y);
  long long t1 = clock64();
  for (int i = 0; i < 1024; i++) x = __dmul_rn(x, y);
  long long t2 = clock64();
  for (int i = 0; i < 1024; i++) x = fma(x, y, a);
  long long t3 = clock64();
  for (int i = 0; i < 128; i++) x = __ddiv_rn(b, x);
  long long t4 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}

__global__ void k_lds(int* out, long long* cyc, int n) {
  __shared__ int nxt[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) nxt[i] = (i * 97 + 13) & 4095;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) p = nxt[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}


__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ double lds64(unsigned a) { double v; asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a)); return v; }
__device__ __forceinline__ unsigned lds32(unsigned a) { unsigned v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a)); return v; }
__device__ __forceinline__ void sts64(unsigned a, double v) { asm volatile("st.shared.f64 [%0], %1;" :: "r"(a), "d"(v) : "memory"); }
__device__ __forceinline__ unsigned opaque(unsigned v) { asm volatile("mov.u32 %0, %0;" : "+r"(v)); return v; }
__device__ __forceinline__ void sts64_if(unsigned p, unsigned a, double v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %0, 0;\n @q st.shared.f64 [%1], %2;\n}" :: "r"(p), "r"(a), "d"(v) : "memory");
}
constexpr int kB = 8;
template <int MAXJ, int VAR>
__global__ void k_slice(const double* gval, const unsigned* gcol, const unsigned short* glen, const double* gf, int R, int W,
                        double* out, long long* cyc, int reps) {
  extern __shared__ double sm[];
  double* val = sm;                    // W*R
  double* fv = val + W * R;            // R
  double* xloc = fv + R;               // 8192
  unsigned* col = (unsigned*)(xloc + 8192);
  unsigned short* len = (unsigned short*)(col + W * R);
  for (int i = threadIdx.x; i < W * R; i += blockDim.x) { val[i] = gval[i]; col[i] = gcol[i]; }
  for (int i = threadIdx.x; i < R; i += blockDim.x) { fv[i] = gf[i]; len[i] = glen[i]; }
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) xloc[i] = 1.0 + 1e-3 * i;
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  long long best = 1LL << 60;
  for (int rep = 0; rep < reps; rep++) {
    __syncwarp();
    long long t0 = clock64();
    const int myl = lane < R ? (int)len[lane] : 0;
    const double f = lane < R ? fv[lane] : 0.0;
    double s = 0.0, n2 = 0.0;
    if (VAR == 0) {  // as in k2 v3: cached xr[MAXJ], batches of 8, guarded
      double xr[MAXJ];
#pragma unroll
      for (int jb = 0; jb < MAXJ; jb += kB) {
        if (jb < W) {
          unsigned c[kB];
#pragma unroll
          for (int u = 0; u < kB; u++) c[u] = (jb + u < myl) ? col[(jb + u) * R + lane] : 0u;
#pragma unroll
          for (int u = 0; u < kB; u++) xr[jb + u] = (jb + u < myl) ? xloc[c[u]] : 0.0;
#pragma unroll
          for (int u = 0; u < kB; u++)
            if (jb + u < myl) {
              const double a = val[(jb + u) * R + lane];
              s = __dadd_rn(s, __dmul_rn(a, xr[jb + u]));
              n2 = __dadd_rn(n2, __dmul_rn(a, a));
            }
        }
      }
      const double alpha = __ddiv_rn(__dsub_rn(f, s), n2);
#pragma unroll
      for (int jb = 0; jb < MAXJ; jb += kB) {
        if (jb < W) {
#pragma unroll
          for (int u = 0; u < kB; u++)
            if (jb + u < myl) {
              const unsigned c = col[(jb + u) * R + lane];
              xloc[c] = __dadd_rn(xr[jb + u], __dmul_rn(alpha, val[(jb + u) * R + lane]));
            }
        }
      }
    } else if (VAR == 1) {  // rolled loops, no register cache; pass 2 re-gathers from smem
      for (int j = 0; j < myl; j++) {
        const double a = val[j * R + lane];
        const double x = xloc[col[j * R + lane]];
        s = __dadd_rn(s, __dmul_rn(a, x));
        n2 = __dadd_rn(n2, __dmul_rn(a, a));
      }
      const double alpha = __ddiv_rn(__dsub_rn(f, s), n2);
      for (int j = 0; j < myl; j++) {
        const unsigned c = col[j * R + lane];
        xloc[c] = __dadd_rn(xloc[c], __dmul_rn(alpha, val[j * R + lane]));
      }
    } else if (VAR == 2) {  // unroll 8 with predication only (no per-batch branch), re-gather in pass 2
      for (int jb = 0; jb < W; jb += kB) {
        double av[kB], xv[kB];
#pragma unroll
        for (int u = 0; u < kB; u++) {
          const bool act = jb + u < myl;
          const unsigned c = act ? col[(jb + u) * R + lane] : 0u;
          av[u] = act ? val[(jb + u) * R + lane] : 0.0;
          xv[u] = act ? xloc[c] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kB; u++)
          if (jb + u < myl) { s = __dadd_rn(s, __dmul_rn(av[u], xv[u])); n2 = __dadd_rn(n2, __dmul_rn(av[u], av[u])); }
      }
      const double alpha = __ddiv_rn(__dsub_rn(f, s), n2);
      for (int jb = 0; jb < W; jb += kB) {
        unsigned cc[kB]; double av[kB], xv[kB];
#pragma unroll
        for (int u = 0; u < kB; u++) {
          const bool act = jb + u < myl;
          cc[u] = act ? col[(jb + u) * R + lane] : 0u;
          av[u] = act ? val[(jb + u) * R + lane] : 0.0;
          xv[u] = act ? xloc[cc[u]] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kB; u++)
          if (jb + u < myl) xloc[cc[u]] = __dadd_rn(xv[u], __dmul_rn(alpha, av[u]));
      }
    } else if (VAR == 3 || VAR == 4) {  // shared-window u32 addresses, unconditional loads, predicated math
      const unsigned vb = su32(val) + lane * 8, cb = su32(col) + lane * 4, xb = su32(xloc);
      const unsigned vs = R * 8, cs = R * 4;
      double xr[MAXJ];
#pragma unroll
      for (int jb = 0; jb < MAXJ; jb += kB) {
        if (jb < W) {
          unsigned c[kB]; double av[kB];
#pragma unroll
          for (int u = 0; u < kB; u++) c[u] = lds32(cb + min(jb + u, W - 1) * cs);
#pragma unroll
          for (int u = 0; u < kB; u++) xr[jb + u] = lds64(xb + c[u] * 8);
#pragma unroll
          for (int u = 0; u < kB; u++) av[u] = lds64(vb + min(jb + u, W - 1) * vs);
#pragma unroll
          for (int u = 0; u < kB; u++)
            if (jb + u < myl) { s = __dadd_rn(s, __dmul_rn(av[u], xr[jb + u])); n2 = __dadd_rn(n2, __dmul_rn(av[u], av[u])); }
        }
      }
      const double alpha = __ddiv_rn(__dsub_rn(f, s), n2);
#pragma unroll
      for (int jb = 0; jb < MAXJ; jb += kB) {
        if (jb < W) {
          unsigned c[kB]; double av[kB];
#pragma unroll
          for (int u = 0; u < kB; u++) { c[u] = lds32(cb + min(jb + u, W - 1) * cs); av[u] = lds64(vb + min(jb + u, W - 1) * vs); }
#pragma unroll
          for (int u = 0; u < kB; u++) {
            const double xo = VAR == 3 ? xr[jb + u] : lds64(xb + c[u] * 8);
            if (jb + u < myl) sts64(xb + c[u] * 8, __dadd_rn(xo, __dmul_rn(alpha, av[u])));
          }
        }
      }
    } else if (VAR == 5 || VAR == 6) {  // + zero-slot padding: unpredicated math, predicated stores
      const unsigned vb = su32(val) + lane * 8, cb = su32(col) + lane * 4, xb = su32(xloc);
      const unsigned vs = R * 8, cs = R * 4;
      double xr[MAXJ];
#pragma unroll
      for (int jb = 0; jb < MAXJ; jb += kB) {
        if (jb < W) {
          unsigned c[kB]; double av[kB];
#pragma unroll
          for (int u = 0; u < kB; u++) c[u] = lds32(cb + min(jb + u, W - 1) * cs);
#pragma unroll
          for (int u = 0; u < kB; u++) xr[jb + u] = lds64(xb + c[u] * 8);
#pragma unroll
          for (int u = 0; u < kB; u++) av[u] = lds64(vb + min(jb + u, W - 1) * vs);
#pragma unroll
          for (int u = 0; u < kB; u++)
            if (VAR == 6 || jb + u < W) { s = __dadd_rn(s, __dmul_rn(av[u], xr[jb + u])); n2 = __dadd_rn(n2, __dmul_rn(av[u], av[u])); }
        }
      }
      long long tA = clock64();
      const double alpha = __ddiv_rn(__dsub_rn(f, s), n2);
      double alpha2 = alpha;
      asm volatile("mov.b64 %0, %0;" : "+d"(alpha2));
      long long tB = clock64();
      if (lane == 0 && rep == reps - 1) { cyc[1] = tA - t0; cyc[2] = tB - tA; }
#pragma unroll
      for (int jb = 0; jb < MAXJ; jb += kB) {
        if (jb < W) {
          unsigned c[kB]; double av[kB];
#pragma unroll
          for (int u = 0; u < kB; u++) { c[u] = lds32(cb + min(jb + u, W - 1) * cs); av[u] = lds64(vb + min(jb + u, W - 1) * vs); }
#pragma unroll
          for (int u = 0; u < kB; u++) {
            const double xn = __dadd_rn(xr[jb + u], __dmul_rn(alpha2, av[u]));
            if (jb + u < myl) sts64(xb + c[u] * 8, xn);
          }
        }
      }
    } else if (VAR == 8 || VAR == 9) {  // opaque u32 bases, zero-slot padding, unpredicated math, predicated asm stores
      const int ln = lane < R ? lane : 0;
      const unsigned vb = opaque(su32(val) + ln * 8), cb = opaque(su32(col) + ln * 4), xb = opaque(su32(xloc));
      const unsigned vs = R * 8, cs = R * 4;
      double xr[MAXJ];
#pragma unroll
      for (int jb = 0; jb < MAXJ; jb += kB) {
        if (jb < W) {
          unsigned c[kB]; double av[kB];
#pragma unroll
          for (int u = 0; u < kB; u++) c[u] = lds32(cb + min(jb + u, W - 1) * cs);
#pragma unroll
          for (int u = 0; u < kB; u++) xr[jb + u] = lds64(xb + c[u] * 8);
#pragma unroll
          for (int u = 0; u < kB; u++) av[u] = lds64(vb + min(jb + u, W - 1) * vs);
#pragma unroll
          for (int u = 0; u < kB; u++)
            if (VAR == 9 || jb + u < W) { s = __dadd_rn(s, __dmul_rn(av[u], xr[jb + u])); n2 = __dadd_rn(n2, __dmul_rn(av[u], av[u])); }
        }
      }
      const double alpha = __ddiv_rn(__dsub_rn(f, s), n2);
#pragma unroll
      for (int jb = 0; jb < MAXJ; jb += kB) {
        if (jb < W) {
          unsigned c[kB]; double av[kB];
#pragma unroll
          for (int u = 0; u < kB; u++) { c[u] = lds32(cb + min(jb + u, W - 1) * cs); av[u] = lds64(vb + min(jb + u, W - 1) * vs); }
#pragma unroll
          for (int u = 0; u < kB; u++) sts64_if(jb + u < myl, xb + c[u] * 8, __dadd_rn(xr[jb + u], __dmul_rn(alpha, av[u])));
        }
      }
    } else if (VAR == 10) {  // all loads first (uniform batch guards), then math; val re-read in the math loop
      const int ln = lane < R ? lane : 0;
      const unsigned vb = opaque(su32(val) + ln * 8), cb = opaque(su32(col) + ln * 4), xb = opaque(su32(xloc));
      const unsigned vs = R * 8, cs = R * 4;
      double xr[MAXJ];
      unsigned c[MAXJ];
#pragma unroll
      for (int jb = 0; jb < MAXJ; jb += kB)
        if (jb < W) {
#pragma unroll
          for (int u = 0; u < kB; u++) c[jb + u] = lds32(cb + min(jb + u, W - 1) * cs);
        }
#pragma unroll
      for (int jb = 0; jb < MAXJ; jb += kB)
        if (jb < W) {
#pragma unroll
          for (int u = 0; u < kB; u++) xr[jb + u] = lds64(xb + c[jb + u] * 8);
        }
#pragma unroll
      for (int jb = 0; jb < MAXJ; jb += kB)
        if (jb < W) {
#pragma unroll
          for (int u = 0; u < kB; u++)
            if (jb + u < W) {
              const double a = lds64(vb + (jb + u) * vs);
              s = __dadd_rn(s, __dmul_rn(a, xr[jb + u]));
              n2 = __dadd_rn(n2, __dmul_rn(a, a));
            }
        }
      const double alpha = __ddiv_rn(__dsub_rn(f, s), n2);
#pragma unroll
      for (int jb = 0; jb < MAXJ; jb += kB) {
        if (jb < W) {
          double av[kB];
#pragma unroll
          for (int u = 0; u < kB; u++) av[u] = lds64(vb + min(jb + u, W - 1) * vs);
#pragma unroll
          for (int u = 0; u < kB; u++) sts64_if(jb + u < myl, xb + c[jb + u] * 8, __dadd_rn(xr[jb + u], __dmul_rn(alpha, av[u])));
        }
      }
    } else if (VAR == 7) {  // empty: timing overhead
      s = f;
    }
    __syncwarp();
    long long t1 = clock64();
    if (t1 - t0 < best) best = t1 - t0;
    if (lane == 0 && rep == reps - 1) out[0] = s + n2;
  }
  if (lane == 0) cyc[0] = best;
}

int main() {
  double* dout; long long* dcyc; int* iout;
  CK(cudaMalloc(&dout, 4096 * 8)); CK(cudaMalloc(&dcyc, 64)); CK(cudaMalloc(&iout, 4096 * 4));
  long long h[4];
  k_chain<<<1, 32>>>(dout, dcyc, 1.0000001, 0.9999999); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h, dcyc, 32, cudaMemcpyDeviceToHost));
  printf("latency (cycles/op): dadd %.2f dmul %.2f dfma %.2f ddiv %.2f\n", h[0] / 1024.0, h[1] / 1024.0, h[2] / 1024.0, h[3] / 128.0);
  k_lds<<<1, 32>>>(iout, dcyc, 4096); CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h, dcyc, 8, cudaMemcpyDeviceToHost));
  printf("lds dependent chain %.2f cycles/load\n", h[0] / 4096.0);
  std::mt19937 rng(1);
  for (int W : {8, 17, 24}) {
    const int R = 32;
    std::vector<double> val(W * R), f(R); std::vector<unsigned> col(W * R); std::vector<unsigned short> len(R);
    for (int r = 0; r < R; r++) { len[r] = W - (r * 2 / R); f[r] = 1.0 + r; }
    std::vector<unsigned> perm(8192); for (int i = 0; i < 8192; i++) perm[i] = i; std::shuffle(perm.begin(), perm.end(), rng);
    for (int i = 0; i < W * R; i++) { val[i] = 0.5 + (rng() % 1000) * 1e-3; col[i] = perm[i % 8192]; }
    double *dv, *df; unsigned* dc; unsigned short* dl;
    CK(cudaMalloc(&dv, W * R * 8)); CK(cudaMalloc(&df, R * 8)); CK(cudaMalloc(&dc, W * R * 4)); CK(cudaMalloc(&dl, R * 2));
    CK(cudaMemcpy(dv, val.data(), W * R * 8, cudaMemcpyHostToDevice)); CK(cudaMemcpy(df, f.data(), R * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dc, col.data(), W * R * 4, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dl, len.data(), R * 2, cudaMemcpyHostToDevice));
    size_t sm = (W * R + R + 8192) * 8 + W * R * 4 + R * 2 + 64;
    auto run = [&](auto kern, const char* nm) {
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      kern<<<1, 128, sm>>>(dv, dc, dl, df, R, W, dout, dcyc, 20); CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(h, dcyc, 8, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(h, dcyc, 24, cudaMemcpyDeviceToHost));
      printf("slice W=%d %s: %lld cycles (pass1 %lld, ddiv %lld)\n", W, nm, h[0], h[1], h[2]);
      CK(cudaMemset(dcyc, 0, 24));
    };
    run(k_slice<24, 0>, "v3 (cached, batch-branches)");
    run(k_slice<24, 1>, "rolled, regather");
    run(k_slice<24, 2>, "unroll8 predicated, regather");
    run(k_slice<24, 3>, "u32 smem asm, cached");
    run(k_slice<24, 4>, "u32 smem asm, regather");
    run(k_slice<24, 5>, "u32 + zero-slot pad (math guarded by W only)");
    run(k_slice<24, 6>, "u32 + zero-slot pad (no guard; pad rows to batch)");
    run(k_slice<24, 8>, "opaque bases + zero-slot + asm pred stores");
    run(k_slice<24, 9>, "  same, math over whole batches");
    run(k_slice<24, 10>, "all loads first, then math");
    run(k_slice<16, 10>, "all loads first, then math (MAXJ 16)");
    run(k_slice<24, 7>, "empty");
  }
  return 0;
}
