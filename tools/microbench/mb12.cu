// Cluster barrier and DSMEM round-trip cost on sm_100a (development aid): C CTAs of one cluster
// run N iterations of (a) barrier.cluster arrive.release + wait.acquire alone, (b) the same plus
// one remote ld/st.shared::cluster per thread.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned rank() { unsigned r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ unsigned nctas() { unsigned r; asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r)); return r; }
__global__ void mb12(int n, int mode, long long* out) {
  __shared__ double buf[256];
  buf[threadIdx.x] = threadIdx.x;
  csync();
  unsigned a = (unsigned)__cvta_generic_to_shared(&buf[threadIdx.x]), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"((rank() + 1) % nctas()));
  long long t0 = clock64();
  double v = 0;
  for (int i = 0; i < n; i++) {
    if (mode == 1) {
      double w;
      asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(w) : "r"(ra) : "memory");
      v += w;
      asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
    }
    if (mode != 2) csync();
    else __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && rank() == 0) out[mode] = (t1 - t0) / n;
  if (v == -1) out[9] = 1;
}
int main() {
  long long* out;
  cudaMallocManaged(&out, 128);
  for (int C : {2, 8, 16}) {
    cudaFuncSetAttribute(mb12, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int mode = 0; mode < 3; mode++) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(C); cfg.blockDim = dim3(256);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      for (int r = 0; r < 2; r++) cudaLaunchKernelEx(&cfg, mb12, 2000, mode, out);
      cudaError_t e = cudaDeviceSynchronize();
      printf("C=%2d mode=%d (%s): %lld cycles/iter %s\n", C, mode, mode == 0 ? "cluster sync" : mode == 1 ? "dsmem ld+st + cluster sync" : "__syncthreads", out[mode], e ? cudaGetErrorString(e) : "");
    }
  }
  return 0;
}
