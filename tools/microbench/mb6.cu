// Standalone timing of K2's boundary-slice code (BSlice pre/poll/post) and interior-slice code on
// a synthetic slice: one warp alone, mailboxes already full (development aid).
#include "../../paper_2401_00672_b200/csrc/cuda/k2_wavefront.cu"
#include <random>

namespace pobk {
__global__ void mb6(const unsigned char* gblk, int bytes, int R, int W, unsigned long long* mbox, long long NB, long long* out,
                    int mode, unsigned long long* trp) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* blk = sm;
  double* xloc = (double*)(sm + ((bytes + 127) & ~127));
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) blk[i] = gblk[i];
  for (int i = threadIdx.x; i < 8192 + 1; i += blockDim.x) xloc[i] = i < 8192 ? 1.0 + 1e-4 * i : 0.0;
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const unsigned xb = opaque(smem_u32(xloc)), bs = opaque(smem_u32(blk));
  long long best[4] = {1LL << 60, 1LL << 60, 1LL << 60, 1LL << 60};
  for (int rep = 0; rep < 50; rep++) {
    // refill the mailboxes this slice reads (parity 0)
    for (long long i = lane; i < NB; i += 32) mbox[i] = 0x3FF0000000000000ull;
    for (int i = lane; i < bytes; i += 32) blk[i] = gblk[i];  // pre() rewrites the slice in place
    __syncwarp();
    __threadfence();
    long long t0 = clock64();
    const SliceAddr S(bs, R, W, mode == 0, lane);
    if (mode == 0) {
      BSlice B;
      B.pre(S, W, xb);
      long long t1 = clock64();
      unsigned long long* mbox_in = mbox + (size_t)(lane < R ? lane : 0) * ((W + 3) & ~3);
      B.poll(S, W, R, mbox_in);
      __syncwarp();
      long long t2 = clock64();
      if (rep == 49 && lane == 0) trp[1] = gtimer();
      B.post(S, W, xb, mbox_in, mbox, (unsigned)NB, (unsigned)NB, R, rep == 49 ? trp : nullptr);
      if (rep == 49) { __syncwarp(); if (lane == 0) trp[10] = gtimer(); }
      __syncwarp();
      long long t3 = clock64();
      best[0] = min(best[0], t1 - t0);
      best[1] = min(best[1], t2 - t1);
      best[2] = min(best[2], t3 - t2);
    } else {
      slice_interior(S, W, xb);
      __syncwarp();
      best[3] = min(best[3], clock64() - t0);
    }
  }
  if (lane == 0)
    for (int i = 0; i < 4; i++) out[i] = best[i];
}
}  // namespace pobk

int main() {
  using namespace pobk;
  const int R = 32, W = 24;
  std::mt19937 rng(7);
  for (int mode = 0; mode < 2; mode++) {
    const bool bnd = mode == 0;
    SliceLayout L(R, W, bnd);
    std::vector<unsigned char> h(L.bytes, 0);
    double* val = (double*)h.data();
    double* fv = (double*)(h.data() + L.o_f);
    unsigned* col = (unsigned*)(h.data() + L.o_col);
    unsigned* mout = (unsigned*)(h.data() + L.o_mout);
    unsigned short* len = (unsigned short*)(h.data() + L.o_len);
    for (int r = 0; r < R; r++) {
      len[r] = (unsigned short)(W - (r * 6) / R);
      fv[r] = 1.0 + r;
      for (int j = 0; j < W; j++) {
        const int e = j * R + r;
        if (j < len[r]) {
          val[e] = 0.5 + (rng() % 1000) * 1e-3;
          const bool sh = bnd && (rng() % 2 == 0);
          col[e] = sh ? (0x80000000u | (unsigned)(rng() % 100000)) : (unsigned)(rng() % 8192);
          if (bnd) mout[e] = sh ? (unsigned)(rng() % (((W + 3) & ~3) * R)) : 0u;
        } else {
          col[e] = 8192;  // zero slot
        }
      }
    }
    unsigned char* d;
    unsigned long long* mb;
    long long* out;
    unsigned long long* trp;
    cudaMalloc(&trp, 16 * 8);
    cudaMalloc(&d, h.size());
    cudaMalloc(&mb, 2 * ((W + 3) & ~3) * R * 8);
    cudaMalloc(&out, 32);
    cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
    const size_t sm = ((h.size() + 127) & ~127) + 8193 * 8;
    cudaFuncSetAttribute(mb6, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    mb6<<<1, 128, sm>>>(d, (int)h.size(), R, W, mb, ((W + 3) & ~3) * R, out, mode, trp);
    cudaError_t e = cudaDeviceSynchronize();
    long long o[4];
    cudaMemcpy(o, out, 32, cudaMemcpyDeviceToHost);
    unsigned long long ht[16]; cudaMemcpy(ht, trp, 128, cudaMemcpyDeviceToHost);
    if (mode == 0) fprintf(stderr, "  post stamps (ns): sum %lld ddiv %lld pass2 %lld\n", (long long)(ht[2] - ht[1]), (long long)(ht[9] - ht[2]), (long long)(ht[10] - ht[9]));
    if (mode == 0) fprintf(stderr, "boundary slice R=%d W=%d: pre %lld  poll %lld  post %lld cycles (%s)\n", R, W, o[0], o[1], o[2], cudaGetErrorString(e));
    else fprintf(stderr, "interior slice R=%d W=%d: %lld cycles (%s)\n", R, W, o[3], cudaGetErrorString(e));
  }
  return 0;
}
