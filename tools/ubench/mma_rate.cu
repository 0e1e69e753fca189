// Back-to-back tcgen05.mma issue rate from one elected thread, one commit at
// the end: the cost per MMA of the fused bypass's shapes.
//   shape 0: shrink   M=128 N=r   K=16, A K-major SW128, B interleave
//   shape 1: expand   M=128 N=rows K=16, A and B interleave (swap-AB)
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"
using namespace atmm::ptx;

__global__ void k(long long* out, int shape, int n, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tslot, 256);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tb = tslot;
  const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 65536);
  long long t0 = clock64(), t1 = 0, t2 = 0;
  if (threadIdx.x < 32) {
    if (elect_one()) {
      const uint32_t idesc = idesc_bf16(128, n);
      if (shape >= 2) {  // precomputed descriptors, advanced by adds only
        const uint64_t ad0 = shape == 2 ? smem_desc(a0, 16u, 1024u, kLayoutSW128) : smem_desc(a0, 128u, 256u, kLayoutNone);
        const uint64_t bd0 = shape == 2 ? smem_desc(b0, 128u, 1024u, kLayoutNone) : smem_desc(b0, 128u, 256u, kLayoutNone);
        for (int i = 0; i < iters; ++i) {
          const uint64_t ad = ad0 + static_cast<uint64_t>(shape == 2 ? (i & 3) * 2 : (i & 7) * 256);
          const uint64_t bd = bd0 + static_cast<uint64_t>(shape == 2 ? (i & 3) * 16 : 0);
          mma_bf16(tb, ad, bd, idesc, i > 0 ? 1u : 0u);
        }
      } else
      for (int i = 0; i < iters; ++i) {
        uint64_t ad, bd;
        if (shape == 0) {
          ad = smem_desc(a0 + (i & 3) * 32u + ((i >> 2) & 7) * 16384u, 16u, 1024u, kLayoutSW128);
          bd = smem_desc(b0 + (i & 3) * 256u, 128u, 1024u, kLayoutNone);
        } else {
          ad = smem_desc(a0 + (i & 7) * 4096u, 128u, 256u, kLayoutNone);
          bd = smem_desc(b0, 128u, 256u, kLayoutNone);
        }
        mma_bf16(tb, ad, bd, idesc, i > 0 ? 1u : 0u);
      }
      t1 = clock64();
      mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    t2 = clock64();
  }
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tb, 256); }
}

int main() {
  long long* d; cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int shape = 0; shape < 4; ++shape)
    for (int n : {16, 32, 64, 128, 256})
      for (int iters : {8, 32}) {
        long long h[2] = {0, 0};
        for (int rep = 0; rep < 3; ++rep) {
          k<<<1, 128, 200 * 1024>>>(d, shape, n, iters);
          cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        }
        printf("shape %d (%s) N=%3d iters %2d: issue %5lld cyc (%.1f/mma), done %5lld cyc (%.1f/mma)\n", shape,
               shape == 0 ? "shrink" : shape == 1 ? "expand" : shape == 2 ? "shrink-pre" : "expand-pre", n, iters, h[0], (double)h[0] / iters, h[1], (double)h[1] / iters);
      }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
