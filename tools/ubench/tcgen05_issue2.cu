// Issue cost of tcgen05.mma + commit: single divergent lane vs converged warp
// with elect.sync, descriptors computed per iteration (as in the kernel).
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"
using namespace atmm::ptx;

__global__ void k(long long* out, int mode, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tslot;
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); mbar_init(&bar[1], 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tslot, 256);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tb = tslot;
  const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 16384);
  long long t0 = clock64();
  if (mode == 0) {  // single lane (divergent), like the kernel today
    if (threadIdx.x == 0) {
      for (int i = 0; i < iters; ++i) {
        mbar_wait(&bar[1], 1);  // already-complete wait (parity trick)
        tc_fence_after();
        const uint64_t ad = smem_desc(a0 + (i & 3) * 32u, 16u, 1024u, kLayoutSW128);
        const uint64_t bd = smem_desc(b0 + (i & 3) * 256u, 128u, 1024u, kLayoutNone);
        mma_bf16(tb + (i & 3) * 64, ad, bd, idesc_bf16(128, 64), 0);
        mma_commit(&bar[0]);
      }
    }
  } else {  // whole warp converged, elect one to issue
    if (threadIdx.x < 32) {
      for (int i = 0; i < iters; ++i) {
        mbar_wait(&bar[1], 1);
        tc_fence_after();
        const uint64_t ad = smem_desc(a0 + (i & 3) * 32u, 16u, 1024u, kLayoutSW128);
        const uint64_t bd = smem_desc(b0 + (i & 3) * 256u, 128u, 1024u, kLayoutNone);
        if (elect_one()) {
          mma_bf16(tb + (i & 3) * 64, ad, bd, idesc_bf16(128, 64), 0);
          mma_commit(&bar[0]);
        }
        __syncwarp();
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tb, 256); }
}

int main() {
  long long* d; cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int mode = 0; mode < 2; ++mode)
    for (int rep = 0; rep < 2; ++rep) {
      k<<<1, 128, 64 * 1024>>>(d, mode, 64);
      long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      if (rep) printf("mode %d (%s): %lld cyc per (wait + mma + commit)\n", mode, mode ? "converged+elect" : "single lane", h / 64);
    }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
