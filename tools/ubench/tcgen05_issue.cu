// Microbenchmark: issue cost of tcgen05.mma / tcgen05.commit on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2411_00915_b200/csrc tcgen05_issue.cu
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"
using namespace atmm::ptx;

__global__ void k(long long* out, int mode, int iters, int n) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tslot, 256);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 16384);
    uint64_t ad = smem_desc(a0, 16u, 1024u, kLayoutSW128);
    uint64_t bd = smem_desc(b0, 128u, 1024u, kLayoutNone);
    uint32_t id = idesc_bf16(128, n);
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      mma_bf16(tb, ad, bd, id, i > 0);
      if (mode >= 1) mma_commit(&bar);
      if (mode == 2) { mbar_wait(&bar, ph); ph ^= 1; }
    }
    long long t1 = clock64();
    if (mode == 0) { mma_commit(&bar); mbar_wait(&bar, 0); }
    if (mode == 1) { /* drain: wait for last phase */ }
    long long t2 = clock64();
    out[0] = t1 - t0; out[1] = t2 - t0;
  }
  __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc(tb, 256); }
}

int main() {
  long long* d; cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int n : {16, 64, 128}) {
    for (int mode = 0; mode < 3; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        k<<<1, 128, 64 * 1024>>>(d, mode, 64, n);
        long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        if (rep == 1) printf("N=%3d mode=%d (0: mma only, 1: mma+commit, 2: mma+commit+wait): issue %lld cyc/iter, total %lld cyc/iter\n",
                             n, mode, h[0] / 64, h[1] / 64);
      }
    }
  }
  cudaError_t e = cudaDeviceSynchronize(); printf("%s\n", cudaGetErrorString(e));
}
