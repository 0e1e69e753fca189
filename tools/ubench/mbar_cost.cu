// Cost of an mbarrier wait whose phase is already complete (fresh barrier,
// parity 1), from one thread: try_wait vs test_wait, 16 different barriers.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"
using namespace atmm::ptx;
__device__ __forceinline__ bool test1(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(phase) : "memory");
  return ok;
}
__device__ __forceinline__ bool try1(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(phase) : "memory");
  return ok;
}
__global__ void k(long long* out) {
  __shared__ uint64_t bars[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < 16; ++i) acc += test1(&bars[i], 1);
  long long t1 = clock64();
  for (int i = 0; i < 16; ++i) acc += try1(&bars[i], 1);
  long long t2 = clock64();
  for (int i = 0; i < 16; ++i) mbar_wait(&bars[i], 1);
  long long t3 = clock64();
  for (int i = 0; i < 16; ++i) acc += test1(&bars[i], 0);  // incomplete phase: false
  long long t4 = clock64();
  for (int i = 0; i < 16; ++i) acc += try1(&bars[i], 0);  // incomplete: may suspend then false
  long long t5 = clock64();
  for (int i = 0; i < 16; ++i) mbar_arrive(&bars[i]);
  long long t6 = clock64();
  for (int i = 0; i < 16; ++i) mbar_wait(&bars[i], 0);  // now complete
  long long t7 = clock64();
  out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4; out[5] = t6 - t5; out[6] = t7 - t6;
  out[7] = acc;
}
int main() {
  long long* d;
  cudaMalloc(&d, 64);
  for (int r = 0; r < 3; ++r) k<<<1, 32>>>(d);
  long long h[8];
  cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
  printf("16x test_wait(complete) %lld cyc\n16x try_wait(complete) %lld\n16x mbar_wait(complete) %lld\n16x test_wait(incomplete) %lld\n"
         "16x try_wait(incomplete) %lld\n16x arrive %lld\n16x mbar_wait(just completed) %lld\nacc %lld\n", h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
}
