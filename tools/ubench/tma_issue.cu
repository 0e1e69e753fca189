// Pure issue cost of TMA instructions from one thread: N loads back to back on
// one mbarrier, clock before / after the issue loop, then wait.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"
using namespace atmm::ptx;
constexpr int COLS = 4096, ROWS = 1024;
__global__ void k(const __grid_constant__ CUtensorMap m, const uint16_t* src, int variant, int N, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint64_t bars[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(&bars[i], 1);
    mbar_init(&bar, 1);
    fence_mbar_init();
    if (variant & 1) tma_prefetch_desc(&m);
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int rep = 0; rep < 3; ++rep) {
    const int bb = (variant & 4) ? 2048 : 16384;
    if (variant & 8) {
      const long long t0 = clock64();
      for (int i = 0; i < N; ++i) {
        mbar_arrive_expect_tx(&bars[i], 16384);
        tma_load_2d(sm + i * 16384, &m, &bars[i], (i % 64) * 64, rep * 128);
      }
      const long long t1 = clock64();
      for (int i = 0; i < N; ++i) mbar_wait(&bars[i], rep & 1);
      const long long t2 = clock64();
      out[2 * rep] = t1 - t0;
      out[2 * rep + 1] = t2 - t0;
      continue;
    }
    if (variant & 32) {  // expect_tx + load + wait on an already-complete barrier
      __shared__ uint64_t done_bar;
      if (rep == 0) { mbar_init(&done_bar, 1); fence_mbar_init(); }
      const long long t0 = clock64();
      for (int i = 0; i < N; ++i) {
        mbar_arrive_expect_tx(&bars[i], 16384);
        tma_load_2d(sm + i * 16384, &m, &bars[i], (i % 64) * 64, rep * 128);
        mbar_wait(&done_bar, 1);
      }
      const long long t1 = clock64();
      for (int i = 0; i < N; ++i) mbar_wait(&bars[i], rep & 1);
      const long long t2 = clock64();
      out[2 * rep] = t1 - t0;
      out[2 * rep + 1] = t2 - t0;
      continue;
    }
    if (variant & 64) {  // expect_tx + load + clock read + shared store
      __shared__ long long sink[16];
      const long long t0 = clock64();
      for (int i = 0; i < N; ++i) {
        mbar_arrive_expect_tx(&bars[i], 16384);
        tma_load_2d(sm + i * 16384, &m, &bars[i], (i % 64) * 64, rep * 128);
        sink[i] = clock64();
      }
      const long long t1 = clock64();
      for (int i = 0; i < N; ++i) mbar_wait(&bars[i], rep & 1);
      const long long t2 = clock64();
      out[2 * rep] = t1 - t0;
      out[2 * rep + 1] = t2 - t0 + sink[0] * 0;
      continue;
    }
    if (variant & 16) {  // expect_tx only
      const long long t0 = clock64();
      for (int i = 0; i < N; ++i) mbar_arrive_expect_tx(&bars[i], 0);
      const long long t1 = clock64();
      out[2 * rep] = t1 - t0;
      out[2 * rep + 1] = t1 - t0;
      continue;
    }
    mbar_arrive_expect_tx(&bar, bb * N);
    const long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
      if (variant & 2) bulk_g2s(sm + i * bb, src + size_t(i) * 8192 + rep * 64, bb, &bar);
      else tma_load_2d(sm + i * 16384, &m, &bar, (i % 64) * 64, rep * 128);
    }
    const long long t1 = clock64();
    mbar_wait(&bar, rep & 1);
    const long long t2 = clock64();
    out[2 * rep] = t1 - t0;
    out[2 * rep + 1] = t2 - t0;
  }
}
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  uint16_t* src;
  cudaMalloc(&src, size_t(ROWS) * COLS * 2);
  cudaMemset(src, 1, size_t(ROWS) * COLS * 2);
  long long* d;
  cudaMalloc(&d, 8 * 16);
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[2] = {COLS, ROWS}, str[1] = {COLS * 2};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  ((EncodeFn)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int variant : {8, 32, 64})
    for (int N : {1, 4, 12}) {
      for (int r = 0; r < 2; ++r) k<<<1, 32, 220 * 1024>>>(m, src, variant, N, d);
      long long h[6];
      cudaMemcpy(h, d, 48, cudaMemcpyDeviceToHost);
      printf("variant %2d N=%2d: issue %5lld cyc (%.0f/instr)  done %5lld cyc   [rep0 issue %lld done %lld]\n", variant, N, h[4],
             double(h[4]) / N, h[5], h[0], h[1]);
    }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
