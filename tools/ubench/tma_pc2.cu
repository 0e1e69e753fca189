// Bisect the slow producer loop: 12 loads into 12 stages (no stage reuse).
//  mode 0: producer only (other warp idle)
//  mode 1: + consumer warp polling full[] with try_wait
//  mode 2: + consumer warp polling with test_wait + nanosleep(128)
//  mode 3: producer only, coordinates like tma_pc (row modulo)
//  mode 4: producer waits empty[s] (fresh, parity 1) before each load
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"
using namespace atmm::ptx;
constexpr int COLS = 4096, ROWS = 1024;
__global__ void k(const __grid_constant__ CUtensorMap m, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[12], empty[12];
  __shared__ long long tiss[12], tdone[12];
  if (threadIdx.x == 0) {
    for (int s = 0; s < 12; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    fence_mbar_init();
  }
  __syncthreads();
  const long long t0 = clock64();
  if (mode >= 5) {
    const int S = 4, iters = 64;
    if (threadIdx.x == 0) {
      if (mode == 6) tma_prefetch_desc(&m);
      for (int i = 0; i < iters; ++i) {
        const int s = i % S;
        mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[s], 16384);
        tma_load_2d(sm + s * 16384, &m, &full[s], (i % 64) * 64, 0);
        if (i < 12) tiss[i] = clock64() - t0;
      }
    } else if (threadIdx.x == 32) {
      for (int i = 0; i < iters; ++i) {
        const int s = i % S;
        mbar_wait(&full[s], (i / S) & 1);
        if (i < 12) tdone[i] = clock64() - t0;
        mbar_arrive(&empty[s]);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) for (int i = 0; i < 12; ++i) { out[i] = tiss[i]; out[12 + i] = tdone[i]; }
    return;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 12; ++i) {
      if (mode == 4) mbar_wait(&empty[i], 1);
      mbar_arrive_expect_tx(&full[i], 16384);
      const int row = mode == 3 ? ((i / 64) * 128 + blockIdx.x * 128) % (ROWS - 128) : 0;
      tma_load_2d(sm + i * 16384, &m, &full[i], (i % 64) * 64, row);
      tiss[i] = clock64() - t0;
    }
  } else if (threadIdx.x == 32 && (mode == 1 || mode == 2)) {
    for (int i = 0; i < 12; ++i) {
      if (mode == 1) mbar_wait(&full[i], 0);
      else mbar_wait_sleep(&full[i], 0, 128);
      tdone[i] = clock64() - t0;
    }
  }
  if (threadIdx.x == 0 && mode != 1 && mode != 2) {
    for (int i = 0; i < 12; ++i) { mbar_wait(&full[i], 0); tdone[i] = clock64() - t0; }
  }
  __syncthreads();
  if (threadIdx.x == 0) for (int i = 0; i < 12; ++i) { out[i] = tiss[i]; out[12 + i] = tdone[i]; }
}
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  uint16_t* src;
  cudaMalloc(&src, size_t(ROWS) * COLS * 2);
  cudaMemset(src, 1, size_t(ROWS) * COLS * 2);
  long long* d;
  cudaMalloc(&d, 8 * 24);
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[2] = {COLS, ROWS}, str[1] = {COLS * 2};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  ((EncodeFn)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int mode = 4; mode < 7; ++mode) {
    for (int r = 0; r < 3; ++r) k<<<1, 64, 220 * 1024>>>(m, mode, d);
    long long h[24];
    cudaMemcpy(h, d, 8 * 24, cudaMemcpyDeviceToHost);
    printf("mode %d issue:", mode);
    for (int i = 0; i < 12; ++i) printf(" %lld", h[i]);
    printf("\n       done :");
    for (int i = 0; i < 12; ++i) printf(" %lld", h[12 + i]);
    printf("\n");
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
