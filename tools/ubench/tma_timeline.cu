// Streaming TMA ring from one thread: record when each load is issued and
// when its wait returns (first 40 iterations), S stages.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "ptx.cuh"
using namespace atmm::ptx;
constexpr int COLS = 4096, ROWS = 1024;
__global__ void k(const __grid_constant__ CUtensorMap m, int S, int variant, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[16];
  const int bb = 16384, iters = 40;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const long long t0 = clock64();
  for (int i = 0; i < iters + S; ++i) {
    if (i >= S) {
      mbar_wait(&full[i % S], ((i - S) / S) & 1);
      out[2 * (i - S) + 1] = clock64() - t0;
    }
    if (i < iters) {
      const int s = i % S;
      mbar_arrive_expect_tx(&full[s], bb);
      const int col = variant == 0 ? (i % 64) * 64 : ((i * 17) % 64) * 64;
      const int row = variant == 0 ? 0 : ((i * 37) % 7) * 128;
      tma_load_2d(sm + s * bb, &m, &full[s], col, row);
      out[2 * i] = clock64() - t0;
    }
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
  cudaMalloc(&d, 8 * 100);
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[2] = {COLS, ROWS}, str[1] = {COLS * 2};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  ((EncodeFn)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int variant = 0; variant < 2; ++variant)
    for (int S : {4, 8}) {
      for (int rep = 0; rep < 3; ++rep) k<<<1, 32, 200 * 1024>>>(m, S, variant, d);
      long long h[100];
      cudaMemcpy(h, d, 8 * 80, cudaMemcpyDeviceToHost);
      printf("variant %d S=%d\n issue: ", variant, S);
      for (int i = 0; i < 24; ++i) printf("%lld ", h[2 * i]);
      printf("\n done : ");
      for (int i = 0; i < 24; ++i) printf("%lld ", h[2 * i + 1]);
      printf("\n");
    }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
