// Issue S TMA 2-D box loads (64 x R, SW128) back to back from one thread, each
// on its own mbarrier, then wait for all: cycles vs S separates latency from
// per-SM issue/service throughput.  Also the same with S issuing lanes.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "ptx.cuh"
using namespace atmm::ptx;
constexpr int COLS = 4096, ROWS = 2048;

__global__ void k(const __grid_constant__ CUtensorMap m, int S, int box_rows, int lanes, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[32];
  const int bb = box_rows * 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 32; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  for (int rep = 0; rep < 3; ++rep) {
    __syncwarp();
    long long t0 = clock64();
    if (lanes == 1) {
      if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
          mbar_arrive_expect_tx(&bar[s], bb);
          tma_load_2d(sm + s * bb, &m, &bar[s], ((s + rep * S) % 64) * 64, (blockIdx.x * 256 + rep * 512) % (ROWS - box_rows));
        }
      }
    } else if (threadIdx.x < S) {
      const int s = threadIdx.x;
      mbar_arrive_expect_tx(&bar[s], bb);
      tma_load_2d(sm + s * bb, &m, &bar[s], ((s + rep * S) % 64) * 64, (blockIdx.x * 256 + rep * 512) % (ROWS - box_rows));
    }
    if (threadIdx.x == 0) {
      for (int s = 0; s < S; ++s) mbar_wait(&bar[s], rep & 1);
      if (blockIdx.x == 0) out[rep] = clock64() - t0;
    }
    __syncthreads();
  }
}
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  uint16_t* src;
  cudaMalloc(&src, size_t(ROWS) * COLS * 2);
  std::vector<uint16_t> h(size_t(ROWS) * COLS, 0x3f80);
  cudaMemcpy(src, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  long long* d;
  cudaMalloc(&d, 64);
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int br : {32, 64, 128, 256}) {
    CUtensorMap m;
    cuuint64_t dims[2] = {COLS, ROWS}, str[1] = {COLS * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)br}, es[2] = {1, 1};
    ((EncodeFn)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int lanes : {1, 32})
      for (int S : {1, 2, 4, 8, 12}) {
        if (S * br * 128 > 200 * 1024) continue;
        for (int G : {1, 148}) {
          k<<<G, 32, 220 * 1024>>>(m, S, br, lanes, d);
          long long o[3];
          cudaMemcpy(o, d, 24, cudaMemcpyDeviceToHost);
          printf("box 64x%-3d lanes %2d S=%2d G=%3d: %6lld cyc (warm %6lld)  %.1f B/cyc\n", br, lanes, S, G, o[0], o[2],
                 double(S) * br * 128 / o[2]);
        }
      }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
