// Microbenchmark: per-SM / chip load throughput of scattered-row loads into
// shared memory on sm_100a: TMA tile::gather4 (4 rows x 128 B per request),
// TMA 2-D tile (box 64 x 4 rows), and cp.async 16 B (LDGSTS) with manual
// 128-byte swizzle.  Rows are random (gather) over a 64 MiB bf16 matrix.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include "ptx.cuh"
using namespace atmm::ptx;

constexpr int D = 4096;   // columns (bf16)
constexpr int N = 8192;   // rows -> 64 MiB
constexpr int BLK = 16384;

__global__ void __launch_bounds__(128) k_gather4(const __grid_constant__ CUtensorMap m, const int* rows, int reqs,
                                                 long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    if (lane == 0) mbar_arrive_expect_tx(&bar, reqs * 512u);
    __syncwarp();
    for (int r = lane; r < reqs; r += 32) {
      const int* rr = rows + ((blockIdx.x * 977 + r * 4) % (N - 4));
      const int col = (r * 64) % D;
      tma_gather4(sm + (r % 32) * 512 + ((r / 32) % 8) * BLK, &m, &bar, col, rr[0], rr[1], rr[2], rr[3]);
    }
    mbar_wait(&bar, 0);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

__global__ void __launch_bounds__(128) k_tile(const __grid_constant__ CUtensorMap m, int reqs, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  long long t0 = clock64();
  if (threadIdx.x < 32) {
    if (lane == 0) mbar_arrive_expect_tx(&bar, reqs * 512u);
    __syncwarp();
    for (int r = lane; r < reqs; r += 32) {
      const int row = ((blockIdx.x * 977 + r * 131) * 4) % (N - 4);
      tma_load_2d(sm + (r % 32) * 512 + ((r / 32) % 8) * BLK, &m, &bar, (r * 64) % D, row);
    }
    mbar_wait(&bar, 0);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

// cp.async: each warp moves 4 rows x 128 B per "request" (same bytes as gather4)
__global__ void __launch_bounds__(128) k_cpasync(const uint16_t* x, const int* rows, int reqs, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long t0 = clock64();
  for (int r = warp; r < reqs; r += 4) {
    const int* rr = rows + ((blockIdx.x * 977 + r * 4) % (N - 4));
    const int i = lane >> 3, c = lane & 7;
    const int col = (r * 64) % D;
    const uint16_t* src = x + (size_t)rr[i] * D + col + c * 8;
    uint32_t dst = smem_u32(sm + (r % 32) * 512 + ((r / 32) % 8) * BLK + i * 128 + ((c ^ i) << 4));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src) : "memory");
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  uint16_t* x; cudaMalloc(&x, (size_t)N * D * 2); cudaMemset(x, 0, (size_t)N * D * 2);
  std::vector<int> h(N); std::mt19937 g(1); for (int i = 0; i < N; ++i) h[i] = g() % N;
  int* rows; cudaMalloc(&rows, N * 4); cudaMemcpy(rows, h.data(), N * 4, cudaMemcpyHostToDevice);
  long long* out; cudaMalloc(&out, 1024 * 8);
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)p;
  CUtensorMap mg, mt;
  cuuint64_t dims[2] = {D, N}, str[1] = {D * 2};
  cuuint32_t boxg[2] = {64, 1}, boxt[2] = {64, 4}, es[2] = {1, 1};
  enc(&mg, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, str, boxg, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&mt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, str, boxt, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int smem = 8 * BLK;
  cudaFuncSetAttribute(k_gather4, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int grid : {1, 148}) {
    for (int reqs : {64, 256, 1024}) {
      for (int kind = 0; kind < 3; ++kind) {
        float best = 1e9; long long cyc = 0;
        for (int rep = 0; rep < 4; ++rep) {
          cudaEventRecord(e0);
          if (kind == 0) k_gather4<<<grid, 128, smem>>>(mg, rows, reqs, out);
          if (kind == 1) k_tile<<<grid, 128, smem>>>(mt, reqs, out);
          if (kind == 2) k_cpasync<<<grid, 128, smem>>>(x, rows, reqs, out);
          cudaEventRecord(e1); cudaEventSynchronize(e1);
          float ms; cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) { best = ms; cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost); }
        }
        const double bytes = (double)grid * reqs * 512;
        printf("grid %3d reqs %5d %-9s: CTA0 %7lld cyc (%.1f B/cyc/SM)  kernel %.2f us  chip %.0f GB/s\n", grid, reqs,
               kind == 0 ? "gather4" : kind == 1 ? "tile2d" : "cp.async", cyc, reqs * 512.0 / cyc, best * 1e3,
               bytes / (best * 1e-3) / 1e9);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
