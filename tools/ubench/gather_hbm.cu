// Scattered-row load throughput from HBM (1 GiB matrix, random rows) into
// smem on sm_100a, all SMs busy: TMA gather4 (512 B/request), TMA 1-D bulk
// (1 KiB row slices), cp.async 16 B with W issuing warps per CTA.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include "ptx.cuh"
using namespace atmm::ptx;

constexpr int D = 8192;            // bf16 columns (16 KiB rows)
constexpr int N = 65536;           // rows -> 1 GiB
constexpr int RING = 96 * 1024;    // smem ring reused cyclically

// Each CTA moves `bytes_per_cta` bytes; kind 0: gather4, 1: bulk 1 KiB, 2: cp.async
__global__ void __launch_bounds__(256) k(const __grid_constant__ CUtensorMap m, const uint16_t* x,
                                         const int* rows, int kind, int warps, long long bytes_per_cta,
                                         long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < 8) mbar_init(&bar[threadIdx.x], 1);
  fence_mbar_init();
  __syncthreads();
  long long t0 = clock64();
  const int nreq = (int)(bytes_per_cta / (kind == 0 ? 512 : kind == 1 ? 1024 : 512));
  if (kind < 2) {
    if (warp == 0) {
      // 8 batches on 8 barriers, each batch = nreq/8 requests (ring slots reused)
      const int per = nreq / 8;
      for (int b = 0; b < 8; ++b) {
        if (lane == 0) mbar_arrive_expect_tx(&bar[b], per * (kind == 0 ? 512u : 1024u));
        __syncwarp();
        for (int r = lane; r < per; r += 32) {
          const int q = b * per + r;
          const int* rr = rows + ((blockIdx.x * 7919 + q * 4) & (N - 1) & ~3);
          uint8_t* dst = sm + (q * (kind == 0 ? 512 : 1024)) % RING;
          if (kind == 0) {
            tma_gather4(dst, &m, &bar[b], (q * 64) % D, rr[0], rr[1], rr[2], rr[3]);
          } else {
            bulk_g2s(dst, x + (size_t)rr[0] * D + (q * 512) % D, 1024u, &bar[b]);
          }
        }
      }
      for (int b = 0; b < 8; ++b) mbar_wait(&bar[b], 0);
    }
  } else if (warp < warps) {
    // cp.async: 8 lanes per 128-byte row slice, 4 rows per warp-instruction
    const int per_warp = nreq / warps;  // 512-byte units
    for (int q = 0; q < per_warp; ++q) {
      const int u = warp * per_warp + q;
      const int* rr = rows + ((blockIdx.x * 7919 + u * 4) & (N - 1) & ~3);
      const int i = lane >> 3, c = lane & 7;
      const uint16_t* src = x + (size_t)rr[i] * D + (u * 64) % D + c * 8;
      uint32_t dst = smem_u32(sm + (u * 512) % RING + i * 128 + ((c ^ i) << 4));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src) : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
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
  long long* out; cudaMalloc(&out, 4096 * 8);
  uint8_t* flush; cudaMalloc(&flush, 512 << 20);
  void* p; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)p;
  CUtensorMap mg;
  cuuint64_t dims[2] = {D, N}, str[1] = {D * 2};
  cuuint32_t boxg[2] = {64, 1}, es[2] = {1, 1};
  enc(&mg, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, str, boxg, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, RING);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const long long per_cta = 1 << 20;  // 1 MiB per CTA
  struct Cfg { int kind, warps, ctas_per_sm; const char* name; };
  Cfg cfgs[] = {{0, 1, 1, "gather4  1cta"}, {0, 1, 2, "gather4  2cta"}, {1, 1, 1, "bulk1K   1cta"},
                {1, 1, 2, "bulk1K   2cta"}, {2, 1, 1, "cp.async 1w 1cta"}, {2, 2, 1, "cp.async 2w 1cta"},
                {2, 4, 1, "cp.async 4w 1cta"}, {2, 8, 1, "cp.async 8w 1cta"}, {2, 2, 2, "cp.async 2w 2cta"},
                {2, 4, 2, "cp.async 4w 2cta"}};
  for (auto c : cfgs) {
    const int grid = 148 * c.ctas_per_sm;
    const long long bytes = per_cta / c.ctas_per_sm;
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemsetAsync(flush, rep, 512 << 20);
      cudaEventRecord(e0);
      k<<<grid, 256, RING>>>(mg, x, rows, c.kind, c.warps, bytes, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("%-18s: %.1f us for %.0f MiB -> %.0f GB/s (%.1f B/cyc/SM @1.9GHz)\n", c.name, best * 1e3,
           grid * bytes / 1048576.0, grid * bytes / (best * 1e-3) / 1e9, grid * bytes / (best * 1e-3) / 148 / 1.9e9);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
