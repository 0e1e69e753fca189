// Microbenchmark: time for a one-shot CTA to land `rows` scattered row slices
// of `slice` bytes from each of two HBM matrices (the fused bypass's X and Y
// loads at cfg2: 32 rows x 1 KiB x 2 per CTA) into shared memory, for the
// load mechanisms available on sm_100a.  Reports the kernel span (min CTA
// start -> max CTA done, %globaltimer) and the chip-wide rate it implies.
//   m0 gather4    : TMA tile::gather4, 4 rows x 128 B per request, W issuing warps
//   m1 bulk       : cp.async.bulk 1-D, one request per row slice, W issuing warps
//   m2 cp.async   : 16-byte LDGSTS by all 8 warps, mbarrier completion
//   m3 ldg        : 16-byte LDG into registers by all 8 warps, then STS
//   m4 bulk2      : as m1, the slice split over two requests per row
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <algorithm>
#include "ptx.cuh"
using namespace atmm::ptx;

constexpr int D = 8192;      // bf16 columns (16 KiB rows)
constexpr int N = 32768;     // rows -> 512 MiB per matrix

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(256) k(const __grid_constant__ CUtensorMap mx, const __grid_constant__ CUtensorMap my,
                                         const uint16_t* x, const uint16_t* y, const int* rows, int method, int issuers,
                                         int nrows, int slice, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[2];
  const uint64_t t0 = gtimer();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], method == 2 ? 256 : 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int* rr = rows + (blockIdx.x * 64) % (N - 64);
  const int col0 = (blockIdx.x * (slice / 2)) % (D - slice / 2);
  const int total = nrows * slice;  // bytes per matrix
  uint8_t* sx = sm;
  uint8_t* sy = sm + total;
  if (method == 5) {
    // contiguous baseline: each CTA reads its own contiguous 2 x total bytes in 4 KiB requests
    if (warp == 0) {
      if (lane == 0) mbar_arrive_expect_tx(&bar[0], 2 * total);
      __syncwarp();
      const uint8_t* base = reinterpret_cast<const uint8_t*>(x) + (size_t)blockIdx.x * 2 * total;
      for (int t = lane; t < 2 * total / 4096; t += 32) bulk_g2s(sm + t * 4096, base + (size_t)t * 4096, 4096, &bar[0]);
    }
    mbar_wait(&bar[0], 0);
  } else if (method == 0 || method == 1 || method == 4) {
    if (warp < issuers) {
      if (warp == 0 && lane == 0) mbar_arrive_expect_tx(&bar[0], 2 * total);
      __syncwarp();
      // each issuing lane handles requests t = warp*32+lane, stride issuers*32
      const int per_row = slice / 128;
      if (method == 0) {
        const int reqs = (nrows / 4) * per_row;
        for (int t = warp * 32 + lane; t < 2 * reqs; t += issuers * 32) {
          const bool isy = t >= reqs;
          const int q = isy ? t - reqs : t;
          const int g = q / per_row, c = q % per_row;
          tma_gather4((isy ? sy : sx) + q * 512, isy ? &my : &mx, &bar[0], col0 + c * 64, rr[4 * g], rr[4 * g + 1],
                      rr[4 * g + 2], rr[4 * g + 3]);
        }
      } else {
        const int parts = method == 4 ? 2 : 1;
        const int psz = slice / parts;
        const int reqs = nrows * parts;
        for (int t = warp * 32 + lane; t < 2 * reqs; t += issuers * 32) {
          const bool isy = t >= reqs;
          const int q = isy ? t - reqs : t;
          const int r = q / parts, pp = q % parts;
          const uint16_t* src = (isy ? y : x) + (size_t)rr[r] * D + col0 + pp * psz / 2;
          bulk_g2s((isy ? sy : sx) + q * psz, src, psz, &bar[0]);
        }
      }
    }
    mbar_wait(&bar[0], 0);
  } else if (method == 2) {
    const int chunks = total / 16;  // per matrix
    for (int t = threadIdx.x; t < 2 * chunks; t += 256) {
      const bool isy = t >= chunks;
      const int q = isy ? t - chunks : t;
      const int r = q / (slice / 16), c = q % (slice / 16);
      const uint16_t* src = (isy ? y : x) + (size_t)rr[r] * D + col0 + c * 8;
      const uint32_t dst = smem_u32((isy ? sy : sx) + q * 16);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&bar[0])) : "memory");
    mbar_wait(&bar[0], 0);
  } else {
    const int chunks = total / 16;
    constexpr int kMax = 16;
    uint4 v[kMax];
    int n = 0;
#pragma unroll
    for (int j = 0; j < kMax; ++j) {
      const int t = threadIdx.x + j * 256;
      if (t < 2 * chunks) {
        const bool isy = t >= chunks;
        const int q = isy ? t - chunks : t;
        const int r = q / (slice / 16), c = q % (slice / 16);
        v[j] = __ldcs(reinterpret_cast<const uint4*>((isy ? y : x) + (size_t)rr[r] * D + col0 + c * 8));
        n = j + 1;
      }
    }
#pragma unroll
    for (int j = 0; j < kMax; ++j) {
      const int t = threadIdx.x + j * 256;
      if (j < n) *reinterpret_cast<uint4*>(sm + t * 16) = v[j];
    }
    __syncthreads();
  }
  __syncthreads();
  const uint64_t t1 = gtimer();
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = t0;
    out[2 * blockIdx.x + 1] = t1;
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  uint16_t *x, *y;
  cudaMalloc(&x, (size_t)N * D * 2);
  cudaMalloc(&y, (size_t)N * D * 2);
  cudaMemset(x, 0, (size_t)N * D * 2);
  cudaMemset(y, 0, (size_t)N * D * 2);
  std::vector<int> h(N);
  std::mt19937 g(1);
  for (int i = 0; i < N; ++i) h[i] = g() % N;
  int* rows;
  cudaMalloc(&rows, N * 4);
  cudaMemcpy(rows, h.data(), N * 4, cudaMemcpyHostToDevice);
  unsigned long long* out;
  cudaMalloc(&out, 4096 * 16);
  uint8_t* flush;
  cudaMalloc(&flush, 512 << 20);
  void* p;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)p;
  CUtensorMap mx, my;
  cuuint64_t dims[2] = {D, N}, str[1] = {D * 2};
  cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
  enc(&mx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&my, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, y, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* names[] = {"gather4", "bulk", "cp.async", "ldg", "bulk2", "contig"};
  struct Case { int grid, nrows, slice; };
  for (Case cs : {Case{128, 32, 1024}, Case{256, 32, 512}, Case{296, 32, 512}, Case{148, 64, 1024},
                  Case{296, 16, 1024}, Case{640, 64, 1024}}) {
    const int smem = 2 * cs.nrows * cs.slice;
    const double bytes = 2.0 * cs.grid * cs.nrows * cs.slice;
    printf("--- grid %d, %d rows x %d B x 2 matrices per CTA (%.1f MiB total)\n", cs.grid, cs.nrows, cs.slice,
           bytes / 1048576.0);
    for (int m = 0; m < 6; ++m) {
      for (int iss : {1, 2, 4, 8}) {
        if ((m == 2 || m == 3 || m == 5) && iss != 8) continue;
        if (m == 3 && 2 * cs.nrows * cs.slice / 16 > 256 * 16) continue;
        std::vector<double> spans;
        for (int rep = 0; rep < 5; ++rep) {
          cudaMemsetAsync(flush, rep, 512 << 20);
          k<<<cs.grid, 256, smem>>>(mx, my, x, y, rows, m, iss, cs.nrows, cs.slice, out);
          cudaDeviceSynchronize();
          std::vector<unsigned long long> o(2 * cs.grid);
          cudaMemcpy(o.data(), out, o.size() * 8, cudaMemcpyDeviceToHost);
          unsigned long long a = ~0ull, b = 0;
          for (int i = 0; i < cs.grid; ++i) {
            a = std::min(a, o[2 * i]);
            b = std::max(b, o[2 * i + 1]);
          }
          spans.push_back((b - a) * 1e-3);
        }
        std::sort(spans.begin(), spans.end());
        const double us = spans[2];
        printf("  %-9s issuers %d: span %6.2f us -> %6.0f GB/s\n", names[m], iss, us, bytes / (us * 1e-6) / 1e9);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
