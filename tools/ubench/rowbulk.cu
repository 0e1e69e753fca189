// Microbenchmark: chip-wide HBM throughput of SCATTERED ROW loads into shared
// memory with every SM streaming (one CTA per SM), by load mechanism and
// contiguous piece size -- the data-movement ceiling of the split bypass path
// (cfg3 / cfg5: X and Y rows of 8-10 KB gathered by segment).
//   bulk  : cp.async.bulk 1-D global -> shared, one request per row piece of
//           `piece` bytes, issued by `issuers` threads, S-stage ring of
//           `per_stage` pieces (mbarrier expect_tx per stage)
//   lsu   : 16-byte cp.async (LDGSTS) by 256 threads, same pieces and ring
// Source: 1 GiB bf16 matrix of 8 KiB rows (>> L2), random row order.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2411_00915_b200/csrc -o rowbulk rowbulk.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#include "ptx.cuh"
using namespace atmm::ptx;

constexpr int ROW_BYTES = 8192;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr int64_t NROWS = (1ll << 30) / ROW_BYTES;

__global__ void __launch_bounds__(256, 1) k_bulk(const uint8_t* src, const int* rows, int piece, int per_stage,
                                                 int stages, int iters, int issuers, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bars[16];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < stages; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int pieces_per_row = ROW_BYTES / piece;
  const uint32_t stage_bytes = static_cast<uint32_t>(piece * per_stage);
  const unsigned long long t0 = gtimer();
  const int nthr = ((issuers + 31) / 32) * 32;  // whole warps take part in the syncs
  if (tid < nthr) {
    for (int it = 0; it < iters; ++it) {
      const int st = it % stages;
      if (it >= stages) {
        if (tid == 0) mbar_wait(&bars[st], static_cast<uint32_t>(((it / stages) - 1) & 1));
        asm volatile("bar.sync 1, %0;" ::"r"(nthr));
      }
      if (tid == 0) mbar_arrive_expect_tx(&bars[st], stage_bytes);
      asm volatile("bar.sync 1, %0;" ::"r"(nthr));
      for (int q = tid; tid < issuers && q < per_stage; q += issuers) {
        const int g = (blockIdx.x * 7919 + it * per_stage + q);
        const int row = rows[g % (1 << 20)];
        const int pc = g % pieces_per_row;
        bulk_g2s(sm + st * stage_bytes + q * piece, src + static_cast<int64_t>(row) * ROW_BYTES + pc * piece,
                 static_cast<uint32_t>(piece), &bars[st]);
      }
    }
    if (tid == 0) {
      for (int it = iters - stages; it < iters; ++it) {
        if (it >= 0) mbar_wait(&bars[it % stages], static_cast<uint32_t>((it / stages) & 1));
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    out[blockIdx.x * 2] = t0;
    out[blockIdx.x * 2 + 1] = gtimer();
  }
}

__global__ void __launch_bounds__(256, 1) k_lsu(const uint8_t* src, const int* rows, int piece, int per_stage,
                                                int stages, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int tid = threadIdx.x;
  const int pieces_per_row = ROW_BYTES / piece;
  const int chunks = piece / 16;
  const uint32_t stage_bytes = static_cast<uint32_t>(piece * per_stage);
  const unsigned long long t0 = gtimer();
  for (int it = 0; it < iters; ++it) {
    const int st = it % stages;
    for (int c = tid; c < per_stage * chunks; c += 256) {
      const int q = c / chunks, k = c % chunks;
      const int g = (blockIdx.x * 7919 + it * per_stage + q);
      const int row = rows[g % (1 << 20)];
      const int pc = g % pieces_per_row;
      cp_async16(smem_u32(sm + st * stage_bytes + q * piece + k * 16),
                 src + static_cast<int64_t>(row) * ROW_BYTES + pc * piece + k * 16, 16u);
    }
    cp_async_commit();
    if (it >= stages - 1) cp_async_wait<7>(stages - 1);
  }
  cp_async_wait<0>(0);
  __syncthreads();
  if (tid == 0) {
    out[blockIdx.x * 2] = t0;
    out[blockIdx.x * 2 + 1] = gtimer();
  }
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* src;
  cudaMalloc(&src, static_cast<size_t>(NROWS) * ROW_BYTES);
  cudaMemset(src, 1, static_cast<size_t>(NROWS) * ROW_BYTES);
  std::vector<int> hr(1 << 20);
  std::mt19937 g(1);
  for (auto& v : hr) v = static_cast<int>(g() % NROWS);
  int* rows;
  cudaMalloc(&rows, hr.size() * 4);
  cudaMemcpy(rows, hr.data(), hr.size() * 4, cudaMemcpyHostToDevice);
  unsigned long long* out;
  cudaMalloc(&out, sms * 16);
  std::vector<unsigned long long> h(sms * 2);
  const size_t smem = 200 * 1024;
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  cudaFuncSetAttribute(k_lsu, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  auto report = [&](const char* name, int piece, int per_stage, int stages, int iters, int issuers) {
    cudaMemcpy(h.data(), out, sms * 16, cudaMemcpyDeviceToHost);
    unsigned long long a = ~0ull, b = 0;
    for (int i = 0; i < sms; ++i) {
      a = std::min(a, h[2 * i]);
      b = std::max(b, h[2 * i + 1]);
    }
    const double bytes = double(sms) * iters * per_stage * piece;
    const double ns = double(b - a);
    printf("%-5s piece %5d B  stage %6d B x %2d  issuers %3d : %7.1f GB/s chip, %5.1f B/cycle/SM @1.965GHz\n", name,
           piece, piece * per_stage, stages, issuers, bytes / ns, bytes / ns / sms / 1.965);
  };
  for (int piece : {512, 1024, 2048, 4096, 8192}) {
    const int stage_bytes = 32768;
    const int per_stage = stage_bytes / piece;
    const int stages = 6;
    const int iters = 400;
    for (int issuers : {1, 32, 128}) {
      if (issuers > per_stage && issuers != 1) continue;
      k_bulk<<<sms, 256, smem>>>(src, rows, piece, per_stage, stages, iters, issuers, out);
      cudaDeviceSynchronize();
      k_bulk<<<sms, 256, smem>>>(src, rows, piece, per_stage, stages, iters, issuers, out);
      cudaDeviceSynchronize();
      report("bulk", piece, per_stage, stages, iters, issuers);
    }
    k_lsu<<<sms, 256, smem>>>(src, rows, piece, per_stage, stages, iters, out);
    cudaDeviceSynchronize();
    k_lsu<<<sms, 256, smem>>>(src, rows, piece, per_stage, stages, iters, out);
    cudaDeviceSynchronize();
    report("lsu", piece, per_stage, stages, iters, 256);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
