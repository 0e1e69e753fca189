// Per-SM throughput of TMA 2-D tiled loads (the layer-forward GEMM's X / W
// operand path) vs 1-D bulk copies, from an L2-resident source.
//   grid G CTAs; one thread per CTA streams `iters` boxes through an S-stage
//   smem ring (expect_tx + wait per stage); reports bytes / cycle / SM.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <dlfcn.h>
#include <vector>
#include "ptx.cuh"
using namespace atmm::ptx;

constexpr int COLS = 4096, ROWS = 1024;  // bf16, 8 MiB

__device__ __forceinline__ void wait_test(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "TW_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TW_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void wait_hint(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "TH_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra TH_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(20)
      : "memory");
}
__global__ void __launch_bounds__(128) k(const __grid_constant__ CUtensorMap m, const uint16_t* src, int mode, int box_rows,
                                         int box_bytes, int S, int iters, long long* out) {
  const int wmode = mode >> 4;
  mode &= 15;
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[16];
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const long long t0 = clock64();
    for (int i = 0; i < iters + S; ++i) {
      if (i >= S) {
        if (wmode == 0) mbar_wait(&full[i % S], ((i - S) / S) & 1);
        else if (wmode == 1) wait_test(&full[i % S], ((i - S) / S) & 1);
        else if (wmode == 2) wait_hint(&full[i % S], ((i - S) / S) & 1);
        else mbar_wait_sleep(&full[i % S], ((i - S) / S) & 1, wmode == 3 ? 32 : 256);
      }
      if (i < iters) {
        const int s = i % S;
        uint8_t* dst = sm + s * box_bytes;
        mbar_arrive_expect_tx(&full[s], box_bytes);
        const int kb = (i + blockIdx.x * 7) % (COLS / 64);
        const int r0 = ((i / (COLS / 64)) * box_rows + blockIdx.x * 128) % (ROWS - box_rows + 1);
        if (mode == 0) {
          for (int c = 0; c < box_bytes / (box_rows * 128); ++c) tma_load_2d(dst + c * box_rows * 128, &m, &full[s], kb * 64 + c * 64, r0);
        } else {
          bulk_g2s(dst, src + (size_t(r0) * COLS + kb * 64) % (size_t(ROWS) * COLS - box_bytes / 2), box_bytes, &full[s]);
        }
      }
    }
    out[blockIdx.x] = clock64() - t0;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  uint16_t* src;
  cudaMalloc(&src, size_t(ROWS) * COLS * 2);
  {
    std::vector<uint16_t> h(size_t(ROWS) * COLS);
    for (size_t i = 0; i < h.size(); ++i) h[i] = uint16_t(i * 2654435761u >> 7);
    cudaMemcpy(src, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  }
  long long* d_out;
  cudaMalloc(&d_out, 148 * 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int wm = 0; wm < 5; ++wm)
    for (int box_rows : {128}) {
      CUtensorMap m;
      cuuint64_t dims[2] = {COLS, ROWS};
      cuuint64_t str[1] = {COLS * 2};
      cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
      cuuint32_t es[2] = {1, 1};
      enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      for (int G : {1, 148})
        for (int S : {2, 4, 8}) {
          const int bb = box_rows * 128;
          const int iters = 256;
          for (int rep = 0; rep < 2; ++rep) k<<<G, 128, 200 * 1024>>>(m, src, 0 | (wm << 4), box_rows, bb, S, iters, d_out);
          long long h[148];
          cudaMemcpy(h, d_out, G * 8, cudaMemcpyDeviceToHost);
          double avg = 0;
          for (int i = 0; i < G; ++i) avg += h[i];
          avg /= G;
          printf("wait=%d tma2d box=64x%-3d G=%3d S=%d: %.0f cyc/iter %.1f B/cyc/SM\n", wm,
                 box_rows, G, S, avg / iters, double(bb) * iters / avg);
        }
    }
  for (int wm = 0; wm < 0; ++wm)
    for (int bb : {2048, 16384})
      for (int G : {1, 148}) {
        const int S = 8;
        CUtensorMap m{};
        const int iters = 256;
        for (int rep = 0; rep < 2; ++rep) k<<<G, 128, 200 * 1024>>>(m, src, 1 | (wm << 4), 128, bb, S, iters, d_out);
        long long h[148];
        cudaMemcpy(h, d_out, G * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < G; ++i) avg += h[i];
        avg /= G;
        printf("wait=%s bulk1d %6d B G=%3d S=%d: %.0f cyc/iter %.1f B/cyc/SM\n", wm == 0 ? "try " : wm == 1 ? "test" : "hint", bb, G, S,
               avg / iters, double(bb) * iters / avg);
      }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
