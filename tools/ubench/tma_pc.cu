// Producer / consumer TMA ring (the GEMM's structure): warp 0 lane 0 waits
// empty[s] then issues a 64 x 128 SW128 box into stage s; warp 1 lane 0 waits
// full[s] then arrives on empty[s].  cycles per stage vs S and G.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "ptx.cuh"
using namespace atmm::ptx;
constexpr int COLS = 4096, ROWS = 1024;
__device__ __forceinline__ void wait_mode(uint64_t* bar, uint32_t phase, int mode) {
  if (mode == 0) { mbar_wait(bar, phase); return; }
  while (true) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(phase) : "memory");
    if (ok) return;
    if (mode == 2) __nanosleep(32);
    if (mode == 3) __nanosleep(128);
  }
}
__global__ void k(const __grid_constant__ CUtensorMap m, int S, int iters, int boxes, long long* out) {
  const int wm = boxes >> 4;
  boxes &= 15;
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[16], empty[16];
  __shared__ long long tiss[32], tdone[32];
  const int bb = 16384 * boxes;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
    tma_prefetch_desc(&m);
  }
  __syncthreads();
  const long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % S;
      wait_mode(&empty[s], ((i / S) & 1) ^ 1, wm);
      mbar_arrive_expect_tx(&full[s], bb);
      for (int b = 0; b < boxes; ++b)
        tma_load_2d(sm + s * bb + b * 16384, &m, &full[s], ((i * boxes + b) % 64) * 64, ((i / 64) * 128 + blockIdx.x * 128) % (ROWS - 128));
      if (i < 32) tiss[i] = clock64() - t0;
    }
  } else if (threadIdx.x == 32) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % S;
      wait_mode(&full[s], (i / S) & 1, wm);
      if (i < 32) tdone[i] = clock64() - t0;
      mbar_arrive(&empty[s]);
    }
    out[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    for (int i = 0; i < 32; ++i) out[200 + i] = tiss[i];
    for (int i = 0; i < 32; ++i) out[240 + i] = tdone[i];
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
  cudaMalloc(&d, 8 * 300);
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[2] = {COLS, ROWS}, str[1] = {COLS * 2};
  cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
  ((EncodeFn)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int wm = 0; wm < 4; ++wm)
  for (int boxes : {1, 3})
    for (int G : {1, 148})
      for (int S : {4}) {
        if (S * boxes * 16384 > 200 * 1024) continue;
        const int iters = 512;
        for (int r = 0; r < 2; ++r) k<<<G, 64, 220 * 1024>>>(m, S, iters, boxes | (wm << 4), d);
        long long h[148];
        cudaMemcpy(h, d, 8 * G, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < G; ++i) avg += h[i];
        avg /= G;
        printf("wait %d boxes/stage %d G=%3d S=%d: %.0f cyc/stage  %.1f B/cyc/SM\n", wm, boxes, G, S, avg / iters, 16384.0 * boxes * iters / avg);
        if (G == 1) {
          long long t[80];
          cudaMemcpy(t, d + 200, 8 * 72, cudaMemcpyDeviceToHost);
          printf("  issue:");
          for (int i = 0; i < 20; ++i) printf(" %lld", t[i]);
          printf("\n  full :");
          for (int i = 0; i < 20; ++i) printf(" %lld", t[40 + i]);
          printf("\n");
        }
      }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
