// Microbenchmark: programmatic dependent launch (PDL) semantics on sm_100a.
//  (1) Which threads of a CTA must execute griddepcontrol.launch_dependents
//      for the CTA to count as triggered (all threads / one warp / one
//      thread)?  Kernel A triggers per `mode` at its start, then spins ~20 us;
//      kernel B (launched with programmatic stream serialization) records
//      %globaltimer at its start: B starting long before A ends = triggered.
//  (2) Latency from the primary grid's last CTA exit to griddepcontrol.wait
//      returning in the dependent grid, and to the dependent's CTAs starting
//      when the primary triggers only at exit.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pdl_trigger pdl_trigger.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void gwait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// out: [cta][2] = start, end
__global__ void __launch_bounds__(256) kA(int mode, uint64_t spin_ns, uint64_t* out, uint4* sink, int sink_per_cta) {
  const uint64_t t0 = gtime();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  bool me = false;
  switch (mode) {
    case 0: me = true; break;                       // every thread
    case 1: me = threadIdx.x == 0; break;           // one thread
    case 2: me = warp == 0; break;                  // one full warp
    case 3: me = lane == 0; break;                  // lane 0 of every warp
    case 4: me = false; break;                      // nobody: trigger at exit
    default: me = warp < 4; break;                  // half the warps
  }
  if (me) trigger();
  while (gtime() - t0 < spin_ns) {
  }
  for (int i = threadIdx.x; i < sink_per_cta; i += blockDim.x) sink[(size_t)blockIdx.x * sink_per_cta + i] = make_uint4(i, 1, 2, 3);
  __syncthreads();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 2] = t0;
    out[blockIdx.x * 2 + 1] = gtime();
  }
}

// out: [cta][2] = start, wait returned
__global__ void __launch_bounds__(256) kB(uint64_t* out) {
  const uint64_t t0 = gtime();
  gwait();
  const uint64_t t1 = gtime();
  if (threadIdx.x == 0) {
    out[blockIdx.x * 2] = t0;
    out[blockIdx.x * 2 + 1] = t1;
  }
}

static void launchB(int grid, uint64_t* out, cudaStream_t s, int cluster) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute a[2];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = 1;
  a[1].id = cudaLaunchAttributeClusterDimension;
  a[1].val.clusterDim.x = cluster;
  a[1].val.clusterDim.y = 1;
  a[1].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, kB, out);
}
static void launchA(int grid, cudaStream_t s, int cluster, int mode, uint64_t spin, uint64_t* out, uint4* sink, int per) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute a[2];
  a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a[0].val.programmaticStreamSerializationAllowed = 1;
  a[1].id = cudaLaunchAttributeClusterDimension;
  a[1].val.clusterDim.x = cluster;
  a[1].val.clusterDim.y = 1;
  a[1].val.clusterDim.z = 1;
  cfg.attrs = a;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, kA, mode, spin, out, sink, per);
}

int main() {
  const int G = 128;
  uint64_t *oa, *ob;
  cudaMalloc(&oa, G * 2 * 8);
  cudaMalloc(&ob, G * 2 * 8);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const char* names[] = {"all threads", "thread 0 only", "warp 0 only", "lane 0 of each warp", "none (exit)",
                         "warps 0-3"};
  std::vector<uint64_t> ha(G * 2), hb(G * 2);
  uint4* sink;
  cudaMalloc(&sink, (size_t)G * 2048 * 16);
  for (int cl : {1, 8}) for (int per : {0, 2048}) for (int rep = 0; rep < 2; ++rep) {
    if (rep == 1) printf("--- cluster %d, %d KB written per CTA before exit\n", cl, per * 16 / 1024);
    for (int mode = 0; mode < 6; ++mode) {
      for (uint64_t spin : {20000ull, 1000ull}) {
        launchA(G, s, cl, mode, spin, oa, sink, per);
        launchB(G, ob, s, cl);
        cudaStreamSynchronize(s);
        cudaMemcpy(ha.data(), oa, G * 16, cudaMemcpyDeviceToHost);
        cudaMemcpy(hb.data(), ob, G * 16, cudaMemcpyDeviceToHost);
        uint64_t a0 = ~0ull, aend = 0, b0 = ~0ull, bmax = 0, wmin = ~0ull, wmax = 0;
        for (int i = 0; i < G; ++i) {
          a0 = std::min(a0, ha[2 * i]);
          aend = std::max(aend, ha[2 * i + 1]);
          b0 = std::min(b0, hb[2 * i]);
          bmax = std::max(bmax, hb[2 * i]);
          wmin = std::min(wmin, hb[2 * i + 1]);
          wmax = std::max(wmax, hb[2 * i + 1]);
        }
        if (rep == 1) {
          printf("trigger=%-22s spin=%5llu ns | B first start %+8.2f us, last start %+8.2f us rel. A's last exit; "
                 "wait returned %+6.2f .. %+6.2f us\n",
                 names[mode], (unsigned long long)spin, ((double)b0 - (double)aend) / 1e3,
                 ((double)bmax - (double)aend) / 1e3, ((double)wmin - (double)aend) / 1e3,
                 ((double)wmax - (double)aend) / 1e3);
        }
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
