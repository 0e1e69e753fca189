// forward_kernels.cu -- the layer forward of the serving model on sm_100a:
//   cur_{l+1} = tanh(cur_l . W_l + bypass_l(cur_l))        (model.hpp:213-246)
// (forward_merged, model.hpp:192-211, is the same launch without bypass;
// forward_mixture, model.hpp:248-328, uses combined mixture slots).
//
// Two launches per layer, chained with programmatic dependent launch:
//   fwd_shrink_kernel  mid = scale * cur . down_a for every (row tile,
//                      segment, 32-rank chunk), written as the bf16 A image
//                      of a K-extension block (rows outside the segment 0).
//                      K split over a thread-block cluster, fixed-order DSMEM
//                      reduction (bit-identical reruns).
//   fwd_gemm_kernel    persistent tcgen05 GEMM, 128 x bn tiles, TMA ring of
//                      64-wide K blocks (X K-major SW128, W MN-major SW128),
//                      then the tile's K-extension blocks (mid . up^T, up^T
//                      read straight from the registry) into the SAME TMEM
//                      accumulator, tanh + bf16 in the epilogue.  Double-
//                      buffered TMEM so tile i's epilogue overlaps tile i+1's
//                      MMAs.  The last layer scatters rows back to the
//                      caller's order.
// Rows run in segment-sorted order ("Layer forward").
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <map>
#include <mutex>
#include <cstdlib>

#include "device_types.hpp"
#include "ptx.cuh"

namespace atmm {
using namespace ptx;

namespace {

constexpr int kFwdThreads = 192;  // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue
constexpr uint32_t kFwdA = 16384;  // 128 rows x 64 bf16 (one K block of X)

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
// mid = hi + lo with hi = bf16(mid), lo = bf16(mid - hi): the K-extension
// carries mid to ~16 mantissa bits (two bf16 MMAs against the same up^T),
// so rounding mid costs nothing next to the fp32 GEMM accumulation.
__device__ __forceinline__ void split_bf16x2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat16 ha = __float2bfloat16_rn(a), hb = __float2bfloat16_rn(b);
  const __nv_bfloat162 h2(ha, hb);
  hi = *reinterpret_cast<const uint32_t*>(&h2);
  lo = pack_bf16x2(a - __bfloat162float(ha), b - __bfloat162float(hb));
}
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void st_global_v4(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void st_global_v2(void* p, uint32_t a, uint32_t b) {
  asm volatile("st.global.v2.b32 [%0], {%1, %2};" ::"l"(p), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ float4 ld_cluster_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr));
  return v;
}

// Epilogue store of 8 accumulator columns [c, c + 8) of one output row:
// tanh (layer forward) or identity (plain GEMM), bf16 or fp32 out.
__device__ __forceinline__ void store8(const FwdParams& p, int64_t orow, int col, const float (&a)[8]) {
  if (p.act_none) {
    if (p.out_f32) {
      float* o = reinterpret_cast<float*>(p.out) + orow * p.ldo + col;
      st_global_v4(o, __float_as_uint(a[0]), __float_as_uint(a[1]), __float_as_uint(a[2]), __float_as_uint(a[3]));
      st_global_v4(o + 4, __float_as_uint(a[4]), __float_as_uint(a[5]), __float_as_uint(a[6]), __float_as_uint(a[7]));
    } else {
      st_global_v4(p.out + orow * p.ldo + col, pack_bf16x2(a[0], a[1]), pack_bf16x2(a[2], a[3]), pack_bf16x2(a[4], a[5]),
                   pack_bf16x2(a[6], a[7]));
    }
    return;
  }
  st_global_v4(p.out + orow * p.ldo + col, pack_bf16x2(tanh_fast(a[0]), tanh_fast(a[1])),
               pack_bf16x2(tanh_fast(a[2]), tanh_fast(a[3])), pack_bf16x2(tanh_fast(a[4]), tanh_fast(a[5])),
               pack_bf16x2(tanh_fast(a[6]), tanh_fast(a[7])));
}

// Element offset of (row, col) in a K-extension A image: 128 x kk bf16 in
// 8x8 core matrices, [row / 8][col / 8][row % 8][col % 8] (K-major,
// no swizzle: LBO 128 B, SBO kk * 16 B).  The images hold [mid_hi | mid_lo],
// i.e. kk = 2 x the rank chunk.
__device__ __forceinline__ int64_t ext_a_index(int row, int col, int kk) {
  return (static_cast<int64_t>(row >> 3) * (kk >> 3) + (col >> 3)) * 64 + (row & 7) * 8 + (col & 7);
}

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Debug trace: shrink CTAs at [0, 4096) x 16 events, GEMM CTAs after them.
#define FTRACE(base, ev)                                                                      \
  do {                                                                                        \
    if (p.trace) p.trace[(static_cast<size_t>(base) + blockIdx.y * gridDim.x + blockIdx.x) * 16 + (ev)] = gtime(); \
  } while (0)

}  // namespace

// -------------------------------------------------------------------------
// Shrink: one CTA per (K slice, work item); the K slices of an item form a
// cluster and reduce through DSMEM in rank order.
// smem: [stages x (A 16 KB | B sbytes = max ncols x 128 B)] [red: 128 x (ncols + 4) fp32]
// -------------------------------------------------------------------------
__global__ void __launch_bounds__(kFwdThreads, 1)
    fwd_shrink_kernel(const __grid_constant__ CUtensorMap xmap, const FwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = align1024(smem_raw);
  __shared__ uint64_t full[8], empty[8], done, recv_bar;
  __shared__ uint32_t tslot;
  __shared__ FwdExt sx[8];  // the item's chunks (<= 128 columns, >= 16 each)
  const uint32_t kStage = kFwdA + static_cast<uint32_t>(p.sbytes);
  const int S = p.stages;
  const int warp = static_cast<int>(threadIdx.x >> 5), lane = static_cast<int>(threadIdx.x & 31);
  const FwdItem item = p.items[blockIdx.y];
  const int ks = p.ks, kr = static_cast<int>(blockIdx.x);
  const int kb0 = static_cast<int>(int64_t(p.nkb) * kr / ks);
  const int kb1 = static_cast<int>(int64_t(p.nkb) * (kr + 1) / ks);
  const int ncols = item.ncols;
  const int pitch = ncols + 4;  // fp32 words per red row (16-byte skew)
  float* red = reinterpret_cast<float*>(sm + S * kStage);  // this CTA's partial, 128 x pitch
  const int rows_per = kTileM / ks;                        // rows each cluster rank finalises
  const uint32_t slot_bytes = static_cast<uint32_t>(rows_per * pitch) * 4u;
  float* recv = red + kTileM * pitch;                      // ks slots: the senders' partials of my rows

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    mbar_init(&recv_bar, 1);
    fence_mbar_init();
    tma_prefetch_desc(&xmap);
    if (ks > 1) mbar_arrive_expect_tx(&recv_bar, static_cast<uint32_t>(ks - 1) * slot_bytes);  // own slot stays in red
  }
  if (warp == 1) tmem_alloc(&tslot, 128);
  const int ne = item.e_end - item.e_begin;
  if (warp == 2 && lane < ne) sx[lane] = p.exts[item.e_begin + lane];
  tc_fence_before();
  if (ks > 1) {
    cluster_sync();  // every rank's recv_bar is initialised before any partial is pushed
  } else {
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tmem = tslot;

  if (threadIdx.x == 0) FTRACE(0, 0);
  // Release the GEMM launch once the previous grid (which wrote cur) is
  // complete: the GEMM's main loop reads cur without a wait of its own.
  griddep_wait();
  griddep_launch_dependents();
  if (warp == 0) {
    if (elect_one()) {
      griddep_wait();  // cur is the previous launch's output
      FTRACE(0, 1);
      // per-chunk invariants in registers: source at K block kb0, bytes per K block
      const uint16_t* src[8];
      uint32_t dst_off[8], bytes[8], kstep[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (e < ne) {
          const FwdExt& x = sx[e];
          src[e] = x.down_t + int64_t(p.layer) * x.down_ls + int64_t(kb0) * x.r_pad * kBK + x.kc * 2048;
          kstep[e] = static_cast<uint32_t>(x.r_pad) * kBK;
          dst_off[e] = static_cast<uint32_t>(x.col) * 128u;
          bytes[e] = static_cast<uint32_t>(x.kk) * 128u;
        }
      }
      const uint32_t tx = kFwdA + static_cast<uint32_t>(ncols) * 128u;
      const int row0 = item.tile * kTileM;
      for (int kb = kb0, i = 0; kb < kb1; ++kb, ++i) {
        const int s = i % S;
        const uint32_t ph = static_cast<uint32_t>(i / S) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        uint8_t* a = sm + s * kStage;
        uint8_t* b = a + kFwdA;
        mbar_arrive_expect_tx(&full[s], tx);
        tma_load_2d(a, &xmap, &full[s], kb * kBK, row0);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (e < ne) {
            bulk_g2s(b + dst_off[e], src[e], bytes[e], &full[s]);
            src[e] += kstep[e];
          }
        }
      }
      FTRACE(0, 2);
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      const uint32_t idesc = idesc_bf16(128, static_cast<uint32_t>(ncols));
      for (int kb = kb0, i = 0; kb < kb1; ++kb, ++i) {
        const int s = i % S;
        const uint32_t ph = static_cast<uint32_t>(i / S) & 1u;
        mbar_wait(&full[s], ph);
        if (i == 0) FTRACE(0, 3);
        tc_fence_after();
        const uint32_t a = smem_u32(sm + s * kStage), b = a + kFwdA;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          mma_bf16(tmem, smem_desc(a + k * 32, 16, 1024, kLayoutSW128), smem_desc(b + k * 256, 128, 1024, kLayoutNone),
                   idesc, (i > 0 || k > 0) ? 1u : 0u);
        }
        mma_commit(&empty[s]);
      }
      FTRACE(0, 4);
      mma_commit(&done);
    }
    __syncwarp();
  } else {
    // Epilogue warps: warp w reads TMEM lanes 32 (w % 4) .. +32 = tile rows.
    const int q = warp & 3;
    const int row = q * 32 + lane;
    mbar_wait_sleep(&done, 0, 64);
    if (threadIdx.x == 64) FTRACE(0, 5);
    tc_fence_after();
    for (int e = 0; e < ne; ++e) {
      const FwdExt& x = sx[e];
      const bool valid = row >= x.lo && row < x.hi;
      for (int cc = 0; cc < x.kk; cc += 16) {
        uint32_t v[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(x.col + cc), v);
        tmem_wait_ld();
        if (kb1 <= kb0) {  // empty K slice (never planned): a zero partial
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = 0u;
        }
        if (ks == 1) {
          uint16_t* img = reinterpret_cast<uint16_t*>(p.ext + x.a_off);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t hi[4], lo[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float f0 = valid ? __uint_as_float(v[h * 8 + 2 * j]) * x.scale : 0.f;
              const float f1 = valid ? __uint_as_float(v[h * 8 + 2 * j + 1]) * x.scale : 0.f;
              split_bf16x2(f0, f1, hi[j], lo[j]);
            }
            st_global_v4(img + ext_a_index(row, cc + h * 8, 2 * x.kk), hi[0], hi[1], hi[2], hi[3]);
            st_global_v4(img + ext_a_index(row, x.kk + cc + h * 8, 2 * x.kk), lo[0], lo[1], lo[2], lo[3]);
          }
        } else {
          const uint32_t dst = smem_u32(red + row * pitch + x.col + cc);
#pragma unroll
          for (int j = 0; j < 4; ++j) st_shared_v4(dst + j * 16, v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
        }
      }
    }
    if (ks > 1) {
      // Push rows [q*rows_per, +rows_per) of the partial to rank q's slot kr
      // (one bulk DSMEM copy per rank), then wait for the ks slots of mine.
      fence_proxy_async_smem();
      named_bar_sync(1, 128);
      if (threadIdx.x == 64) {
        const uint32_t src0 = smem_u32(red), dst0 = smem_u32(recv) + static_cast<uint32_t>(kr) * slot_bytes;
        for (int q2 = 0; q2 < ks; ++q2) {
          if (q2 == kr) continue;  // my own rows are reduced straight from red
          bulk_s2cluster(map_cta(dst0, static_cast<uint32_t>(q2)), src0 + static_cast<uint32_t>(q2) * slot_bytes, slot_bytes,
                         map_cta(smem_u32(&recv_bar), static_cast<uint32_t>(q2)));
        }
      }
      mbar_wait_cluster(&recv_bar, 0);
    }
  }

  if (threadIdx.x == 64) FTRACE(0, 6);
  if (ks > 1) {
    // Fixed-order reduction of my rows over the ks received slots; the
    // cluster barrier (arrive now, wait at exit) keeps every rank's partial
    // alive until all pushes out of it have landed.
    cluster_arrive();
    if (threadIdx.x == 64) FTRACE(0, 7);
    if (warp >= 2) {
      const int tid = static_cast<int>(threadIdx.x) - 64;
      const int groups = ncols / 4;
      const uint32_t recv_base = smem_u32(recv);
      for (int u = tid; u < rows_per * groups; u += 128) {
        const int lr = u / groups;
        const int row = kr * rows_per + lr;
        const int c = (u % groups) * 4;
        const uint32_t off = recv_base + static_cast<uint32_t>(lr * pitch + c) * 4u;
        const uint32_t own = smem_u32(red) + static_cast<uint32_t>(row * pitch + c) * 4u;  // slot kr = my partial
        uint4 v[16];
#pragma unroll
        for (int q2 = 0; q2 < 16; ++q2)
          if (q2 < ks) v[q2] = ld_shared_v4(q2 == kr ? own : off + static_cast<uint32_t>(q2) * slot_bytes);
        float4 acc = make_float4(__uint_as_float(v[0].x), __uint_as_float(v[0].y), __uint_as_float(v[0].z),
                                 __uint_as_float(v[0].w));
#pragma unroll
        for (int q2 = 1; q2 < 16; ++q2) {
          if (q2 < ks) {
            acc.x += __uint_as_float(v[q2].x);
            acc.y += __uint_as_float(v[q2].y);
            acc.z += __uint_as_float(v[q2].z);
            acc.w += __uint_as_float(v[q2].w);
          }
        }
        int e = 0;
        while (e + 1 < ne && sx[e + 1].col <= c) ++e;
        const FwdExt& x = sx[e];
        const bool valid = row >= x.lo && row < x.hi;
        const float sc = valid ? x.scale : 0.f;
        uint16_t* img = reinterpret_cast<uint16_t*>(p.ext + x.a_off);
        uint32_t hi0, lo0, hi1, lo1;
        split_bf16x2(acc.x * sc, acc.y * sc, hi0, lo0);
        split_bf16x2(acc.z * sc, acc.w * sc, hi1, lo1);
        st_global_v2(img + ext_a_index(row, c - x.col, 2 * x.kk), hi0, hi1);
        st_global_v2(img + ext_a_index(row, x.kk + c - x.col, 2 * x.kk), lo0, lo1);
      }
    }
    if (threadIdx.x == 64) FTRACE(0, 8);
    cluster_wait();
  }
  if (threadIdx.x == 64) FTRACE(0, 9);
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 128);
  }
}

// -------------------------------------------------------------------------
// Persistent base GEMM + K-extension bypass + tanh.
// smem: [stages x (A 16 KB | B bn x 128 B)]
// -------------------------------------------------------------------------
__global__ void __launch_bounds__(kFwdThreads, 1)
    fwd_gemm_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap wmap,
                    const FwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = align1024(smem_raw);
  __shared__ uint64_t full[8], empty[8], tfull[2], tempty[2], recv_bar;
  __shared__ uint32_t tslot;
  const int S = p.stages, bn = p.bn;
  // bk2 (plain GEMM, K % 64 == 0): 128-deep K stages, A as two 64-wide atoms
  // in one 3-D TMA box, W as 128-row boxes: half the TMA instructions and
  // barrier round trips per K
  const bool bk2 = p.bk2 != 0;
  const uint32_t kA = bk2 ? 2u * kFwdA : kFwdA;
  const uint32_t kStage = kA + static_cast<uint32_t>(bn) * (bk2 ? 256u : 128u);
  const int warp = static_cast<int>(threadIdx.x >> 5), lane = static_cast<int>(threadIdx.x & 31);
  // Split-K (small batches): a cluster of kz CTAs shares one tile, rank z
  // accumulates K blocks [kb0, kb1) and the last rank adds the K-extension
  // blocks; partial rows meet their owner rank by bulk DSMEM pushes and are
  // summed in rank order (deterministic), then tanh.  One tile per cluster.
  // A multicast (mc > 1, small batches, no split-K): a cluster of mc CTAs
  // runs mc adjacent N tiles of one row tile in lockstep; each CTA loads
  // 128 / mc rows of every A block and multicasts them to all, so the A
  // traffic per SM drops mc-fold.  A stage is refilled once every CTA of the
  // cluster has consumed it (empty count mc, commits multicast).
  const int kz = p.kz, mc = p.mc;
  const int csize = kz * mc;
  const int crank = static_cast<int>(blockIdx.x) % csize;
  const int z = kz > 1 ? crank : 0;
  const int mr = mc > 1 ? crank : 0;
  const uint16_t mc_mask = static_cast<uint16_t>((1u << mc) - 1u);
  const int cl = static_cast<int>(blockIdx.x) / csize, ncl = static_cast<int>(gridDim.x) / csize;
  // work units: tiles (mc == 1) or groups of mc N tiles (tile of this CTA: tile_of)
  const int gpr = p.ntn / mc, ngroups = p.num_tiles / mc;
  auto tile_of = [&](int g) { return mc == 1 ? g : (g / gpr) * p.ntn + (g % gpr) * mc + mr; };
  const int kb0 = p.nkb * z / kz, kb1 = p.nkb * (z + 1) / kz;
  const int nk2 = (p.nkb + 1) / 2, j0 = nk2 * z / kz, j1 = nk2 * (z + 1) / kz;  // bk2: 128-deep K blocks
  // K-extension (bypass) blocks of a split-K tile are dealt round-robin over
  // the cluster's ranks (ext e to rank (e - first) % kz): no rank's K loop is
  // longer than the others' by all of them
  const bool do_ext = p.exts != nullptr;
  // split-K: one tile per cluster; only its valid rows (a batch of n < 128
  // rows pads the tile) are staged, exchanged and reduced, rows_per per rank
  const int64_t left = p.n - int64_t(cl / (p.ntn > 0 ? p.ntn : 1)) * kTileM;
  const int valid = kz > 1 ? static_cast<int>(left < 0 ? 0 : (left > kTileM ? kTileM : left)) : kTileM;
  const int rows_per = kz > 1 ? ((valid + kz - 1) / kz + 7) & ~7 : kTileM;
  const int pitch = bn + 4;  // fp32 words per staged row (16-byte skew)
  const uint32_t slot_bytes = static_cast<uint32_t>(rows_per * pitch) * 4u;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], static_cast<uint32_t>(mc));
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    mbar_init(&recv_bar, 1);
    fence_mbar_init();
    tma_prefetch_desc(&xmap);
    tma_prefetch_desc(&wmap);
    if (kz > 1) mbar_arrive_expect_tx(&recv_bar, static_cast<uint32_t>(kz - 1) * slot_bytes);  // own slot stays in stage
  }
  if (threadIdx.x == 0) FTRACE(4096, 0);
  if (warp == 1) tmem_alloc(&tslot, static_cast<uint32_t>(2 * bn));
  tc_fence_before();
  if (csize > 1) {
    cluster_sync();  // (mc: every CTA's barriers exist before any multicast lands)
  } else {
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tmem = tslot;
  // Release the next launch at once (every thread): it waits for this grid
  // itself before reading what this grid writes; its CTAs only get SMs as
  // these exit, so this just removes the launch gap.
  griddep_launch_dependents();

  if (warp == 0) {
    if (elect_one()) {
      // Without a bypass the previous launch is the previous layer's GEMM,
      // which releases its dependents before its epilogue is done.  With one,
      // the shrink launch in between only released this grid after its own
      // griddep_wait, so cur is complete; the A images are waited for below.
      bool waited = p.exts == nullptr;
      if (waited) griddep_wait();
      FTRACE(4096, 7);
      int i = 0;
      for (int g = cl; g < ngroups; g += ncl) {
        const int tile = tile_of(g);
        const int t = tile / p.ntn;
        const int n0 = (tile % p.ntn) * bn;
        if (bk2) {
          for (int j = j0; j < j1; ++j, ++i) {
            const int s = i % S;
            mbar_wait(&empty[s], (static_cast<uint32_t>(i / S) & 1u) ^ 1u);
            uint8_t* a = sm + s * kStage;
            uint8_t* b = a + kA;
            mbar_arrive_expect_tx(&full[s], kStage);
            tma_load_3d(a, &xmap, &full[s], 0, t * kTileM, 2 * j);
            for (int c = 0; c < bn; c += 64) tma_load_3d(b + c * 256, &wmap, &full[s], n0 + c, j * 2 * kBK, p.layer);
          }
        } else {
          // K order rotated per tile (per group under mc: the cluster's A
          // blocks must match) so concurrent CTAs spread over the L2 lines
          const int nk = kb1 - kb0, rot = p.krot ? (g % max(gpr, 1)) % max(nk, 1) : 0;
          for (int j = 0; j < nk; ++j, ++i) {
            const int kb = kb0 + (j + rot < nk ? j + rot : j + rot - nk);
            const int s = i % S;
            const uint32_t ph = static_cast<uint32_t>(i / S) & 1u;
            mbar_wait(&empty[s], ph ^ 1u);
            uint8_t* a = sm + s * kStage;
            uint8_t* b = a + kFwdA;
            mbar_arrive_expect_tx(&full[s], kStage);
            if (mc > 1) {
              const int rows = kTileM / mc;
              tma_load_2d_mc(a + mr * rows * 128, &xmap, &full[s], kb * kBK, t * kTileM + mr * rows, mc_mask);
            } else {
              tma_load_2d(a, &xmap, &full[s], kb * kBK, t * kTileM);
            }
            for (int c = 0; c < bn; c += 64) tma_load_3d(b + c * 128, &wmap, &full[s], n0 + c, kb * kBK, p.layer);
          }
        }
        if (!do_ext) continue;
        for (int e = p.ext_begin[t] + z; e < p.ext_begin[t + 1]; e += kz, ++i) {
          if (!waited) {
            griddep_wait();  // the A images are the shrink launch's output
            FTRACE(4096, 3);
            waited = true;
          }
          const FwdExt& x = p.exts[e];
          const int s = i % S;
          const uint32_t ph = static_cast<uint32_t>(i / S) & 1u;
          mbar_wait(&empty[s], ph ^ 1u);
          uint8_t* a = sm + s * kStage;
          uint8_t* b = a + kFwdA;
          const int g_pad = static_cast<int>(x.up_ls / x.r_pad / 8);  // up^T row groups in the registry
          const int g_n = min(bn / 8, g_pad - n0 / 8);
          const uint32_t a_bytes = static_cast<uint32_t>(x.kk) * 512u;  // [hi | lo]
          const uint32_t g_bytes = static_cast<uint32_t>(x.kk) * 16u;
          mbar_arrive_expect_tx(&full[s], a_bytes + g_bytes * static_cast<uint32_t>(g_n));
          bulk_g2s(a, p.ext + x.a_off, a_bytes, &full[s]);
          const uint16_t* ub = x.up_t + int64_t(p.layer) * x.up_ls + int64_t(n0 / 8) * x.r_pad * 8 + x.kc * 256;
          if (x.kk == x.r_pad) {
            bulk_g2s(b, ub, g_bytes * static_cast<uint32_t>(g_n), &full[s]);
          } else {
            for (int gg = 0; gg < g_n; ++gg) bulk_g2s(b + gg * g_bytes, ub + int64_t(gg) * x.r_pad * 8, g_bytes, &full[s]);
          }
        }
      }
      if (mc > 1) {  // every CTA's commits to this CTA's empty barriers have landed
        for (int j = 0; j < S; ++j, ++i) mbar_wait(&empty[i % S], (static_cast<uint32_t>(i / S) & 1u) ^ 1u);
      }
      griddep_launch_dependents();
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      const uint32_t idesc_main = idesc_bf16(128, static_cast<uint32_t>(bn), 0, 1);
      const uint32_t idesc_ext = idesc_bf16(128, static_cast<uint32_t>(bn));
      int i = 0, it = 0;
      for (int g = cl; g < ngroups; g += ncl, ++it) {
        const int t = tile_of(g) / p.ntn;
        const int acc = it & 1;
        mbar_wait(&tempty[acc], (static_cast<uint32_t>(it >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem + static_cast<uint32_t>(acc * bn);
        if (bk2) {
          for (int j = j0; j < j1; ++j, ++i) {
            const int s = i % S;
            mbar_wait(&full[s], static_cast<uint32_t>(i / S) & 1u);
            tc_fence_after();
            const uint32_t a = smem_u32(sm + s * kStage), b = a + kA;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              mma_bf16(d, smem_desc(a + (k >> 2) * kFwdA + (k & 3) * 32, 16, 1024, kLayoutSW128),
                       smem_desc(b + k * 2048, 16384, 1024, kLayoutSW128), idesc_main, (j > j0 || k > 0) ? 1u : 0u);
            }
            mma_commit(&empty[s]);
          }
        } else {
          for (int kb = kb0; kb < kb1; ++kb, ++i) {  // (the producer's rotated K order: the sum is order-free here)
            const int s = i % S;
            mbar_wait(&full[s], static_cast<uint32_t>(i / S) & 1u);
            if (it == 0 && kb == kb0) FTRACE(4096, 1);
            tc_fence_after();
            const uint32_t a = smem_u32(sm + s * kStage), b = a + kFwdA;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              mma_bf16(d, smem_desc(a + k * 32, 16, 1024, kLayoutSW128), smem_desc(b + k * 2048, 8192, 1024, kLayoutSW128),
                       idesc_main, (kb > kb0 || k > 0) ? 1u : 0u);
            }
            if (mc > 1) {
              mma_commit_mc(&empty[s], mc_mask);
            } else {
              mma_commit(&empty[s]);
            }
          }
        }
        if (do_ext) {
          for (int e = p.ext_begin[t] + z; e < p.ext_begin[t + 1]; e += kz, ++i) {
            const int kk = p.exts[e].kk;
            const int s = i % S;
            mbar_wait(&full[s], static_cast<uint32_t>(i / S) & 1u);
            tc_fence_after();
            const uint32_t a = smem_u32(sm + s * kStage), b = a + kFwdA;
            const uint32_t sbo_a = static_cast<uint32_t>(kk) * 32u, sbo_b = static_cast<uint32_t>(kk) * 16u;
            for (int k = 0; k < kk / 16; ++k) {
              const uint64_t bd = smem_desc(b + k * 256, 128, sbo_b, kLayoutNone);
              mma_bf16(d, smem_desc(a + k * 256, 128, sbo_a, kLayoutNone), bd, idesc_ext, 1u);
              mma_bf16(d, smem_desc(a + kk * 16 + k * 256, 128, sbo_a, kLayoutNone), bd, idesc_ext, 1u);
            }
            if (mc > 1) {
              mma_commit_mc(&empty[s], mc_mask);
            } else {
              mma_commit(&empty[s]);
            }
          }
        }
        if (it == 0) FTRACE(4096, 2);
        mma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else if (kz == 1) {
    const int q = warp & 3;
    int it = 0;
    for (int g = cl; g < ngroups; g += ncl, ++it) {
      const int tile = tile_of(g);
      const int t = tile / p.ntn;
      const int n0 = (tile % p.ntn) * bn;
      const int acc = it & 1;
      const int64_t srow = int64_t(t) * kTileM + q * 32 + lane;
      const bool rv = srow < p.n;
      const int64_t orow = rv && p.out_rows ? p.out_rows[srow] : srow;
      mbar_wait_sleep(&tfull[acc], static_cast<uint32_t>(it >> 1) & 1u, 32);
      if (it == 0 && threadIdx.x == 64) FTRACE(4096, 4);
      tc_fence_after();
      const uint32_t tbase = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * bn);
      for (int c = 0; c < bn; c += 32) {
        uint32_t v[32];
        tmem_ld32(tbase + static_cast<uint32_t>(c), v);
        tmem_wait_ld();
        if (rv) {
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            float a8[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) a8[j] = __uint_as_float(v[8 * g + j]);
            if (n0 + c + 8 * g < p.d) store8(p, orow, n0 + c + 8 * g, a8);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (it == 0 && threadIdx.x == 64) FTRACE(4096, 5);
    }
  } else {
    // Split-K epilogue (one tile per cluster; the ring is idle once the
    // accumulator is complete, so it holds the staged partial and the
    // receive slots).
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int tile = cl;
    const int t = tile / p.ntn;
    const int n0 = (tile % p.ntn) * bn;
    float* stage = reinterpret_cast<float*>(sm);                 // 128 x pitch
    float* recv = stage + kTileM * pitch;                         // kz slots x rows_per x pitch
    if (tile < p.num_tiles) {
      mbar_wait_sleep(&tfull[0], 0, 32);
      if (threadIdx.x == 64) FTRACE(4096, 4);
      tc_fence_after();
      const uint32_t tbase = tmem + (static_cast<uint32_t>(q * 32) << 16);
      // quadrants wholly past the exchanged rows stage nothing
      for (int c = 0; q * 32 < rows_per * kz && c < bn; c += 32) {
        uint32_t v[32];
        tmem_ld32(tbase + static_cast<uint32_t>(c), v);
        tmem_wait_ld();
        const uint32_t dst = smem_u32(stage + row * pitch + c);
#pragma unroll
        for (int j = 0; j < 8; ++j) st_shared_v4(dst + j * 16, v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      }
    }
    fence_proxy_async_smem();
    if (threadIdx.x == 64) FTRACE(4096, 5);
  }
  if (kz > 1) {
    // every rank's MMAs are done (its ring is free for the receive slots) and
    // its partial is staged before anything is pushed
    cluster_sync();
    if (threadIdx.x == 64) FTRACE(4096, 8);
  }
  if (warp >= 2 && kz > 1) {
    const int tile = cl;
    const int t = tile / p.ntn;
    const int n0 = (tile % p.ntn) * bn;
    float* stage = reinterpret_cast<float*>(sm);
    float* recv = stage + kTileM * pitch;
    if (threadIdx.x == 64) {
      const uint32_t src0 = smem_u32(stage), dst0 = smem_u32(recv) + static_cast<uint32_t>(z) * slot_bytes;
      for (int r2 = 0; r2 < kz; ++r2) {
        if (r2 == z) continue;  // my own rows are reduced straight from stage
        bulk_s2cluster(map_cta(dst0, static_cast<uint32_t>(r2)), src0 + static_cast<uint32_t>(r2) * slot_bytes, slot_bytes,
                       map_cta(smem_u32(&recv_bar), static_cast<uint32_t>(r2)));
      }
    }
    mbar_wait_cluster(&recv_bar, 0);
    if (threadIdx.x == 64) FTRACE(4096, 9);
    if (tile < p.num_tiles) {
      const int tid = static_cast<int>(threadIdx.x) - 64;
      const int groups = bn / 8;
      const uint32_t recv_base = smem_u32(recv);
      for (int u = tid; u < rows_per * groups; u += 128) {
        const int lr = u / groups;
        const int c = (u % groups) * 8;
        const int64_t srow = int64_t(t) * kTileM + z * rows_per + lr;
        if (srow >= p.n || n0 + c >= p.d) continue;
        float acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.f;
        for (int r2 = 0; r2 < kz; ++r2) {  // rank order: deterministic
          const uint32_t off = r2 == z ? smem_u32(stage) + static_cast<uint32_t>((z * rows_per + lr) * pitch + c) * 4u
                                       : recv_base + static_cast<uint32_t>(r2) * slot_bytes + static_cast<uint32_t>(lr * pitch + c) * 4u;
          const uint4 v0 = ld_shared_v4(off), v1 = ld_shared_v4(off + 16);
          acc[0] += __uint_as_float(v0.x);
          acc[1] += __uint_as_float(v0.y);
          acc[2] += __uint_as_float(v0.z);
          acc[3] += __uint_as_float(v0.w);
          acc[4] += __uint_as_float(v1.x);
          acc[5] += __uint_as_float(v1.y);
          acc[6] += __uint_as_float(v1.z);
          acc[7] += __uint_as_float(v1.w);
        }
        const int64_t orow = p.out_rows ? p.out_rows[srow] : srow;
        store8(p, orow, n0 + c, acc);
      }
    }
  }
  if (threadIdx.x == 64) FTRACE(4096, 6);
  if (threadIdx.x == 64 && p.trace) p.trace[(4096 + blockIdx.x) * 16 + 15] = clock64();
  tc_fence_before();
  if (csize > 1) {
    cluster_sync();  // every pushed partial / multicast block has landed before any rank leaves
  } else {
    __syncthreads();
  }
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, static_cast<uint32_t>(2 * bn));
  }
}

// Row gather into segment-sorted order: dst[i] = x[order[i]] (one warp per row).
__global__ void fwd_gather_rows_kernel(const uint16_t* __restrict__ x, int64_t ldx, uint16_t* __restrict__ dst,
                                       int64_t ldd, const int32_t* __restrict__ order, int64_t n, int64_t d) {
  griddep_wait();
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  const int lane = static_cast<int>(threadIdx.x & 31);
  for (int64_t r = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    const uint4* src = reinterpret_cast<const uint4*>(x + int64_t(order[r]) * ldx);
    uint4* out = reinterpret_cast<uint4*>(dst + r * ldd);
    for (int64_t c = lane; c < d / 8; c += 32) out[c] = src[c];
  }
  griddep_launch_dependents();
}

// ------------------------------------------------------------- launchers --
namespace {
template <typename K>
cudaError_t set_smem(K kernel, size_t smem) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
}
// Programmatic dependent launch is always on: every kernel waits
// (griddepcontrol.wait) before touching its predecessor's outputs.
constexpr bool fwd_pdl() { return true; }
}  // namespace

cudaError_t launch_fwd_gather(const uint16_t* x, int64_t ldx, uint16_t* dst, int64_t ldd, const int32_t* order,
                              int64_t n, int64_t d, cudaStream_t stream) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(256, 1, 1);
  cfg.gridDim = dim3(static_cast<unsigned>(std::min<int64_t>((n + 7) / 8, 148 * 8)), 1, 1);
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = fwd_pdl() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, fwd_gather_rows_kernel, x, ldx, dst, ldd, order, n, d);
}

cudaError_t launch_fwd_shrink(const CUtensorMap& xmap, const FwdParams& p, size_t smem, cudaStream_t stream) {
  cudaError_t e = set_smem(fwd_shrink_kernel, smem);
  if (e != cudaSuccess) return e;
  if (p.ks > 8) {  // 16-CTA clusters are non-portable
    static bool done = false;
    if (!done) {
      e = cudaFuncSetAttribute(fwd_shrink_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
      done = true;
    }
  }
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(p.ks);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kFwdThreads, 1, 1);
  cfg.gridDim = dim3(static_cast<unsigned>(p.ks), static_cast<unsigned>(p.num_items), 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = fwd_pdl() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, fwd_shrink_kernel, xmap, p);
}

cudaError_t launch_fwd_gemm(const CUtensorMap& xmap, const CUtensorMap& wmap, const FwdParams& p, int grid, size_t smem,
                            cudaStream_t stream) {
  cudaError_t e = set_smem(fwd_gemm_kernel, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;  // split-K cluster (1: plain)
  attr[0].val.clusterDim.x = static_cast<unsigned>(p.kz * p.mc);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kFwdThreads, 1, 1);
  cfg.gridDim = dim3(static_cast<unsigned>(grid), 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = fwd_pdl() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, fwd_gemm_kernel, xmap, wmap, p);
}

}  // namespace atmm

namespace atmm {
using namespace ptx;

// -------------------------------------------------------------------------
// CTA-pair GEMM (cta_group::2): a cluster of 2 CTAs on one TPC computes a
// 256 x bn tile (rank r owns row tile 2 pi + r); the leader issues
// tcgen05.mma with M = 256, each SM stages its 128 rows of X and HALF of the
// W columns, so per-SM operand traffic per MMA cycle halves against the
// 1-SM kernel.  The pair runs the union of its two row tiles' K-extension
// chunks (a row tile without rows in a chunk streams a zero A image).
// smem per CTA: [stages x (A 16 KB | B bn/2 x 128 B)]
// -------------------------------------------------------------------------
__global__ void __launch_bounds__(kFwdThreads, 1)
    fwd_gemm_pair_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap wmap,
                         const __grid_constant__ CUtensorMap amap, const FwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = align1024(smem_raw);
  __shared__ uint64_t full[8], empty[8], tfull[2], tempty[2];
  __shared__ uint32_t tslot;
  const int S = p.stages, bn = p.bn, hb = p.bn / 2;
  const bool bk2 = p.bk2 != 0;  // 128-deep K stages, as in fwd_gemm_kernel
  const uint32_t kA = bk2 ? 2u * kFwdA : kFwdA;
  const uint32_t kStage = kA + static_cast<uint32_t>(hb) * (bk2 ? 256u : 128u);
  const int warp = static_cast<int>(threadIdx.x >> 5), lane = static_cast<int>(threadIdx.x & 31);
  const int rank = static_cast<int>(cluster_ctarank());
  const bool leader = rank == 0;
  const int pair_id = static_cast<int>(blockIdx.x) / 2, npairs = static_cast<int>(gridDim.x) / 2;
  const int row_tiles = static_cast<int>((p.n + kTileM - 1) / kTileM);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);   // the leader's expect_tx arrive; both CTAs' bytes count as tx
      mbar_init(&empty[s], 1);  // the leader's MMA commit (multicast to both)
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is the one used)
    }
    fence_mbar_init();
    tma_prefetch_desc(&xmap);
    tma_prefetch_desc(&wmap);
  }
  if (threadIdx.x == 0) FTRACE(4096, 0);
  if (warp == 1) tmem_alloc_cg2(&tslot, static_cast<uint32_t>(2 * bn));
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = tslot;
  griddep_launch_dependents();  // as in fwd_gemm_kernel

  if (warp == 0) {
    if (elect_one()) {
      bool waited = p.exts == nullptr;
      if (waited) griddep_wait();
      const uint32_t lead_full0 = map_cta(smem_u32(&full[0]), 0);
      int i = 0;
      for (int g = pair_id; g < p.num_tiles; g += npairs) {
        const int pi = g / p.ntn;
        const int t = 2 * pi + rank;
        const int n0 = (g % p.ntn) * bn;
        const int nh = n0 + rank * hb;  // this CTA's half of the N tile
        // K order rotated per N tile: the CTAs that share a row tile then read
        // different A blocks at any moment instead of all hitting the same L2 lines
        if (bk2) {
          for (int j = 0; j < (p.nkb + 1) / 2; ++j, ++i) {
            const int s = i % S;
            mbar_wait(&empty[s], (static_cast<uint32_t>(i / S) & 1u) ^ 1u);
            uint8_t* a = sm + s * kStage;
            uint8_t* b = a + kA;
            const uint32_t lf = lead_full0 + static_cast<uint32_t>(s) * 8u;
            if (leader) mbar_arrive_expect_tx(&full[s], 2u * kStage);
            tma_load_3d_cg2(a, &xmap, lf, 0, t * kTileM, 2 * j);
            for (int c = 0; c < hb; c += 64) tma_load_3d_cg2(b + c * 256, &wmap, lf, nh + c, j * 2 * kBK, p.layer);
          }
        } else {
        const int rot = p.krot ? (g % p.ntn) % p.nkb : 0;
        for (int j = 0; j < p.nkb; ++j, ++i) {
          const int kb = j + rot < p.nkb ? j + rot : j + rot - p.nkb;
          const int s = i % S;
          mbar_wait(&empty[s], (static_cast<uint32_t>(i / S) & 1u) ^ 1u);
          uint8_t* a = sm + s * kStage;
          uint8_t* b = a + kFwdA;
          const uint32_t lf = lead_full0 + static_cast<uint32_t>(s) * 8u;
          if (leader) mbar_arrive_expect_tx(&full[s], 2u * kStage);
          tma_load_2d_cg2(a, &xmap, lf, kb * kBK, t * kTileM);
          for (int c = 0; c < hb; c += 64) tma_load_3d_cg2(b + c * 128, &wmap, lf, nh + c, kb * kBK, p.layer);
        }
        }
        if (p.exts == nullptr) continue;
        for (int e = p.pext_begin[pi]; e < p.pext_begin[pi + 1]; ++e, ++i) {
          if (!waited) {
            griddep_wait();  // the A images are the shrink launch's output
            waited = true;
          }
          // Both CTAs: their own A image (or the zero image) and their half of
          // the up^T chunk, by TMA onto the leader's barrier.
          const int mine = p.pext[2 * e + rank];
          const FwdExt& x = p.exts[p.pext[2 * e] >= 0 ? p.pext[2 * e] : p.pext[2 * e + 1]];
          const int s = i % S;
          mbar_wait(&empty[s], (static_cast<uint32_t>(i / S) & 1u) ^ 1u);
          uint8_t* a = sm + s * kStage;
          uint8_t* b = a + kFwdA;
          const uint32_t lf = lead_full0 + static_cast<uint32_t>(s) * 8u;
          const uint32_t boxc = static_cast<uint32_t>(min(4, x.r_pad / 8));  // up^T core-matrix columns per row group
          if (leader) mbar_arrive_expect_tx(&full[s], 2u * (kFwdA + static_cast<uint32_t>(hb / 8) * boxc * 128u));
          const int img = mine >= 0 ? static_cast<int>(p.exts[mine].a_off >> 14) : p.zero_img;
          tma_load_2d_cg2(a, &amap, lf, 0, img * kTileM);
          const int g_pad = static_cast<int>(x.up_ls / x.r_pad / 8);
          tma_load_3d_cg2(b, p.umaps + x.umap, lf, 0, 4 * x.kc, p.layer * g_pad + nh / 8);
        }
        (void)row_tiles;
      }
      griddep_launch_dependents();
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader && elect_one()) {
      const uint32_t idesc_main = idesc_bf16(256, static_cast<uint32_t>(bn), 0, 1);
      const uint32_t idesc_ext = idesc_bf16(256, static_cast<uint32_t>(bn));
      int i = 0, it = 0;
      for (int g = pair_id; g < p.num_tiles; g += npairs, ++it) {
        const int pi = g / p.ntn;
        const int acc = it & 1;
        mbar_wait(&tempty[acc], (static_cast<uint32_t>(it >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem + static_cast<uint32_t>(acc * bn);
        if (bk2) {
          for (int j = 0; j < (p.nkb + 1) / 2; ++j, ++i) {
            const int s = i % S;
            mbar_wait_cluster(&full[s], static_cast<uint32_t>(i / S) & 1u);
            tc_fence_after();
            const uint32_t a = smem_u32(sm + s * kStage), b = a + kA;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              mma_bf16_cg2(d, smem_desc(a + (k >> 2) * kFwdA + (k & 3) * 32, 16, 1024, kLayoutSW128),
                           smem_desc(b + k * 2048, 16384, 1024, kLayoutSW128), idesc_main, (j > 0 || k > 0) ? 1u : 0u);
            }
            mma_commit_cg2(&empty[s], 3);
          }
        }
        for (int kb = 0; kb < (bk2 ? 0 : p.nkb); ++kb, ++i) {
          const int s = i % S;
          mbar_wait_cluster(&full[s], static_cast<uint32_t>(i / S) & 1u);
          tc_fence_after();
          const uint32_t a = smem_u32(sm + s * kStage), b = a + kFwdA;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            mma_bf16_cg2(d, smem_desc(a + k * 32, 16, 1024, kLayoutSW128), smem_desc(b + k * 2048, 8192, 1024, kLayoutSW128),
                         idesc_main, (kb > 0 || k > 0) ? 1u : 0u);
          }
          mma_commit_cg2(&empty[s], 3);
        }
        if (p.exts != nullptr) {
          for (int e = p.pext_begin[pi]; e < p.pext_begin[pi + 1]; ++e, ++i) {
            const int e0 = p.pext[2 * e] >= 0 ? p.pext[2 * e] : p.pext[2 * e + 1];
            const int kk = p.exts[e0].kk;
            const int s = i % S;
            mbar_wait_cluster(&full[s], static_cast<uint32_t>(i / S) & 1u);
            tc_fence_after();
            const uint32_t a = smem_u32(sm + s * kStage), b = a + kFwdA;
            // A image: 2 kk columns [hi | lo] (SBO 2 kk x 16 B); up^T: 4 core-matrix columns per row group
            const uint32_t sbo_a = static_cast<uint32_t>(kk) * 32u;
            const uint32_t sbo_b = static_cast<uint32_t>(min(4, p.exts[e0].r_pad / 8)) * 128u;
            for (int k = 0; k < kk / 16; ++k) {
              const uint64_t bd = smem_desc(b + k * 256, 128, sbo_b, kLayoutNone);
              mma_bf16_cg2(d, smem_desc(a + k * 256, 128, sbo_a, kLayoutNone), bd, idesc_ext, 1u);
              mma_bf16_cg2(d, smem_desc(a + kk * 16 + k * 256, 128, sbo_a, kLayoutNone), bd, idesc_ext, 1u);
            }
            mma_commit_cg2(&empty[s], 3);
          }
        }
        mma_commit_cg2(&tfull[acc], 3);
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3;
    int it = 0;
    for (int g = pair_id; g < p.num_tiles; g += npairs, ++it) {
      const int pi = g / p.ntn;
      const int t = 2 * pi + rank;
      const int n0 = (g % p.ntn) * bn;
      const int acc = it & 1;
      const int64_t srow = int64_t(t) * kTileM + q * 32 + lane;
      const bool rv = srow < p.n;
      const int64_t orow = rv && p.out_rows ? p.out_rows[srow] : srow;
      mbar_wait_sleep(&tfull[acc], static_cast<uint32_t>(it >> 1) & 1u, 32);
      tc_fence_after();
      const uint32_t tbase = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * bn);
      for (int c = 0; c < bn; c += 32) {
        uint32_t v[32];
        tmem_ld32(tbase + static_cast<uint32_t>(c), v);
        tmem_wait_ld();
        if (rv) {
#pragma unroll
          for (int gg = 0; gg < 4; ++gg) {
            float a8[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) a8[j] = __uint_as_float(v[8 * gg + j]);
            if (n0 + c + 8 * gg < p.d) store8(p, orow, n0 + c + 8 * gg, a8);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) {
          mbar_arrive(&tempty[acc]);
        } else {
          mbar_arrive_remote(&tempty[acc], 0, 1);
        }
      }
    }
  }
  if (threadIdx.x == 64) FTRACE(4096, 6);
  tc_fence_before();
  cluster_sync();  // no CTA leaves while its peer may still arrive / read its smem
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_cg2(tmem, static_cast<uint32_t>(2 * bn));
  }
}

cudaError_t launch_fwd_gemm_pair(const CUtensorMap& xmap, const CUtensorMap& wmap, const CUtensorMap& amap,
                                 const FwdParams& p, int grid, size_t smem, cudaStream_t stream) {
  cudaError_t e = cudaFuncSetAttribute(fwd_gemm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kFwdThreads, 1, 1);
  cfg.gridDim = dim3(static_cast<unsigned>(grid), 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = fwd_pdl() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, fwd_gemm_pair_kernel, xmap, wmap, amap, p);
}

int fwd_gemm_max_clusters(size_t smem, int csize) {
  static std::mutex mu;
  static std::map<std::pair<int, std::pair<size_t, int>>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({dev, {smem, csize}});
    if (it != cache.end()) return it->second;
  }
  if (cudaFuncSetAttribute(fwd_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
      cudaSuccess)
    return 0;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(csize);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kFwdThreads, 1, 1);
  cfg.gridDim = dim3(static_cast<unsigned>(csize), 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, fwd_gemm_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  std::lock_guard<std::mutex> lk(mu);
  cache[{dev, {smem, csize}}] = n;
  return n;
}

int fwd_gemm_pair_max_clusters(size_t smem) {
  // the occupancy query is slow: cache it per (device, smem)
  static std::mutex mu;
  static std::map<std::pair<int, size_t>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({dev, smem});
    if (it != cache.end()) return it->second;
  }
  if (cudaFuncSetAttribute(fwd_gemm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
      cudaSuccess)
    return 0;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kFwdThreads, 1, 1);
  cfg.gridDim = dim3(2, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, fwd_gemm_pair_kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  std::lock_guard<std::mutex> lk(mu);
  cache[{dev, smem}] = n;
  return n;
}

}  // namespace atmm
