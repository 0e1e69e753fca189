// stream_kernels.cu -- atmm_stream_kernel: the whole batched-LoRA bypass
// (shrink, fixed-order mid reduction, expand + residual) of EVERY tile of a
// plan in ONE persistent launch, one CTA per SM.
//
// Reference: run_bypass (batch.hpp:48-81: per segment gather -> X.down ->
// .up -> scatter) fused with the residual add_inplace(next, bypass)
// (model.hpp:239-241).
//
// Why one launch: the split pair (kernels.cu) runs the shrink and then the
// expand as two persistent grids, one CTA per SM each, so the expand's Y rows
// -- two thirds of the step's bytes -- start moving only as shrink CTAs
// retire; the all-to-all kernel runs one 8-CTA cluster per tile and leaves
// SMs idle when a batch has few tiles.  Here every CTA owns a balanced share
// of BOTH work lists (StreamParams) and streams them through two rings at
// once:
//   warps 0..3   shrink loaders: X rows of a (tile, 64-wide K block) unit by
//                16-byte cp.async into a 128-byte-swizzled A image, the
//                down^T block by one bulk copy;
//   warps 4..7   expand loaders: the 128-column up^T slice of a (tile,
//                128 columns) unit by one bulk copy, its Y rows by cp.async;
//   warp 8       TMEM owner + tcgen05.mma issuer (shrink units, then expand
//                units: swap-AB D[col][row] = up^T . mid^T);
//   warps 9..12  epilogue: shrink partials TMEM -> L2 slot + release count;
//                per expanded tile: acquire the tile's count, sum the
//                partials in FIXED slot order (deterministic) into a bf16
//                mid in shared memory; Y[row][col] += s * acc.
// Ring completion uses cp.async.mbarrier.arrive.noinc (every loader thread
// arrives once its own copies of the stage have landed) plus the bulk
// copy's transaction bytes, so each loader runs as far ahead as its ring.
//
// Progress: a CTA publishes all of its shrink partials before its epilogue
// waits on any tile, and the grid is at most one CTA per SM (co-resident),
// so every awaited count is eventually reached.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "device_types.hpp"
#include "ptx.cuh"

namespace atmm {

using namespace ptx;

namespace {

constexpr int kStreamMaxStages = 16;
constexpr uint32_t kStreamWarpMMA = 8;
constexpr uint32_t kStreamWarpEpi = 9;
constexpr int kStreamThreads = 13 * 32;

__device__ __forceinline__ uint32_t pack_bf16x2_s(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ uint64_t globaltimer_s() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define SSTRACE(ev)                                                                           \
  do {                                                                                        \
    if (p.trace) p.trace[static_cast<size_t>(blockIdx.x) * kTraceEvents + (ev)] = globaltimer_s(); \
  } while (0)

// Byte offset of element (row i, col j) of a K-major "interleave" operand of
// K = kpad columns: [i/8][j/8] core matrices of 8 rows x 16 B.
__device__ __forceinline__ uint32_t ileave_off(uint32_t i, uint32_t j, uint32_t kpad) {
  return (i >> 3) * (kpad * 16u) + (j >> 3) * 128u + (i & 7u) * 16u + (j & 7u) * 2u;
}

__device__ __forceinline__ int32_t ld_acquire_gpu(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_gpu_add(int32_t* p, int32_t v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace

template <typename YT>
__global__ void __launch_bounds__(kStreamThreads, 1) atmm_stream_kernel(const StreamParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  __shared__ uint64_t bars[4 * kStreamMaxStages + 12];
  __shared__ uint32_t tmem_slot;
  __shared__ int32_t yrows_s[kTileM];  // expand loaders: rows of their current tile
  __shared__ int32_t erows_s[kTileM];  // epilogue: rows of its current tile
  constexpr int kEsz = static_cast<int>(sizeof(YT));
  constexpr int kCols = 128;  // expand unit width (tcgen05 M of the swap-AB expand)
  const uint32_t tid = threadIdx.x;
  const uint32_t warp = tid >> 5;
  const uint32_t lane = tid & 31;
  const int SS = p.sstages, ES = p.estages;
  uint64_t* sfull = bars;                            // [SS] 128 loader arrivals + bulk tx
  uint64_t* sempty = sfull + kStreamMaxStages;       // [SS] MMA commit
  uint64_t* efull = sempty + kStreamMaxStages;       // [ES] 128 loader arrivals + bulk tx
  uint64_t* eempty = efull + kStreamMaxStages;       // [ES] 128 epilogue arrivals
  uint64_t* sacc_full = eempty + kStreamMaxStages;   // [2] MMA commit
  uint64_t* sacc_empty = sacc_full + 2;              // [2] 128 epilogue arrivals
  uint64_t* eacc_full = sacc_empty + 2;              // [2] MMA commit
  uint64_t* eacc_empty = eacc_full + 2;              // [2] 128 epilogue arrivals
  uint64_t* mid_full = eacc_empty + 2;               // [2] 128 epilogue arrivals
  uint64_t* mid_empty = mid_full + 2;                // [2] MMA commit
  const int b = static_cast<int>(blockIdx.x);
  const int s_beg = p.s_begin[b], s_end = p.s_begin[b + 1];
  const int e_beg = p.e_begin[b], e_end = p.e_begin[b + 1];
  const uint32_t scols = static_cast<uint32_t>(p.r_pad_max);  // one shrink accumulator
  const uint32_t ecols = static_cast<uint32_t>((p.rows_max + 15) & ~15);
  const uint32_t e_tmem0 = 2 * scols;

  if (tid == 0) SSTRACE(0);
  if (warp == 0) {
    for (int i = static_cast<int>(lane); i < 4 * kStreamMaxStages + 12; i += 32) {
      uint32_t cnt = 1;
      if (i < kStreamMaxStages || (i >= 2 * kStreamMaxStages && i < 3 * kStreamMaxStages)) cnt = 129;  // full
      else if (i >= 3 * kStreamMaxStages && i < 4 * kStreamMaxStages) cnt = 128;                      // eempty
      else if (i >= 4 * kStreamMaxStages) {
        const int k = i - 4 * kStreamMaxStages;  // sacc_full, sacc_empty, eacc_full, eacc_empty, mid_full, mid_empty
        cnt = (k >= 2 && k < 4) || (k >= 6 && k < 8) || (k >= 8 && k < 10) ? 128u : 1u;
      }
      mbar_init(&bars[i], cnt);
    }
    fence_mbar_init();
  }
  if (warp == kStreamWarpMMA) tmem_alloc(&tmem_slot, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_slot;
  const uint32_t smem0 = smem_u32(smem);
  // The next launch may take SMs as CTAs of this one retire; it waits for
  // this grid (griddepcontrol.wait) before it reads anything we write.
  griddep_launch_dependents();

  if (warp < 4) {
    // ===================== shrink loaders =====================
    // X chunk (row, ch): ch = tid & 7 fixed, rows (tid >> 3) + 16 i.
    const int ch = static_cast<int>(tid & 7);
    const int r0 = static_cast<int>(tid >> 3);
    // down^T blocks are weights (not written by the previous launch): the
    // first ring round goes out before griddepcontrol.wait.
    if (tid == 0) {
      for (int item = s_beg; item < min(s_end, s_beg + SS); ++item) {
        const int t = item / p.nkb;
        const int kb = item - t * p.nkb;
        const TileDesc tile = p.tiles[t];
        const int st = item - s_beg;
        const uint32_t bytes = static_cast<uint32_t>(tile.r_pad * kBK * 2);
        mbar_arrive_expect_tx(&sfull[st], bytes);
        bulk_g2s(smem + static_cast<size_t>(st) * p.s_stage_bytes + p.s_a_bytes,
                 tile.down_t + static_cast<int64_t>(p.layer) * tile.down_layer_stride + static_cast<int64_t>(kb) * tile.r_pad * kBK,
                 bytes, &sfull[st]);
      }
    }
    if (!p.x_ready) griddep_wait();  // X may be written by the previous launch
    int cur_t = -1, rows = 0;
    int64_t xoff[8];
    for (int item = s_beg; item < s_end; ++item) {
      const int j = item - s_beg;
      const int t = item / p.nkb;
      const int kb = item - t * p.nkb;
      if (t != cur_t) {
        const TileDesc tile = p.tiles[t];
        cur_t = t;
        rows = tile.rows;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = r0 + 16 * i;
          xoff[i] = r < rows ? static_cast<int64_t>(p.row_index[tile.row_begin + r]) * p.ldx : 0;
        }
      }
      const int st = j % SS;
      mbar_wait(&sempty[st], static_cast<uint32_t>(((j / SS) & 1) ^ 1));
      const uint32_t A = smem0 + static_cast<uint32_t>(st) * p.s_stage_bytes;
      // columns past d_in (last K block) are zero-filled, never read
      const int col = kb * kBK + ch * 8;
      const uint32_t nb = static_cast<uint32_t>(max(0, min(8, p.d_in - col)) * 2);
      const uint16_t* xk = p.x + (nb ? col : 0);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = r0 + 16 * i;
        if (r < rows) cp_async16(A + static_cast<uint32_t>(r * 128 + ((ch ^ (r & 7)) << 4)), xk + xoff[i], nb);
      }
      if (tid == 0 && j >= SS) {
        const TileDesc& tile = p.tiles[t];
        const uint32_t bytes = static_cast<uint32_t>(tile.r_pad * kBK * 2);
        mbar_arrive_expect_tx(&sfull[st], bytes);
        bulk_g2s(smem + static_cast<size_t>(st) * p.s_stage_bytes + p.s_a_bytes,
                 tile.down_t + static_cast<int64_t>(p.layer) * tile.down_layer_stride + static_cast<int64_t>(kb) * tile.r_pad * kBK,
                 bytes, &sfull[st]);
      }
      cp_async_arrive_noinc(&sfull[st]);
    }
    if (tid == 0) SSTRACE(1);
  } else if (warp < 8) {
    // ===================== expand loaders =====================
    const int et = static_cast<int>(tid) - 128;
    if (et == 0) {
      for (int item = e_beg; item < min(e_end, e_beg + ES); ++item) {
        const int t = item / p.nsl;
        const int n0 = (item - t * p.nsl) * kCols;
        const TileDesc tile = p.tiles[t];
        const int st = item - e_beg;
        const uint32_t bytes = static_cast<uint32_t>(kCols * tile.r_pad * 2);
        mbar_arrive_expect_tx(&efull[st], bytes);
        bulk_g2s(smem + p.off_e + static_cast<size_t>(st) * p.e_stage_bytes,
                 tile.up_t + static_cast<int64_t>(p.layer) * tile.up_layer_stride + static_cast<int64_t>(n0 >> 3) * tile.r_pad * 8,
                 bytes, &efull[st]);
      }
    }
    griddep_wait();  // Y is written by the previous launch
    if (et == 0) SSTRACE(9);
    const uint32_t up_bytes = static_cast<uint32_t>(kCols * p.r_pad_max * 2);
    const int64_t ldy_b = p.ldy * kEsz;
    int cur_t = -1;
    for (int item = e_beg; item < e_end; ++item) {
      const int j = item - e_beg;
      const int t = item / p.nsl;
      const int n0 = (item - t * p.nsl) * kCols;
      const int ncols = min(kCols, p.d_out - n0);
      const TileDesc tile = p.tiles[t];
      if (t != cur_t) {  // the tile's Y row offsets, once (no dependent loads in the copy loop)
        cur_t = t;
        named_bar_sync(2, 128);
        yrows_s[et] = et < tile.rows ? p.row_index[tile.row_begin + et] : 0;
        named_bar_sync(2, 128);
      }
      const int st = j % ES;
      mbar_wait(&eempty[st], static_cast<uint32_t>(((j / ES) & 1) ^ 1));
      const uint32_t U = smem0 + p.off_e + static_cast<uint32_t>(st) * p.e_stage_bytes;
      const uint32_t Yb = U + up_bytes;
      if (et == 0 && j >= ES) {
        const uint32_t bytes = static_cast<uint32_t>(kCols * tile.r_pad * 2);
        mbar_arrive_expect_tx(&efull[st], bytes);
        bulk_g2s(smem + p.off_e + static_cast<size_t>(st) * p.e_stage_bytes,
                 tile.up_t + static_cast<int64_t>(p.layer) * tile.up_layer_stride + static_cast<int64_t>(n0 >> 3) * tile.r_pad * 8,
                 bytes, &efull[st]);
      }
      const int cpr = ncols * kEsz / 16;  // 16-byte chunks per row
      const uint8_t* yb = reinterpret_cast<const uint8_t*>(p.y) + static_cast<int64_t>(n0) * kEsz;
      const int total = tile.rows * cpr;
      for (int q = et; q < total; q += 128) {
        const int r = q / cpr;
        const int c = q - r * cpr;
        cp_async16(Yb + static_cast<uint32_t>(r * kCols * kEsz + c * 16), yb + static_cast<int64_t>(yrows_s[r]) * ldy_b + c * 16, 16u);
      }
      cp_async_arrive_noinc(&efull[st]);
    }
    if (et == 0) SSTRACE(2);
  } else if (warp == kStreamWarpMMA) {
    // ===================== MMA issuer =====================
    int seg = 0, r_pad = 16, rt = -1;
    for (int item = s_beg; item < s_end; ++item) {
      const int j = item - s_beg;
      const int t = item / p.nkb;
      const int kb = item - t * p.nkb;
      const bool first = item == s_beg || kb == 0;
      const bool last = item == s_end - 1 || kb == p.nkb - 1;
      if (t != rt) {
        rt = t;
        r_pad = p.tiles[t].r_pad;
      }
      const int buf = seg & 1;
      if (first) mbar_wait(&sacc_empty[buf], static_cast<uint32_t>(((seg >> 1) & 1) ^ 1));
      const int st = j % SS;
      mbar_wait(&sfull[st], static_cast<uint32_t>((j / SS) & 1));
      tc_fence_after();
      fence_proxy_async_smem();
      if (j == 0 && lane == 0) SSTRACE(6);
      if (elect_one()) {
        const uint32_t A = smem0 + static_cast<uint32_t>(st) * p.s_stage_bytes;
        const uint64_t ad0 = smem_desc(A, 16u, 1024u, kLayoutSW128);
        const uint64_t bd0 = smem_desc(A + p.s_a_bytes, 128u, 1024u, kLayoutNone);
        const uint32_t idesc = idesc_bf16(kTileM, static_cast<uint32_t>(r_pad));
        const uint32_t d = tmem_base + static_cast<uint32_t>(buf) * scols;
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk) {
          mma_bf16(d, ad0 + static_cast<uint64_t>(kk * 2), bd0 + static_cast<uint64_t>(kk * 16), idesc,
                   (first && kk == 0) ? 0u : 1u);
        }
        mma_commit(&sempty[st]);
        if (last) mma_commit(&sacc_full[buf]);
      }
      __syncwarp();
      if (last) ++seg;
    }
    if (lane == 0) SSTRACE(7);
    int cur_t = -1, mt = -1, rows16 = 16;
    for (int item = e_beg; item < e_end; ++item) {
      const int j = item - e_beg;
      const int t = item / p.nsl;
      if (t != cur_t) {
        const TileDesc& tile = p.tiles[t];
        rows16 = (tile.rows + 15) & ~15;
        r_pad = tile.r_pad;
        cur_t = t;
        ++mt;
        mbar_wait(&mid_full[mt & 1], static_cast<uint32_t>((mt >> 1) & 1));
      }
      const bool tile_last = item == e_end - 1 || (item + 1) / p.nsl != t;
      const int st = j % ES;
      const int buf = j & 1;
      mbar_wait(&eacc_empty[buf], static_cast<uint32_t>(((j >> 1) & 1) ^ 1));
      mbar_wait(&efull[st], static_cast<uint32_t>((j / ES) & 1));
      tc_fence_after();
      fence_proxy_async_smem();
      if (elect_one()) {
        const uint32_t U = smem0 + p.off_e + static_cast<uint32_t>(st) * p.e_stage_bytes;
        const uint32_t M = smem0 + p.off_mid + static_cast<uint32_t>(mt & 1) * p.mid_bytes;
        const uint32_t sbo = static_cast<uint32_t>(r_pad) * 16u;
        const uint64_t ad0 = smem_desc(U, 128u, sbo, kLayoutNone);
        const uint64_t bd0 = smem_desc(M, 128u, sbo, kLayoutNone);
        const uint32_t idesc = idesc_bf16(kTileM, static_cast<uint32_t>(rows16));
        const uint32_t d = tmem_base + e_tmem0 + static_cast<uint32_t>(buf) * ecols;
        for (int kk = 0; kk < r_pad / 16; ++kk) {
          mma_bf16(d, ad0 + static_cast<uint64_t>(kk * 16), bd0 + static_cast<uint64_t>(kk * 16), idesc, kk > 0 ? 1u : 0u);
        }
        mma_commit(&eacc_full[buf]);
        if (tile_last) mma_commit(&mid_empty[mt & 1]);
      }
      __syncwarp();
      if (j == 0 && lane == 0) SSTRACE(11);
    }
  } else {
    // ===================== epilogue (warps 9..12) =====================
    const uint32_t quad = warp & 3u;
    const int et = static_cast<int>(tid) - static_cast<int>(kStreamWarpEpi) * 32;  // 0..127
    const int row = static_cast<int>(quad * 32 + lane);
    const int T = p.num_tiles;
    // (1) shrink segment partials -> L2 slots, release-counted per tile
    int seg = 0;
    for (int item = s_beg; item < s_end; ++item) {
      const int t = item / p.nkb;
      const int kb = item - t * p.nkb;
      if (!(item == s_end - 1 || kb == p.nkb - 1)) continue;  // act at segment ends
      const TileDesc& tile = p.tiles[t];
      const int rows = tile.rows;
      const int r_pad = tile.r_pad;
      const int buf = seg & 1;
      mbar_wait_sleep(&sacc_full[buf], static_cast<uint32_t>((seg >> 1) & 1), 64);
      tc_fence_after();
      const int sidx = seg == 0 ? p.seg_slot0[b] : 0;
      float* slot = p.part + (static_cast<int64_t>(p.part_off[t] + sidx) * kTileM) * p.r_pad_max;
      if (static_cast<int>(quad * 32) < rows) {
        for (int g = 0; g < r_pad; g += 16) {
          uint32_t v[16];
          tmem_ld16(tmem_base + ((quad * 32u) << 16) + static_cast<uint32_t>(buf) * scols + static_cast<uint32_t>(g), v);
          tmem_wait_ld();
          if (row < rows) {
            float4* dst = reinterpret_cast<float4*>(slot + static_cast<int64_t>(row) * p.r_pad_max + g);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              __stcg(dst + q, make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                          __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3])));
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&sacc_empty[buf]);
      named_bar_sync(1, 128);  // every epilogue thread's partial rows are written
      if (et == 0) {
        __threadfence();
        red_release_gpu_add(p.counter + t, 1);
      }
      ++seg;
    }
    if (et == 0) SSTRACE(3);
    // (2) expand units: per new tile, acquire + fixed-order reduction -> mid slot
    int cur_t = -1, mt = -1;
    float s = 0.f;
    int rows = 0, rows16 = 0, row_begin = 0;
    bool traced = false;
    for (int item = e_beg; item < e_end; ++item) {
      const int j = item - e_beg;
      const int t = item / p.nsl;
      const int n0 = (item - t * p.nsl) * kCols;
      const int ncols = min(kCols, p.d_out - n0);
      if (t != cur_t) {
        const TileDesc& tile = p.tiles[t];
        cur_t = t;
        ++mt;
        rows = tile.rows;
        rows16 = (rows + 15) & ~15;
        row_begin = tile.row_begin;
        s = p.scale * tile.scale;
        const int r_pad = tile.r_pad;
        const int nsg = p.nseg[t];
        mbar_wait(&mid_empty[mt & 1], static_cast<uint32_t>(((mt >> 1) & 1) ^ 1));
        erows_s[et] = et < rows ? p.row_index[row_begin + et] : 0;  // read after the barrier below
        if (et == 0) {
          while (ld_acquire_gpu(p.counter + t) < nsg) __nanosleep(20);
          if (!traced) {
            traced = true;
            SSTRACE(4);
          }
        }
        named_bar_sync(1, 128);
        const float* base = p.part + static_cast<int64_t>(p.part_off[t]) * kTileM * p.r_pad_max;
        const int64_t seg_stride = static_cast<int64_t>(kTileM) * p.r_pad_max;
        const uint32_t M = smem0 + p.off_mid + static_cast<uint32_t>(mt & 1) * p.mid_bytes;
        // items = (row, 4 ranks): every thread issues all of its partial
        // loads before the first add (latency bound: ~1 L2 round trip)
        const int cpr4 = r_pad / 4;
        const int nit = rows * cpr4;
        for (int it0 = et; it0 < nit; it0 += 256) {
          float4 a[2];
          const float* src[2];
          int rr[2], c4[2];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int it = min(it0 + 128 * q, nit - 1);
            rr[q] = it / cpr4;
            c4[q] = it - rr[q] * cpr4;
            src[q] = base + static_cast<int64_t>(rr[q]) * p.r_pad_max + c4[q] * 4;
            a[q] = make_float4(0.f, 0.f, 0.f, 0.f);
          }
          for (int g0 = 0; g0 < nsg; g0 += 8) {
            float4 v[2][8];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                v[q][k] = g0 + k < nsg ? __ldcg(reinterpret_cast<const float4*>(src[q] + (g0 + k) * seg_stride))
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
              }
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
#pragma unroll
              for (int k = 0; k < 8; ++k) {  // fixed slot order
                a[q].x += v[q][k].x;
                a[q].y += v[q][k].y;
                a[q].z += v[q][k].z;
                a[q].w += v[q][k].w;
              }
            }
          }
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (it0 + 128 * q < nit) {
              const uint32_t dst = M + ileave_off(static_cast<uint32_t>(rr[q]), static_cast<uint32_t>(c4[q] * 4), static_cast<uint32_t>(r_pad));
              asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(dst), "r"(pack_bf16x2_s(a[q].x, a[q].y)),
                           "r"(pack_bf16x2_s(a[q].z, a[q].w))
                           : "memory");
            }
          }
        }
        fence_proxy_async_smem();  // mid (generic writes) -> the tensor core
        mbar_arrive(&mid_full[mt & 1]);
        if (mt == 0 && et == 0) SSTRACE(8);
        named_bar_sync(1, 128);  // every thread's partial reads are done
        if (et == 0) {
          const int done = atomicAdd(p.counter + T + t, 1);
          if (done == p.ncons[t] - 1) {  // last consumer: reset for the next launch
            atomicExch(p.counter + t, 0);
            atomicExch(p.counter + T + t, 0);
          }
        }
      }
      const int st = j % ES;
      const int buf = j & 1;
      mbar_wait(&efull[st], static_cast<uint32_t>((j / ES) & 1));  // Y rows landed
      mbar_wait(&eacc_full[buf], static_cast<uint32_t>((j >> 1) & 1));
      tc_fence_after();
      const uint8_t* Yg = smem + p.off_e + static_cast<size_t>(st) * p.e_stage_bytes + static_cast<size_t>(kCols * p.r_pad_max * 2);
      const int m = row;  // output column n0 + m of this thread
      const uint16_t* ysm16 = reinterpret_cast<const uint16_t*>(Yg) + m;
      const uint32_t* ysm32 = reinterpret_cast<const uint32_t*>(Yg) + m;
      const bool col_ok = m < ncols;
      uint8_t* ycol = reinterpret_cast<uint8_t*>(p.y) + static_cast<int64_t>(n0 + m) * kEsz;
      const int64_t ldy_b = p.ldy * kEsz;
      for (int rb = 0; rb < rows16; rb += 32) {
        uint32_t acc[32];
        const uint32_t taddr = tmem_base + ((quad * 32u) << 16) + e_tmem0 + static_cast<uint32_t>(buf) * ecols + static_cast<uint32_t>(rb);
        if (rows16 - rb >= 32) {
          tmem_ld32(taddr, acc);
        } else {
          tmem_ld16(taddr, *reinterpret_cast<uint32_t(*)[16]>(&acc[0]));
        }
        const int nr = min(32, rows - rb);
        // the 32 rows' Y values first (independent shared loads), then the stores
        uint32_t yv[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          yv[i] = 0;
          if (i < nr) {
            if constexpr (kEsz == 2) {
              yv[i] = ysm16[(rb + i) * kCols];
            } else {
              yv[i] = ysm32[(rb + i) * kCols];
            }
          }
        }
        const int myrow = erows_s[rb + static_cast<int>(lane)];  // lane i: row rb + i
        tmem_wait_ld();
        if (nr == 32) {  // full block: no per-row branches; row offsets by shuffle
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int r = __shfl_sync(0xffffffffu, myrow, i);
            uint8_t* gp = ycol + static_cast<int64_t>(r) * ldy_b;
            if constexpr (kEsz == 2) {
              const float v = fmaf(s, __uint_as_float(acc[i]), __uint_as_float(yv[i] << 16));
              if (col_ok) *reinterpret_cast<uint16_t*>(gp) = __bfloat16_as_ushort(__float2bfloat16_rn(v));
            } else {
              if (col_ok) *reinterpret_cast<float*>(gp) = fmaf(s, __uint_as_float(acc[i]), __uint_as_float(yv[i]));
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int r = __shfl_sync(0xffffffffu, myrow, i);
            if (i < nr && col_ok) {
              uint8_t* gp = ycol + static_cast<int64_t>(r) * ldy_b;
              if constexpr (kEsz == 2) {
                const float v = fmaf(s, __uint_as_float(acc[i]), __uint_as_float(yv[i] << 16));
                *reinterpret_cast<uint16_t*>(gp) = __bfloat16_as_ushort(__float2bfloat16_rn(v));
              } else {
                *reinterpret_cast<float*>(gp) = fmaf(s, __uint_as_float(acc[i]), __uint_as_float(yv[i]));
              }
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&eacc_empty[buf]);
      mbar_arrive(&eempty[st]);
      if (j == 0 && et == 0) SSTRACE(10);
    }
    if (et == 0) SSTRACE(5);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kStreamWarpMMA) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

template __global__ void atmm_stream_kernel<__nv_bfloat16>(const StreamParams);
template __global__ void atmm_stream_kernel<float>(const StreamParams);

int stream_threads() { return kStreamThreads; }

cudaError_t launch_stream(int y_dtype, const StreamParams& p, int grid, size_t smem, cudaStream_t stream) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kStreamThreads, 1, 1);
  cfg.gridDim = dim3(static_cast<unsigned>(grid), 1, 1);
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.dynamicSmemBytes = smem;
  if (y_dtype == 0) {
    auto k = atmm_stream_kernel<__nv_bfloat16>;
    static thread_local size_t set_bf16 = 0;
    if (smem > set_bf16) {
      cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      if (e != cudaSuccess) return e;
      set_bf16 = smem;
    }
    return cudaLaunchKernelEx(&cfg, k, p);
  }
  auto k = atmm_stream_kernel<float>;
  static thread_local size_t set_f32 = 0;
  if (smem > set_f32) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    set_f32 = smem;
  }
  return cudaLaunchKernelEx(&cfg, k, p);
}

}  // namespace atmm
