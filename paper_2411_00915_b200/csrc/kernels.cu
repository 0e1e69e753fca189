// kernels.cu -- sm_100a kernels of the ATMM hot path.
//
//  atmm_bypass_kernel : fused batched-LoRA bypass, one thread-block CLUSTER
//      per tile of <= 128 rows of one segment (rows share an adapter):
//        shrink   mid = X_tile . down        K = d_in split across the C CTAs,
//                 X rows gathered by TMA tile::gather4, tcgen05 into TMEM;
//        reduce   the C fp32 partials of mid are reduced through DSMEM in a
//                 FIXED order (deterministic, no atomics) and broadcast as
//                 bf16 to every CTA's shared memory -- mid never leaves chip;
//        expand   Y[rows, Nslice] += s * mid . up   N = d_out split across
//                 the CTAs, tcgen05 into TMEM (double buffered), epilogue
//                 reads TMEM, scales, adds into Y (fp32 math, one rounding).
//      Reference: run_bypass (batch.hpp:48-81) + the residual add
//      add_inplace(next, bypass) (model.hpp:239-241).
//
//  atmm_merge_kernel : W (+)= alpha * A . B with a read-modify-write
//      epilogue; A = down (MN-major operand built from the down^T layout),
//      B = up^T.  Reference: delta_w_into + add/sub_inplace
//      (model.hpp:120-125,144-188); also serves atmm_multiply (atmm.hpp:111)
//      with beta = 0.
//
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM owner +
// single-thread tcgen05.mma issuer, warps 2..5 = epilogue (warp w reads TMEM
// lanes 32*(w%4) .. +31, one tile row per thread).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device_types.hpp"
#include "ptx.cuh"

namespace atmm {

using namespace ptx;

namespace {

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float bf16lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

// Byte offset of element (row i, col j) in a K-major "interleave" operand of
// K = kpad columns: [i/8][j/8] core matrices of 8 rows x 16 B.
__device__ __forceinline__ uint32_t interleave_off(uint32_t i, uint32_t j, uint32_t kpad) {
  return (i >> 3) * (kpad * 16u) + (j >> 3) * 128u + (i & 7u) * 16u + (j & 7u) * 2u;
}

// Y[row, col0 .. col0+32) += s * acc[0..32) ; fp32 math, one rounding.
template <typename YT>
__device__ __forceinline__ void epilogue_store32(YT* yrow, int col0, int d_out, float s,
                                                 const uint32_t (&acc)[32]);

template <>
__device__ __forceinline__ void epilogue_store32<__nv_bfloat16>(__nv_bfloat16* yrow, int col0,
                                                                int d_out, float s,
                                                                const uint32_t (&acc)[32]) {
  if (col0 + 32 <= d_out) {
    uint4* p = reinterpret_cast<uint4*>(yrow + col0);
    uint4 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = p[q];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t w[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float lo = fmaf(s, __uint_as_float(acc[q * 8 + 2 * e]), bf16lo(w[e]));
        const float hi = fmaf(s, __uint_as_float(acc[q * 8 + 2 * e + 1]), bf16hi(w[e]));
        w[e] = pack_bf16x2(lo, hi);
      }
      p[q] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (col0 + j < d_out) {
        const float y = __bfloat162float(yrow[col0 + j]);
        yrow[col0 + j] = __float2bfloat16_rn(fmaf(s, __uint_as_float(acc[j]), y));
      }
    }
  }
}

template <>
__device__ __forceinline__ void epilogue_store32<float>(float* yrow, int col0, int d_out, float s,
                                                        const uint32_t (&acc)[32]) {
  if (col0 + 32 <= d_out) {
    float4* p = reinterpret_cast<float4*>(yrow + col0);
    float4 v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = p[q];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      v[q].x = fmaf(s, __uint_as_float(acc[4 * q + 0]), v[q].x);
      v[q].y = fmaf(s, __uint_as_float(acc[4 * q + 1]), v[q].y);
      v[q].z = fmaf(s, __uint_as_float(acc[4 * q + 2]), v[q].z);
      v[q].w = fmaf(s, __uint_as_float(acc[4 * q + 3]), v[q].w);
      p[q] = v[q];
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (col0 + j < d_out) yrow[col0 + j] = fmaf(s, __uint_as_float(acc[j]), yrow[col0 + j]);
    }
  }
}

// W[row, col0..+32) = beta*W + alpha*acc
template <typename WT>
__device__ __forceinline__ void merge_store32(WT* wrow, int col0, int n, float alpha, float beta,
                                              const uint32_t (&acc)[32]);
template <>
__device__ __forceinline__ void merge_store32<float>(float* wrow, int col0, int n, float alpha,
                                                     float beta, const uint32_t (&acc)[32]) {
  if (col0 + 32 <= n) {
    float4* p = reinterpret_cast<float4*>(wrow + col0);
    float4 v[8];
    if (beta != 0.0f) {
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = p[q];
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      v[q].x = fmaf(alpha, __uint_as_float(acc[4 * q + 0]), v[q].x);
      v[q].y = fmaf(alpha, __uint_as_float(acc[4 * q + 1]), v[q].y);
      v[q].z = fmaf(alpha, __uint_as_float(acc[4 * q + 2]), v[q].z);
      v[q].w = fmaf(alpha, __uint_as_float(acc[4 * q + 3]), v[q].w);
      p[q] = v[q];
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (col0 + j < n) {
        const float w = beta != 0.0f ? wrow[col0 + j] : 0.0f;
        wrow[col0 + j] = fmaf(alpha, __uint_as_float(acc[j]), w);
      }
    }
  }
}
template <>
__device__ __forceinline__ void merge_store32<__nv_bfloat16>(__nv_bfloat16* wrow, int col0, int n,
                                                             float alpha, float beta,
                                                             const uint32_t (&acc)[32]) {
  if (col0 + 32 <= n) {
    uint4* p = reinterpret_cast<uint4*>(wrow + col0);
    uint4 v[4];
    if (beta != 0.0f) {
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = p[q];
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t w[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float lo = fmaf(alpha, __uint_as_float(acc[q * 8 + 2 * e]), bf16lo(w[e]));
        const float hi = fmaf(alpha, __uint_as_float(acc[q * 8 + 2 * e + 1]), bf16hi(w[e]));
        w[e] = pack_bf16x2(lo, hi);
      }
      p[q] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (col0 + j < n) {
        const float w = beta != 0.0f ? __bfloat162float(wrow[col0 + j]) : 0.0f;
        wrow[col0 + j] = __float2bfloat16_rn(fmaf(alpha, __uint_as_float(acc[j]), w));
      }
    }
  }
}

}  // namespace

// =========================================================================
// Fused bypass kernel
// =========================================================================
template <typename YT>
__global__ void __launch_bounds__(kBypassThreads, 1)
    atmm_bypass_kernel(const __grid_constant__ CUtensorMap tmap_x, const BypassParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;

  const uint32_t C = cluster_nctarank();
  const uint32_t crank = cluster_ctarank();
  const TileDesc tile = p.tiles[cluster_id_x()];
  const SlotDesc slot = p.slots[tile.slot];
  const int rows = tile.rows;
  const int r_pad = slot.r_pad;
  const uint16_t* down_t = slot.down_t + static_cast<int64_t>(p.layer) * slot.down_layer_stride;
  const uint16_t* up_t = slot.up_t + static_cast<int64_t>(p.layer) * slot.up_layer_stride;

  // K blocks (64 wide) and N units (32 wide) owned by this CTA.
  const int nkb = (p.d_in + kBK - 1) / kBK;
  const int kb_lo = (nkb * static_cast<int>(crank)) / static_cast<int>(C);
  const int kb_hi = (nkb * static_cast<int>(crank + 1)) / static_cast<int>(C);
  const int nun = (p.d_out + kNUnit - 1) / kNUnit;
  const int nu_lo = (nun * static_cast<int>(crank)) / static_cast<int>(C);
  const int nu_hi = (nun * static_cast<int>(crank + 1)) / static_cast<int>(C);
  const int n_lo = nu_lo * kNUnit;
  const int n_hi = nu_hi * kNUnit;
  const int num_chunks = (n_hi - n_lo + p.bn - 1) / p.bn;

  // Owner partition of the tile rows for the DSMEM reduction.
  const int R = (rows + static_cast<int>(C) - 1) / static_cast<int>(C);
  const int own_lo = min(rows, static_cast<int>(crank) * R);
  const int own_hi = min(rows, static_cast<int>(crank + 1) * R);
  const int owned = own_hi - own_lo;

  uint8_t* ring = smem;
  float* red = reinterpret_cast<float*>(smem + p.off_red);
  uint8_t* mid = smem + p.off_mid;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  const int S = p.stages;
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* shrink_full = bars + 2 * S;
  uint64_t* acc_full = bars + 2 * S + 1;   // [2]
  uint64_t* acc_empty = bars + 2 * S + 3;  // [2]
  uint64_t* red_full = bars + 2 * S + 5;
  uint64_t* mid_full = bars + 2 * S + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 7);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(shrink_full, 1);
    mbar_init(&acc_full[0], 1);
    mbar_init(&acc_full[1], 1);
    mbar_init(&acc_empty[0], 4);
    mbar_init(&acc_empty[1], 4);
    mbar_init(red_full, owned > 0 ? static_cast<uint32_t>(owned) * C : 1u);
    mbar_init(mid_full, static_cast<uint32_t>(rows * (r_pad / 8)));
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) tma_prefetch_desc(&tmap_x);
  if (warp == 1) tmem_alloc(tmem_slot, p.tmem_cols);
  tc_fence_before();
  cluster_sync();  // barrier inits + TMEM address visible cluster-wide
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const uint32_t a_bytes_per_group = 4u * kBK * 2u;  // one gather4 = 4 rows x 128 B
  const int ngroups = (rows + 3) / 4;

  if (warp == 0) {
    // ===================== TMA producer =====================
    YT* y = reinterpret_cast<YT*>(p.y);
    // Warm L2 with this CTA's Y slice and up^T slice: independent of the
    // shrink, so their HBM reads overlap it.
    const int n_hi_c = min(n_hi, p.d_out);
    if (n_hi_c > n_lo) {
      const uint32_t ybytes = static_cast<uint32_t>((n_hi_c - n_lo) * sizeof(YT)) & ~15u;
      for (int i = static_cast<int>(lane); i < rows; i += 32) {
        const int64_t row = p.row_index[tile.row_begin + i];
        if (ybytes) prefetch_l2(y + row * p.ldy + n_lo, ybytes);
      }
    }
    if (lane == 0 && n_hi > n_lo) {
      prefetch_l2(up_t + static_cast<int64_t>(n_lo) * r_pad,
                  static_cast<uint32_t>((n_hi - n_lo) * r_pad * 2));
    }
    // Row coordinates of this lane's gather4 group (constant over K).
    int32_t gr[4] = {0, 0, 0, 0};
    if (static_cast<int>(lane) < ngroups) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = min(static_cast<int>(lane) * 4 + q, rows - 1);
        gr[q] = p.row_index[tile.row_begin + i];
      }
    }
    const uint32_t b_bytes = static_cast<uint32_t>(r_pad) * kBK * 2u;
    const uint32_t a_bytes = static_cast<uint32_t>(ngroups) * a_bytes_per_group;
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = kb_lo; kb < kb_hi; ++kb) {
      uint8_t* st = ring + static_cast<size_t>(stage) * p.stage_bytes;
      if (lane == 0) {
        mbar_wait(&empty[stage], phase ^ 1u);
        mbar_arrive_expect_tx(&full[stage], a_bytes + b_bytes);
      }
      __syncwarp();
      if (static_cast<int>(lane) < ngroups) {
        tma_gather4(st + lane * a_bytes_per_group, &tmap_x, &full[stage], kb * kBK, gr[0], gr[1],
                    gr[2], gr[3]);
      }
      if (lane == 0) {
        bulk_g2s(st + kTileM * kBK * 2, down_t + static_cast<int64_t>(kb) * r_pad * kBK, b_bytes,
                 &full[stage]);
      }
      if (++stage == S) {
        stage = 0;
        phase ^= 1u;
      }
    }
    // Expand operand: up^T rows [n0, n0 + bn_c) of the CTA's N slice.
    for (int c = 0; c < num_chunks; ++c) {
      const int n0 = n_lo + c * p.bn;
      const int bn_c = min(p.bn, n_hi - n0);
      if (lane == 0) {
        uint8_t* st = ring + static_cast<size_t>(stage) * p.stage_bytes;
        const uint32_t bytes = static_cast<uint32_t>(bn_c * r_pad * 2);
        mbar_wait(&empty[stage], phase ^ 1u);
        mbar_arrive_expect_tx(&full[stage], bytes);
        bulk_g2s(st, up_t + static_cast<int64_t>(n0) * r_pad, bytes, &full[stage]);
      }
      if (++stage == S) {
        stage = 0;
        phase ^= 1u;
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t idesc_s = idesc_bf16(kTileM, static_cast<uint32_t>(r_pad));
      for (int kb = kb_lo; kb < kb_hi; ++kb) {
        uint8_t* st = ring + static_cast<size_t>(stage) * p.stage_bytes;
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t a0 = smem_u32(st);
        const uint32_t b0 = smem_u32(st + kTileM * kBK * 2);
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk) {
          const uint64_t ad = smem_desc(a0 + kk * 32u, 16u, 1024u, kLayoutSW128);
          const uint64_t bd = smem_desc(b0 + kk * 256u, 128u, 1024u, kLayoutNone);
          mma_bf16(tmem_base, ad, bd, idesc_s, (kb > kb_lo || kk > 0) ? 1u : 0u);
        }
        mma_commit(&empty[stage]);
        if (++stage == S) {
          stage = 0;
          phase ^= 1u;
        }
      }
      mma_commit(shrink_full);
      // Wait for the reduced bf16 mid (written through DSMEM by the owners).
      mbar_wait_cluster(mid_full, 0);
      tc_fence_after();
      fence_proxy_async_smem();
      const uint32_t mid0 = smem_u32(mid);
      const uint32_t sbo = static_cast<uint32_t>(r_pad) * 16u;
      for (int c = 0; c < num_chunks; ++c) {
        const int n0 = n_lo + c * p.bn;
        const int bn_c = min(p.bn, n_hi - n0);
        const int buf = c & 1;
        mbar_wait(&acc_empty[buf], ((c >> 1) & 1) ^ 1u);
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t b0 = smem_u32(ring + static_cast<size_t>(stage) * p.stage_bytes);
        const uint32_t idesc_e = idesc_bf16(kTileM, static_cast<uint32_t>(bn_c));
        for (int kk = 0; kk < r_pad / 16; ++kk) {
          const uint64_t ad = smem_desc(mid0 + kk * 256u, 128u, sbo, kLayoutNone);
          const uint64_t bd = smem_desc(b0 + kk * 256u, 128u, sbo, kLayoutNone);
          mma_bf16(tmem_base + static_cast<uint32_t>(buf * p.bn), ad, bd, idesc_e,
                   kk > 0 ? 1u : 0u);
        }
        mma_commit(&empty[stage]);
        mma_commit(&acc_full[buf]);
        if (++stage == S) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
    __syncwarp();
  } else {
    // ===================== epilogue (warps 2..5) =====================
    const uint32_t quad = warp & 3u;
    const int row_local = static_cast<int>(quad * 32 + lane);
    const bool valid = row_local < rows;
    const uint32_t lane_addr = (quad * 32u) << 16;
    const int ew = static_cast<int>(warp) - 2;
    const bool warp_active = static_cast<int>(quad * 32) < rows;

    // ---- shrink partial: TMEM -> registers ----
    mbar_wait(shrink_full, 0);
    tc_fence_after();
    uint32_t part[kMaxRank];
    if (warp_active) {
#pragma unroll
      for (int g = 0; g < kMaxRank / 32; ++g) {
        if (g * 32 < r_pad) {
          if (r_pad - g * 32 >= 32) {
            uint32_t v[32];
            tmem_ld32(tmem_base + lane_addr + g * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) part[g * 32 + j] = v[j];
          } else {
            uint32_t v[16];
            tmem_ld16(tmem_base + lane_addr + g * 32, v);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 16; ++j) part[g * 32 + j] = v[j];
          }
        }
      }
    }
    tc_fence_before();
    const uint32_t mid_s = smem_u32(mid);

    if (C == 1) {
      // Single CTA: the partial is the whole mid; write it as bf16.
      if (valid) {
#pragma unroll
        for (int ch = 0; ch < kMaxRank / 8; ++ch) {
          if (ch < r_pad / 8) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              w[e] = pack_bf16x2(__uint_as_float(part[ch * 8 + 2 * e]),
                                 __uint_as_float(part[ch * 8 + 2 * e + 1]));
            }
            st_cluster_v4(mid_s + interleave_off(row_local, ch * 8, r_pad), w[0], w[1], w[2],
                          w[3]);
          }
        }
      }
      fence_proxy_async_cluster();
      __syncwarp();
      const uint32_t nvalid = __popc(__ballot_sync(0xffffffffu, valid));
      if (lane == 0 && nvalid) {
        fence_acq_rel_cluster();
        mbar_arrive_remote(mid_full, crank, nvalid * static_cast<uint32_t>(r_pad / 8));
      }
    } else {
      // ---- 1. scatter fp32 partial rows to their owners' slots ----
      const int owner = valid ? row_local / R : -1;
      if (valid) {
        float* slot_row =
            red + (static_cast<size_t>(crank) * p.red_rows + (row_local - owner * R)) * r_pad;
        const uint32_t dst = map_cta(smem_u32(slot_row), static_cast<uint32_t>(owner));
#pragma unroll
        for (int j = 0; j < kMaxRank; j += 4) {
          if (j < r_pad) st_cluster_v4(dst + j * 4, part[j], part[j + 1], part[j + 2], part[j + 3]);
        }
      }
      __syncwarp();
      if (warp_active) {
        const int first_owner = (quad * 32) / R;
        const int last_row = min(rows - 1, static_cast<int>(quad * 32 + 31));
        const int last_owner = last_row / R;
        if (lane == 0) fence_acq_rel_cluster();
        for (int o = first_owner; o <= last_owner; ++o) {
          const uint32_t cnt = __popc(__ballot_sync(0xffffffffu, owner == o));
          if (lane == 0 && cnt) mbar_arrive_remote(red_full, static_cast<uint32_t>(o), cnt);
        }
      }
      // ---- 2. owner: fixed-order reduction of C partials, bf16 broadcast ----
      if (owned > 0) {
        mbar_wait_cluster(red_full, 0);
        const int cpr = r_pad / 8;  // 8-column chunks per row
        const int items = owned * cpr;
        for (int t = ew * 32 + static_cast<int>(lane); t < items; t += 128) {
          const int rl = t / cpr;
          const int ch = t - rl * cpr;
          float acc[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] = 0.0f;
          for (uint32_t c = 0; c < C; ++c) {
            const float4* src = reinterpret_cast<const float4*>(
                red + (static_cast<size_t>(c) * p.red_rows + rl) * r_pad + ch * 8);
            const float4 u = src[0];
            const float4 v = src[1];
            acc[0] += u.x;
            acc[1] += u.y;
            acc[2] += u.z;
            acc[3] += u.w;
            acc[4] += v.x;
            acc[5] += v.y;
            acc[6] += v.z;
            acc[7] += v.w;
          }
          const uint32_t w0 = pack_bf16x2(acc[0], acc[1]);
          const uint32_t w1 = pack_bf16x2(acc[2], acc[3]);
          const uint32_t w2 = pack_bf16x2(acc[4], acc[5]);
          const uint32_t w3 = pack_bf16x2(acc[6], acc[7]);
          const uint32_t off = mid_s + interleave_off(own_lo + rl, ch * 8, r_pad);
          for (uint32_t q = 0; q < C; ++q) st_cluster_v4(map_cta(off, q), w0, w1, w2, w3);
        }
        fence_proxy_async_cluster();
        __syncwarp();
        const int full_rounds = items / 128;
        const int rem = items - full_rounds * 128;
        const uint32_t cnt =
            static_cast<uint32_t>(full_rounds * 32 + max(0, min(32, rem - ew * 32)));
        if (lane == 0 && cnt) {
          fence_acq_rel_cluster();
          for (uint32_t q = 0; q < C; ++q) mbar_arrive_remote(mid_full, q, cnt);
        }
      }
    }

    // ---- 3. expand epilogue: Y += s * acc ----
    const float s = p.scale * slot.scale;
    YT* yrow = nullptr;
    if (valid) {
      yrow = reinterpret_cast<YT*>(p.y) +
             static_cast<int64_t>(p.row_index[tile.row_begin + row_local]) * p.ldy;
    }
    for (int c = 0; c < num_chunks; ++c) {
      const int n0 = n_lo + c * p.bn;
      const int bn_c = min(p.bn, n_hi - n0);
      const int buf = c & 1;
      mbar_wait(&acc_full[buf], (c >> 1) & 1);
      tc_fence_after();
      if (warp_active) {
        for (int sub = 0; sub < bn_c; sub += 32) {
          uint32_t v[32];
          tmem_ld32(tmem_base + lane_addr + static_cast<uint32_t>(buf * p.bn + sub), v);
          tmem_wait_ld();
          if (valid && n0 + sub < p.d_out) epilogue_store32<YT>(yrow, n0 + sub, p.d_out, s, v);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
  }

  __syncwarp();
  tc_fence_before();
  cluster_sync();  // no CTA leaves while a peer may still touch its smem
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

// =========================================================================
// Merge / GEMM kernel:  W = beta*W + alpha * A . B
//   A (M x K): MN-major operand assembled from the down^T blocked layout.
//   B (N x K): up^T blocked, K-major.
// Persistent: CTA b walks tiles t = b, b + grid, ... ; tile = (m-tile of 128
// rows, n-chunk of bn columns), n fastest so A is reused across n-chunks.
// =========================================================================
template <typename WT>
__global__ void __launch_bounds__(kMergeThreads, 1) atmm_merge_kernel(const MergeParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t lane = threadIdx.x & 31;
  const int S = p.stages;
  const int kp = p.k_pad;
  const int kg = kp / 8;  // K groups of 8

  uint8_t* a_buf = smem;              // 128 x kp bf16, MN-major interleave
  uint8_t* b_ring = smem + p.off_b;   // stages x (bn x kp bf16)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* a_full = bars + 2 * S;
  uint64_t* a_empty = bars + 2 * S + 1;
  uint64_t* acc_full = bars + 2 * S + 2;   // [2]
  uint64_t* acc_empty = bars + 2 * S + 4;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * S + 6);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(a_full, 1);
    mbar_init(a_empty, 1);
    mbar_init(&acc_full[0], 1);
    mbar_init(&acc_full[1], 1);
    mbar_init(&acc_empty[0], 4);
    mbar_init(&acc_empty[1], 4);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, p.tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int num_tiles = p.num_mtiles * p.num_nchunks;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int cur_mt = -1;
      uint32_t a_phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int mt = t / p.num_nchunks;
        const int nc = t - mt * p.num_nchunks;
        if (mt != cur_mt) {
          // A tile: 16 M-groups x kg K-groups of 128 B core matrices, copied
          // from the two 64-wide d_in blocks of the down^T layout.
          mbar_wait(a_empty, a_phase ^ 1u);
          mbar_arrive_expect_tx(a_full, static_cast<uint32_t>(128 * kp * 2));
          for (int h = 0; h < 2; ++h) {
            const int64_t kb = static_cast<int64_t>(mt) * 2 + h;
            for (int g = 0; g < kg; ++g) {
              bulk_g2s(a_buf + g * 2048 + h * 1024, p.a_t + (kb * kg + g) * 512, 1024u, a_full);
            }
          }
          a_phase ^= 1u;
          cur_mt = mt;
        }
        const int n0 = nc * p.bn;
        const int bn_c = min(p.bn, ((p.n + 31) / 32) * 32 - n0);
        const uint32_t bytes = static_cast<uint32_t>(bn_c * kp * 2);
        mbar_wait(&empty[stage], phase ^ 1u);
        mbar_arrive_expect_tx(&full[stage], bytes);
        bulk_g2s(b_ring + static_cast<size_t>(stage) * p.b_stage_bytes,
                 p.b_t + static_cast<int64_t>(n0) * kp, bytes, &full[stage]);
        if (++stage == S) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int cur_mt = -1;
      uint32_t a_phase = 0;
      int local = 0;
      const uint32_t a0 = smem_u32(a_buf);
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++local) {
        const int mt = t / p.num_nchunks;
        const int nc = t - mt * p.num_nchunks;
        const int n0 = nc * p.bn;
        const int bn_c = min(p.bn, ((p.n + 31) / 32) * 32 - n0);
        const int next_t = t + static_cast<int>(gridDim.x);
        const bool last_of_a = next_t >= num_tiles || (next_t / p.num_nchunks) != mt;
        if (mt != cur_mt) {
          mbar_wait(a_full, a_phase);
          a_phase ^= 1u;
          cur_mt = mt;
        }
        const int buf = local & 1;
        mbar_wait(&acc_empty[buf], ((local >> 1) & 1) ^ 1u);
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint32_t b0 = smem_u32(b_ring + static_cast<size_t>(stage) * p.b_stage_bytes);
        const uint32_t idesc = idesc_bf16(kTileM, static_cast<uint32_t>(bn_c), 1u, 0u);
        for (int kk = 0; kk < kp / 16; ++kk) {
          // A MN-major: M-group stride (SBO) 128 B, K-group stride (LBO) 2048 B.
          const uint64_t ad = smem_desc(a0 + kk * 4096u, 2048u, 128u, kLayoutNone);
          const uint64_t bd = smem_desc(b0 + kk * 256u, 128u, static_cast<uint32_t>(kp) * 16u,
                                        kLayoutNone);
          mma_bf16(tmem_base + static_cast<uint32_t>(buf * p.bn), ad, bd, idesc,
                   kk > 0 ? 1u : 0u);
        }
        mma_commit(&empty[stage]);
        mma_commit(&acc_full[buf]);
        if (last_of_a) mma_commit(a_empty);
        if (++stage == S) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
    __syncwarp();
  } else {
    const uint32_t quad = warp & 3u;
    const uint32_t lane_addr = (quad * 32u) << 16;
    int local = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++local) {
      const int mt = t / p.num_nchunks;
      const int nc = t - mt * p.num_nchunks;
      const int n0 = nc * p.bn;
      const int bn_c = min(p.bn, ((p.n + 31) / 32) * 32 - n0);
      const int row = mt * kTileM + static_cast<int>(quad * 32 + lane);
      const int buf = local & 1;
      mbar_wait(&acc_full[buf], (local >> 1) & 1);
      tc_fence_after();
      WT* wrow = reinterpret_cast<WT*>(p.w) + static_cast<int64_t>(row) * p.ldw;
      for (int sub = 0; sub < bn_c; sub += 32) {
        uint32_t v[32];
        tmem_ld32(tmem_base + lane_addr + static_cast<uint32_t>(buf * p.bn + sub), v);
        tmem_wait_ld();
        if (row < p.m && n0 + sub < p.n) merge_store32<WT>(wrow, n0 + sub, p.n, p.alpha, p.beta, v);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

// ---------------------------------------------------------------- utils --
__global__ void f32_to_bf16_kernel(const float* __restrict__ src, uint16_t* __restrict__ dst,
                                   int64_t rows, int64_t cols, int64_t lds, int64_t ldd) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols;
    const int64_t c = i - r * cols;
    __nv_bfloat16 b = __float2bfloat16_rn(src[r * lds + c]);
    dst[r * ldd + c] = *reinterpret_cast<uint16_t*>(&b);
  }
}

// Explicit instantiations reachable from the host launcher.
template __global__ void atmm_bypass_kernel<__nv_bfloat16>(const __grid_constant__ CUtensorMap,
                                                           const BypassParams);
template __global__ void atmm_bypass_kernel<float>(const __grid_constant__ CUtensorMap,
                                                   const BypassParams);
template __global__ void atmm_merge_kernel<float>(const MergeParams);
template __global__ void atmm_merge_kernel<__nv_bfloat16>(const MergeParams);

}  // namespace atmm

// =========================================================================
// Host-side launch helpers (kernel symbols live in this translation unit).
// =========================================================================
namespace atmm {

template <typename K>
static cudaError_t prepare(K kernel, size_t smem, bool nonportable) {
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  if (nonportable) {
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  return e;
}

cudaError_t launch_bypass(int y_dtype, const CUtensorMap& tmap, const BypassParams& p, int C,
                          int num_tiles, size_t smem, cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(C * num_tiles), 1, 1);
  cfg.blockDim = dim3(kBypassThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(C);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (y_dtype == 0) {
    auto k = atmm_bypass_kernel<__nv_bfloat16>;
    cudaError_t e = prepare(k, smem, C > 8);
    if (e != cudaSuccess) return e;
    return cudaLaunchKernelEx(&cfg, k, tmap, p);
  }
  auto k = atmm_bypass_kernel<float>;
  cudaError_t e = prepare(k, smem, C > 8);
  if (e != cudaSuccess) return e;
  return cudaLaunchKernelEx(&cfg, k, tmap, p);
}

int bypass_max_active_clusters(int C, size_t smem) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(C), 1, 1);
  cfg.blockDim = dim3(kBypassThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(C);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto k = atmm_bypass_kernel<__nv_bfloat16>;
  if (prepare(k, smem, C > 8) != cudaSuccess) return -1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess) return -1;
  return n;
}

cudaError_t launch_merge(int w_dtype, const MergeParams& p, int grid, size_t smem,
                         cudaStream_t stream) {
  if (w_dtype == 0) {
    auto k = atmm_merge_kernel<__nv_bfloat16>;
    cudaError_t e = prepare(k, smem, false);
    if (e != cudaSuccess) return e;
    k<<<grid, kMergeThreads, smem, stream>>>(p);
    return cudaGetLastError();
  }
  auto k = atmm_merge_kernel<float>;
  cudaError_t e = prepare(k, smem, false);
  if (e != cudaSuccess) return e;
  k<<<grid, kMergeThreads, smem, stream>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_f32_to_bf16(const float* src, uint16_t* dst, int64_t rows, int64_t cols,
                               int64_t lds, int64_t ldd, cudaStream_t stream) {
  const int64_t total = rows * cols;
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  f32_to_bf16_kernel<<<blocks > 0 ? blocks : 1, 256, 0, stream>>>(src, dst, rows, cols, lds, ldd);
  return cudaGetLastError();
}

}  // namespace atmm
