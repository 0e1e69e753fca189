// device_types.hpp -- POD structs shared by the host launcher and the
// sm_100a kernels (no torch, no STL).
#pragma once

#include <cstdint>

namespace atmm {

constexpr int kTileM = 128;   // tcgen05 M (TMEM lanes); a tile carries <= 128 valid rows
constexpr int kBK = 64;       // K block per pipeline stage: one 128-byte swizzle row of bf16
constexpr int kNUnit = 32;    // expand N granule (one tcgen05.ld 32x32b.x32)
constexpr int kMaxRank = 128; // fused kernel limit on the LoRA rank
constexpr int kMaxCluster = 16;
constexpr int kBypassThreads = 192;  // w0 TMA producer, w1 MMA + TMEM, w2-5 epilogue
constexpr int kMergeThreads = 192;

// One cluster tile: <= 128 rows of one segment (rows = row_index[row_begin ..]).
struct TileDesc {
  int32_t row_begin;
  int32_t rows;
  int32_t slot;
  int32_t pad;
};

// One registry slot (adapter), device resident.  Factors are bf16 in the
// tcgen05 operand layouts:
//   down_t: per layer, [kb = d_in_pad/64][g = r_pad/8][c = 8][8 x 8]   (down^T blocked)
//   up_t:   per layer, [g = d_out_pad/8][c = r_pad/8][8 x 8]            (up^T blocked)
struct SlotDesc {
  const uint16_t* down_t;
  const uint16_t* up_t;
  int64_t down_layer_stride;  // elements
  int64_t up_layer_stride;    // elements
  int32_t rank;
  int32_t r_pad;
  float scale;
  int32_t pad;
};

struct BypassParams {
  const TileDesc* tiles;
  const int32_t* row_index;
  const SlotDesc* slots;
  void* y;
  int64_t ldy;
  int32_t d_in;
  int32_t d_out;
  int32_t layer;
  float scale;
  int32_t stages;
  int32_t bn;           // expand chunk (columns per tcgen05.mma), multiple of 32
  int32_t stage_bytes;  // multiple of 1024
  int32_t red_rows;     // rows per owner slot (ceil(tile_m / C))
  int32_t r_pad_max;
  uint32_t off_red;
  uint32_t off_mid;
  uint32_t off_bar;
  uint32_t tmem_cols;
};

struct MergeParams {
  const uint16_t* a_t;  // down^T blocked (MN-major A): [kb][g][c][8x8], K = r_pad
  const uint16_t* b_t;  // up^T blocked (K-major B):    [g][c][8x8]
  void* w;
  int64_t ldw;
  int32_t m;            // d_in
  int32_t n;            // d_out
  int32_t k_pad;        // r_pad (multiple of 16, <= 128)
  int32_t bn;
  int32_t stages;
  int32_t num_mtiles;
  int32_t num_nchunks;
  float alpha;
  float beta;           // 1: accumulate into W; 0: overwrite
  uint32_t off_b;
  uint32_t off_bar;
  uint32_t b_stage_bytes;
  uint32_t tmem_cols;
};

}  // namespace atmm
