// device_types.hpp -- POD structs shared by the host launcher and the
// sm_100a kernels (no torch, no STL).
#pragma once

#include <cstdint>

#include <cuda.h>

namespace atmm {

constexpr int kTileM = 128;   // tcgen05 M (TMEM lanes); a tile carries <= 128 valid rows
constexpr int kBK = 64;       // K block per pipeline stage: one 128-byte swizzle row of bf16
constexpr int kNUnit = 64;    // expand N granule (one 128-byte Y row slice of bf16)
constexpr int kMaxRank = 128; // fused kernel limit on the LoRA rank
constexpr int kMaxCluster = 16;
constexpr int kSplitParts = 6;  // fp32-faithful path: K slices of the split operand images (precise_kernels.cu)
constexpr int kBypassThreads = 256;  // w0,w7 X/down TMA, w1 MMA + TMEM, w2-5 epilogue, w6 up/Y TMA
constexpr int kMergeThreads = 192;

// One cluster tile: <= 128 rows of one segment (rows = row_index[row_begin ..])
// with its adapter's factor pointers inlined, so a CTA needs one table load.
struct TileDesc {
  const uint16_t* down_t;     // layer-0 base (see SlotDesc)
  const uint16_t* up_t;
  int64_t down_layer_stride;  // elements
  int64_t up_layer_stride;
  int32_t row_begin;
  int32_t rows;
  int32_t r_pad;
  float scale;
  const uint16_t* up_t2 = nullptr;  // up^T with the columns of every (128 up_g)-column slice in MMA
                                    // order (column up_g m + j -> A row 128 j + m): one bulk copy per
                                    // slice in the split expand (up_g 2); layer stride
                                    // round_up(d_out, 128 up_g) r_pad
  int32_t x_row0 = -1;        // the tile's rows are X / Y rows x_row0 .. x_row0 + rows - 1 (one
                              // TMA box, split path), else -1 (gathered row by row)
  int32_t up_g = 0;           // the G of up_t2 (0: none)
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
  const uint16_t* x;    // n x d_in bf16, 16-byte aligned rows
  int64_t ldx;
  void* y;
  int64_t ldy;
  int32_t n_rows;       // batch rows (an out-of-range row coordinate drops TMA stores)
  int32_t d_in;
  int32_t d_out;
  int32_t layer;
  float scale;
  // shrink ring: stages x [A: a_bytes gathered X rows (128-byte swizzle) | B: 64 x r_pad down^T]
  int32_t stages;
  int32_t stage_bytes;
  int32_t a_bytes;
  // up^T ring: ustages x (bn x r_pad bf16)
  int32_t bn;           // expand chunk (columns per tcgen05.mma), multiple of 64
  int32_t ustages;
  int32_t ustage_bytes;
  // Y ring: ny x (rows x 128 B), 128-byte swizzle
  int32_t ny;
  int32_t ycols;        // columns per Y ring buffer (64 bf16 / 32 fp32)
  int32_t ybuf_bytes;
  int32_t red_rows;     // rows per owner slot (ceil(tile rows / C))
  int32_t r_pad_max;
  uint32_t off_up;
  uint32_t off_y;
  uint32_t off_red;
  uint32_t off_mid;
  uint32_t off_bar;
  uint32_t tmem_cols;
  int32_t y_vec;        // 1: Y rows 16-byte aligned -> 128-bit epilogue accesses
  int32_t y_ring;       // 1: Y staged through the smem ring (cp.async in, coalesced stores out)
  int32_t rep;          // replicas of the tile rows in the expand accumulator (128 / rows: 1, 2, 4)
  int32_t nbuf;         // expand accumulator buffers in TMEM (tmem_cols / bn)
  uint64_t* trace;      // debug: per-CTA phase timestamps (kTraceEvents each), or null
  // atmm_bypass_a2a_kernel only: Y slice buffer row pitch (bytes); off_y is
  // the buffer, off_up the whole up^T slice of the CTA.
  int32_t ypitch;
  int32_t gcols;        // output columns owned per epilogue thread (= expand MMAs per CTA: 1, 2, 4, 8)
  int32_t x_ready;      // 1: X is not written by the preceding launch (gathered before griddepcontrol.wait)
  // atmm_bypass_a2a_kernel only: 1 = the launcher proved that the preceding
  // launch on the stream (the only one that can still be running, see the
  // wait-before-trigger protocol in kernels.cu) touches none of this launch's
  // X / Y bytes -> X and Y are loaded before griddepcontrol.wait.
  int32_t early;
  // atmm_bypass_a2a_kernel only: [tile][kTileM] row indices of each tile
  // (rows past the tile's end repeat its last row), this launch's tiles.
  const int32_t* tile_rows;
};

constexpr int kTraceEvents = 32;

// Independent calls (X_c, Y_c, layer_c) of one plan fused into ONE launch of
// the all-to-all kernel (e.g. the q / k / v projections of a decoder layer):
// cluster id = call * num_tiles + tile.  Passed as a __grid_constant__
// parameter so the per-call X tensor maps live in parameter space.
constexpr int kMaxGroup = 8;
struct GroupArgs {
  CUtensorMap x_map[kMaxGroup];
  const void* x[kMaxGroup];
  void* y[kMaxGroup];
  int32_t layer[kMaxGroup];
  int32_t count;
  int32_t num_tiles;
};

// Split path (atmm_shrink_kernel + atmm_expand_kernel) for large batches.
// Both kernels are persistent (one CTA per SM) over host-balanced ranges of a
// flattened work list:
//   shrink items = (tile, 64-wide K block), tile-major.  CTA b runs items
//     [s_begin[b], s_begin[b+1]); the run of one tile inside one CTA is a
//     "segment" whose fp32 partial mid rows go to part[part_off[t] + slot]
//     (slots numbered in CTA order).  In the expand launch every CTA first
//     sums a share of the (tile, row, 4 columns) items over the tile's nseg[t]
//     partials in FIXED slot order, writes bf16 mid[t] in the expand's
//     B-operand (interleave) layout and adds its item count to the tile's
//     readiness counter.
//   expand items = (tile, 128 output columns), tile-major; CTA b runs items
//     [e_begin[b], e_begin[b+1]): Y[rows, cols] += s * mid . up.
// part / mid stay in L2 between the two launches.
struct SplitParams {
  const TileDesc* tiles;
  const int32_t* row_index;
  const uint16_t* x;   // n x d_in bf16
  int64_t ldx;
  void* y;             // n x d_out (bf16 or fp32)
  int64_t ldy;
  int32_t d_in;
  int32_t d_out;
  int32_t layer;
  float scale;
  int32_t num_tiles;
  int32_t nkb;           // 64-wide K blocks per tile
  int32_t expand_g;      // output columns per expand epilogue thread (items of 128 G columns)
  uint32_t e_tmem_cols;  // expand TMEM allocation: >= 2 x G x rows16 (two accumulators)
  int32_t out_staged;    // expand: update Y rows in shared memory, store them with 16-byte accesses
  int32_t contig;        // some tile has consecutive rows (TileDesc::x_row0): X / Y by TMA boxes
  int32_t early;         // shrink: compute before waiting for the preceding launch (the host proved
                         // it writes nothing the shrink reads); wait + release at the shrink's end
  int32_t r_pad_max;
  int32_t stages;        // shrink ring depth
  int32_t estages;       // expand ring depth
  int32_t y_dtype;       // 0 bf16, 1 fp32
  int32_t rows_max;
  const int32_t* s_begin;    // [grid + 1]
  const int32_t* e_begin;    // [grid + 1]
  const int32_t* seg_slot0;  // [grid] slot (within its tile) of the CTA's first segment
  const int32_t* nseg;       // [tile]
  const int32_t* part_off;   // [tile]
  float* part;               // [sum nseg][128][r_pad_max]
  uint16_t* mid;             // [tile][128 x r_pad_max] bf16, interleave layout
  int32_t* counter;          // [0] exited expand CTAs, [1] reserved, then [tile] reduced mid items (reset by the expand's last CTA)
  const int32_t* red_off;    // [tile + 1] prefix of rows x r_pad / 4 reduction items
  const int32_t* red_tile0;  // [grid] tile holding the CTA's first reduction item
  uint64_t* trace;
  const int32_t* tile_rows;  // [tile][kTileM] padded row lists of this launch's tiles
};

// Stream path (atmm_stream_kernel): the shrink AND the expand of every tile
// in ONE persistent launch, one CTA per SM.  Each CTA owns a host-balanced
// range of shrink units (tile, 64-wide K block) and, independently, a range
// of expand units (tile, 128 output columns); two loader groups stream both
// rings from the start, so the Y rows of the expand (2/3 of the bytes) are in
// flight while the shrink runs.  A tile's fp32 partial mid rows (one slot per
// CTA segment, as in SplitParams) are published with a release increment of
// counter[t]; every CTA that expands tile t waits for counter[t] == nseg[t],
// sums the partials in FIXED slot order into a bf16 mid in shared memory and
// runs its units.  The last consumer of a tile (ncons[t]) resets its
// counters for the next launch on the stream.
struct StreamParams {
  const TileDesc* tiles;
  const int32_t* row_index;
  const uint16_t* x;   // n x d_in bf16
  int64_t ldx;
  void* y;             // n x d_out (bf16 or fp32)
  int64_t ldy;
  int32_t d_in;
  int32_t d_out;
  int32_t layer;
  float scale;
  int32_t num_tiles;
  int32_t nkb;         // 64-wide K blocks per tile
  int32_t nsl;         // 128-column expand units per tile
  int32_t r_pad_max;
  int32_t rows_max;
  int32_t sstages;     // shrink ring depth (<= 16)
  int32_t estages;     // expand ring depth (<= 16)
  uint32_t s_stage_bytes;  // [X rows8_max x 128 B, 128-byte swizzle | down^T r_pad_max x 128 B]
  uint32_t s_a_bytes;      // rows8_max x 128
  uint32_t e_stage_bytes;  // [up^T 128 x r_pad_max | Y rows_max x 128 x esz]
  uint32_t off_e;          // expand ring
  uint32_t off_mid;        // 2 mid slots of mid_bytes
  uint32_t mid_bytes;
  uint32_t tmem_cols;
  int32_t x_ready;
  const int32_t* s_begin;    // [grid + 1]
  const int32_t* e_begin;    // [grid + 1]
  const int32_t* seg_slot0;  // [grid]
  const int32_t* nseg;       // [tile]
  const int32_t* part_off;   // [tile]
  const int32_t* ncons;      // [tile] CTAs whose expand range touches the tile
  float* part;               // [sum nseg][128][r_pad_max]
  int32_t* counter;          // [2 tiles]: published segments, finished consumers
  uint64_t* trace;
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
  int32_t w_vec;        // 1: W rows 16-byte aligned -> 128-bit epilogue accesses
  // TMA-staged W (atmm_merge_tma_kernel): W moves through an smem ring of
  // 128-row x 128-byte slabs (128-byte swizzle), loaded and stored by TMA.
  int32_t w_stages;
  uint32_t off_w;
  int32_t slab_cols;    // W columns per slab (64 bf16 / 32 fp32)
  int32_t num_layers;   // TMA-staged path: layers merged by one launch (W is a 3-D tensor map)
  int64_t a_layer_stride;  // elements between consecutive layers' down^T / up^T
  int64_t b_layer_stride;
};

// ---- layer forward (model.hpp:192-328): tanh(cur . W_l + bypass_l(cur)) ----
// Rows run in segment-sorted order (plan order, then the rows no segment
// covers) so a 128-row tile meets few adapters.  The bypass rides the base
// GEMM as extra K blocks: for every (tile, segment, 32-rank chunk) a
// "K-extension" block D += mid_chunk . up_chunk^T, where mid_chunk is the
// 128 x kk bf16 A image (rows outside the segment zero) written by the
// shrink launch and up_chunk is read straight from the registry.  Chunks
// are 32 ranks wide so the [hi | lo] A image (128 x 64 bf16) and the up^T
// slice (bn x 32 bf16) each fit one pipeline stage.
struct FwdExt {
  const uint16_t* down_t;  // slot down^T (layer 0), [kb][g][c][8x8]
  const uint16_t* up_t;    // slot up^T (layer 0),   [g][c][8x8]
  int64_t down_ls;         // elements per layer
  int64_t up_ls;
  int64_t a_off;           // byte offset of the A image in the ext buffer
  int32_t r_pad;
  int32_t kc;              // rank chunk: ranks [32 kc, 32 kc + kk)
  int32_t kk;              // 16 | 32
  int32_t lo, hi;          // tile-local rows [lo, hi) of the segment
  int32_t col;             // first TMEM / B-image column in its shrink item
  float scale;             // slot scale
  int32_t umap;            // pair GEMM: index of the slot's up^T tensor map
};
struct FwdItem {           // one shrink work item: a tile's chunks [e_begin, e_end)
  int32_t tile, e_begin, e_end, ncols;
};
struct FwdParams {
  uint8_t* ext;            // A images
  const FwdExt* exts;
  const int32_t* ext_begin;  // [row tiles + 1]
  const FwdItem* items;
  const int32_t* out_rows;   // sorted row -> output row (nullptr: identity)
  uint16_t* out;
  int64_t ldo;
  int64_t n, d;
  int32_t layer;
  int32_t bn;              // GEMM N tile (128 | 256)
  int32_t ntn;             // N tiles per row tile
  int32_t num_tiles;       // row tiles x ntn
  int32_t nkb;             // K blocks of the base GEMM (ceil(d / 64))
  int32_t ks;              // shrink K split (cluster size)
  int32_t num_items;
  int32_t stages;
  int32_t sbytes;            // shrink: B bytes per stage (max item columns x 128)
  int32_t pair;              // 1: fwd_gemm_pair_kernel (2-SM cta_group::2 tiles of 256 rows)
  // pair mode: the union of the two row tiles' K-extension chunks, per pair:
  // entries [pext_begin[pi], pext_begin[pi+1]) of pext = {ext index for rank 0,
  // ext index for rank 1} (-1: that row tile has no rows in the chunk -> zero image)
  const int32_t* pext;
  const int32_t* pext_begin;
  const uint8_t* zero_a;     // 16 KB of zeros
  const CUtensorMap* umaps;  // pair GEMM: per-slot up^T maps {64, r_pad/8, L * d_out_pad/8}, box {64, 4, bn/16}
  int32_t zero_img;          // pair GEMM: index of the zero A image (A images are 16 KB slots)
  int32_t kz;                // 1-SM GEMM split-K cluster size (1: none; > 1: one tile per cluster)
  int32_t act_none;          // 1: plain GEMM epilogue (no tanh)
  int32_t out_f32;           // plain GEMM: fp32 output (with act_none)
  int32_t mc;                // 1-SM GEMM A-multicast cluster size (1: none; exclusive with kz > 1)
  int32_t krot;              // 1: rotate each tile's K order by its N tile index (spreads A reads over L2)
  int32_t bk2;               // plain GEMM: 128-deep K stages (xmap 3-D {64, rows, K / 64}, wmap box 128 K rows)
  uint64_t* trace;           // debug: per-CTA %globaltimer events (atmm_debug_set_trace)
};

}  // namespace atmm
