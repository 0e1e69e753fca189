// device.cu -- the CUDA-runtime side of the C ABI: device registry of
// adapter factors, batch plans (routing tables in HBM), kernel launch
// resolution (shared memory carve-up, cluster size, TMEM columns), the
// host-buffer parity paths, merge/unmerge, the plain GEMM and the tuner's
// timing primitive.
//
// Reference (proj/include/loraserve/): adapter.hpp:18-110 (registry),
// batch.hpp:28-81 (plan_batch + run_bypass), model.hpp:120-188 (delta_w,
// merge, unmerge), atmm.hpp:111-154 (atmm_multiply_into), atmm.hpp:188-216
// (benchmark_config: median of trials after a warm-up).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <new>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "common.hpp"
#include "device_types.hpp"

namespace atmm {

// kernels.cu
cudaError_t launch_bypass(int y_dtype, const CUtensorMap& tmap_x, const CUtensorMap& tmap_y,
                          const BypassParams& p, int C, int num_tiles, size_t smem, cudaStream_t stream);
int bypass_max_active_clusters(int C, size_t smem);
cudaError_t launch_merge(int w_dtype, const MergeParams& p, int grid, size_t smem,
                         cudaStream_t stream);
cudaError_t launch_bypass_a2a(int y_dtype, const GroupArgs& ga, const BypassParams& p, int C, int num_tiles,
                              size_t smem, cudaStream_t stream);
cudaError_t launch_stream(int y_dtype, const StreamParams& p, int grid, size_t smem, cudaStream_t stream);
cudaError_t launch_permute_up_g2(const uint16_t* src, int64_t src_ls, uint16_t* dst, int64_t dst_ls, int64_t L,
                                 int64_t d_out_pad, int64_t d_out_pad2, int64_t r_pad, int64_t G, cudaStream_t stream);
cudaError_t launch_split(int y_dtype, const CUtensorMap& xtile, const CUtensorMap& ytile, const SplitParams& p, int grid,
                         size_t smem_s, size_t smem_e,
                         cudaStream_t stream);
cudaError_t launch_merge_tma(int w_dtype, const CUtensorMap& tmap_w, const MergeParams& p, int grid,
                             size_t smem, cudaStream_t stream);
cudaError_t launch_f32_to_bf16(const float* src, uint16_t* dst, int64_t rows, int64_t cols,
                               int64_t lds, int64_t ldd, cudaStream_t stream);
cudaError_t launch_scale_bf16_2d(uint16_t* base, int64_t rows, int64_t cols, int64_t ld, float f,
                                 cudaStream_t stream);
cudaError_t launch_fwd_gather(const uint16_t* x, int64_t ldx, uint16_t* dst, int64_t ldd, const int32_t* order,
                              int64_t n, int64_t d, cudaStream_t stream);
cudaError_t launch_fwd_shrink(const CUtensorMap& xmap, const FwdParams& p, size_t smem, cudaStream_t stream);
cudaError_t launch_fwd_gemm(const CUtensorMap& xmap, const CUtensorMap& wmap, const FwdParams& p, int grid, size_t smem,
                            cudaStream_t stream);
cudaError_t launch_fwd_gemm_pair(const CUtensorMap& xmap, const CUtensorMap& wmap, const CUtensorMap& amap,
                                 const FwdParams& p, int grid, size_t smem, cudaStream_t stream);
int fwd_gemm_pair_max_clusters(size_t smem);
int fwd_gemm_max_clusters(size_t smem, int csize);
cudaError_t launch_pack_factors(const float* down, const float* up, int64_t L, int64_t d_in, int64_t d_out,
                                int64_t r, int64_t d_in_pad, int64_t d_out_pad, int64_t r_pad, uint16_t* down_t,
                                uint16_t* up_t, cudaStream_t stream);

namespace {

constexpr size_t kSmemLimit = 232448;  // 227 KiB opt-in per CTA on sm_100
constexpr size_t kSmemPerSM = 233472;  // 228 KiB per SM
constexpr int kMaxStages = 6;

#define CUDA_CHECK(expr)                                                                  \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      fail(ATMM_ERR_CUDA, std::string(#expr) + " failed: " + cudaGetErrorString(e_));      \
    }                                                                                     \
  } while (0)

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

// No CPU fallback: every compute entry point requires an sm_100 device.
void require_device(int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    fail(ATMM_ERR_NO_DEVICE, "no CUDA device visible: the ATMM operator has no CPU fallback");
  }
  if (device < 0 || device >= count) fail(ATMM_ERR_NO_DEVICE, "device ordinal out of range");
  // cudaGetDeviceProperties costs milliseconds: check each device once
  static std::atomic<uint8_t> checked[64] = {};
  if (device < 64 && checked[device].load(std::memory_order_relaxed)) return;
  cudaDeviceProp prop;
  CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    fail(ATMM_ERR_NO_DEVICE, std::string("device ") + prop.name +
                                 " is not sm_100 (Blackwell B200); kernels are built for sm_100a only");
  }
  if (device < 64) checked[device].store(1, std::memory_order_relaxed);
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) CUDA_CHECK(cudaSetDevice(dev));
  }
  // Destructor paths (plan / registry teardown, possibly during process
  // exit after the CUDA runtime shut down) must never throw.
  DeviceGuard(int dev, std::nothrow_t) {
    if (cudaGetDevice(&prev) != cudaSuccess || (prev != dev && cudaSetDevice(dev) != cudaSuccess)) {
      cudaGetLastError();
      prev = -1;
    }
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// ---- TMA tensor map encode through the driver entry point (no -lcuda) ----
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      fn = reinterpret_cast<EncodeTiledFn>(p);
    }
  });
  if (!fn) fail(ATMM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// X (n x d_in bf16, row stride ldx): box = one 64-wide row slice, 128-byte
// swizzle; tile::gather4 loads 4 arbitrary rows per instruction.
CUtensorMap make_x_map(const void* x, int64_t n, int64_t d_in, int64_t ldx) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(d_in), static_cast<cuuint64_t>(n)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldx) * 2};
  const cuuint32_t box[2] = {kBK, 1};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x),
                                 dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(ATMM_ERR_CUDA, "cuTensorMapEncodeTiled(X) failed: " + std::to_string(r));
  return m;
}

// X as 128-row tiles (split shrink, tiles of consecutive rows): box = 128
// rows x one 64-wide K block, 128-byte swizzle = the K-major MMA operand.
CUtensorMap make_x_tile_map(const void* x, int64_t n, int64_t d_in, int64_t ldx) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(d_in), static_cast<cuuint64_t>(n)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldx) * 2};
  const cuuint32_t box[2] = {kBK, kTileM};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x),
                                 dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(ATMM_ERR_CUDA, "cuTensorMapEncodeTiled(X tiles) failed: " + std::to_string(r));
  return m;
}

// Y (n x d_out, bf16 or fp32): box = one 128-byte row slice, 128-byte
// swizzle, gathered 4 rows at a time into the kernel's Y ring.
CUtensorMap make_y_map(const void* y, int64_t n, int64_t d_out, int64_t ldy, int y_dtype) {
  CUtensorMap m;
  const int64_t esz = y_dtype == ATMM_BF16 ? 2 : 4;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(d_out), static_cast<cuuint64_t>(n)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldy * esz)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / esz), 1};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, y_dtype == ATMM_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                 2, const_cast<void*>(y), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(ATMM_ERR_CUDA, "cuTensorMapEncodeTiled(Y) failed: " + std::to_string(r));
  return m;
}

// Y as blocks of box_rows consecutive rows x box_cols columns (split expand,
// tiles of consecutive rows), no swizzle: the stage's dense Y rows.  Cached
// per thread like cached_map.
CUtensorMap y_tile_map(const void* y, int64_t n, int64_t d_out, int64_t ldy, int y_dtype, int box_cols, int box_rows) {
  struct Entry {
    const void* base = nullptr;
    int64_t n = 0, d = 0, ld = 0;
    int dt = 0, bc = 0, br = 0;
    CUtensorMap map;
  };
  thread_local Entry cache[4];
  thread_local int next = 0;
  for (const auto& e : cache) {
    if (e.base == y && e.n == n && e.d == d_out && e.ld == ldy && e.dt == y_dtype && e.bc == box_cols && e.br == box_rows) {
      return e.map;
    }
  }
  Entry& e = cache[next];
  next = (next + 1) % 4;
  const int64_t esz = y_dtype == ATMM_BF16 ? 2 : 4;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(d_out), static_cast<cuuint64_t>(n)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldy * esz)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&e.map, y_dtype == ATMM_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                 2, const_cast<void*>(y), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(ATMM_ERR_CUDA, "cuTensorMapEncodeTiled(Y tiles) failed: " + std::to_string(r));
  e.base = y;
  e.n = n;
  e.d = d_out;
  e.ld = ldy;
  e.dt = y_dtype;
  e.bc = box_cols;
  e.br = box_rows;
  return e.map;
}

// Small per-thread cache of encoded X / Y maps (kind 0: X rows, 1 + y_dtype:
// Y, 3: X tiles).
CUtensorMap cached_map(int kind, const void* base, int64_t rows, int64_t cols, int64_t ld) {
  struct Entry {
    const void* base;
    int64_t rows, cols, ld;
    int kind;
    CUtensorMap map;
  };
  thread_local Entry cache[8];
  thread_local int next = 0;
  thread_local bool init = false;
  if (!init) {
    for (auto& e : cache) e.base = nullptr;
    init = true;
  }
  for (const auto& e : cache) {
    if (e.base == base && e.rows == rows && e.cols == cols && e.ld == ld && e.kind == kind) return e.map;
  }
  Entry& e = cache[next];
  next = (next + 1) % 8;
  e.map = kind == 0   ? make_x_map(base, rows, cols, ld)
          : kind == 3 ? make_x_tile_map(base, rows, cols, ld)
                      : make_y_map(base, rows, cols, ld, kind - 1);
  e.base = base;
  e.rows = rows;
  e.cols = cols;
  e.ld = ld;
  e.kind = kind;
  return e.map;
}

// W (m x n, bf16 or fp32, row stride ldw) for the TMA-staged merge: box =
// 128 rows x one 128-byte column slab, 128-byte swizzle (loads and stores).
// 3-D over layers: (n, m, L) with layer stride w_ls elements (L = 1: one matrix).
CUtensorMap make_w_map(void* w, int64_t m, int64_t n, int64_t ldw, int w_dtype, int64_t L = 1, int64_t w_ls = 0) {
  CUtensorMap map;
  const int64_t esz = w_dtype == ATMM_BF16 ? 2 : 4;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(m), static_cast<cuuint64_t>(L)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(ldw * esz),
                                 static_cast<cuuint64_t>((L > 1 ? w_ls : ldw * m) * esz)};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(128 / esz), static_cast<cuuint32_t>(kTileM), 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode_fn()(&map, w_dtype == ATMM_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                 3, w, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(ATMM_ERR_CUDA, "cuTensorMapEncodeTiled(W) failed: " + std::to_string(r));
  return map;
}

// ---- host packing into the tcgen05 operand layouts ----
// down (d_in x r, row-major, ld) -> down^T blocked
//   [kb = d_in_pad/64][g = r_pad/8][c = 8][row = rank % 8][col = d_in % 8]
void pack_down_t(const float* down, int64_t d_in, int64_t r, int64_t ld, int64_t d_in_pad,
                 int64_t r_pad, uint16_t* out) {
  std::memset(out, 0, static_cast<size_t>(d_in_pad * r_pad) * 2);
  const int64_t G = r_pad / 8;
  for (int64_t i = 0; i < d_in; ++i) {
    const int64_t kb = i / 64, c = (i % 64) / 8, col = i % 8;
    for (int64_t j = 0; j < r; ++j) {
      const int64_t g = j / 8, row = j % 8;
      out[((kb * G + g) * 8 + c) * 64 + row * 8 + col] = f32_to_bf16(down[i * ld + j]);
    }
  }
}
// up (r x d_out, row-major, ld) -> up^T blocked
//   [g = d_out_pad/8][c = r_pad/8][row = d_out % 8][col = rank % 8]
void pack_up_t(const float* up, int64_t r, int64_t d_out, int64_t ld, int64_t d_out_pad,
               int64_t r_pad, uint16_t* out) {
  std::memset(out, 0, static_cast<size_t>(d_out_pad * r_pad) * 2);
  const int64_t Cc = r_pad / 8;
  for (int64_t j = 0; j < r; ++j) {
    const int64_t c = j / 8, col = j % 8;
    for (int64_t nn = 0; nn < d_out; ++nn) {
      const int64_t g = nn / 8, row = nn % 8;
      out[(g * Cc + c) * 64 + row * 8 + col] = f32_to_bf16(up[j * ld + nn]);
    }
  }
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  void alloc(size_t count) {
    release();
    if (count) CUDA_CHECK(cudaMalloc(&p, count * sizeof(T)));
    n = count;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

}  // namespace

// =========================================================================
// Registry
// =========================================================================
struct Slot {
  int32_t id = -1;
  int64_t rank = 0, r_pad = 0;
  int64_t alg_rank = 0;  // FLOP accounting rank: the true rank (a combined slot: the sum of its parts')
  int64_t total_rank = 0;  // the adapter's rank (> rank for chunk 0 of an adapter above kMaxRank)
  float scale = 1.0f;
  uint16_t* down_t = nullptr;
  uint16_t* up_t = nullptr;
  // up^T in the (128 G)-column MMA order for G = 2, 4, 8 (TileDesc::up_t2),
  // each made on a plan's first use of the slot with that G (stream-ordered
  // allocation, so free_slot may release it either way)
  uint16_t* up_tg[3] = {nullptr, nullptr, nullptr};
  bool live = false;
  bool async_owned = false;  // buffers from cudaMallocAsync (put_async): freed stream-ordered
  // fp32-faithful images (precise registries only), bf16 hi / lo splits per layer:
  // (kSplitParts K slices each, precise_kernels.cu)
  uint16_t* p_down_b = nullptr;  // [L][6 kpd x r8]   B-operand image of down (x . down)
  uint16_t* p_up_b = nullptr;    // [L][6 r8 x n8]    B-operand image of up   (mid . up, dW)
  uint16_t* p_down_a = nullptr;  // [L][d_in x 6 r8]  A-operand image of down (dW = down . up)
};

// Frees a slot's device buffers (stream-ordered when `async`: buffers from
// stream-ordered allocation, released after every earlier use on `st`).
static void free_slot(Slot& s, cudaStream_t st = nullptr, bool async = false) {
  for (uint16_t* p : {s.down_t, s.up_t, s.p_down_b, s.p_up_b, s.p_down_a, s.up_tg[0], s.up_tg[1], s.up_tg[2]}) {
    if (!p) continue;
    if (async) {
      cudaFreeAsync(p, st);
    } else {
      cudaFree(p);
    }
  }
  s.down_t = s.up_t = s.p_down_b = s.p_up_b = s.p_down_a = nullptr;
  s.up_tg[0] = s.up_tg[1] = s.up_tg[2] = nullptr;
}

}  // namespace atmm

using namespace atmm;

struct atmm_registry {
  std::mutex up2_mu;  // lazily made Slot::up_tg (plans may be built on several threads)
  int device = 0;
  int64_t L = 0, d_in = 0, d_out = 0, d_in_pad = 0, d_out_pad = 0;
  std::map<int32_t, int> slot_of;
  std::vector<Slot> slots;
  DevBuf<SlotDesc> d_slots;
  // put_async fp32 staging, one grow-only buffer per stream: a swap on
  // stream B never overwrites the buffer a pack kernel on stream A still reads.
  std::vector<std::pair<cudaStream_t, std::unique_ptr<DevBuf<float>>>> stage;
  DevBuf<float>& stage_for(cudaStream_t st) {
    for (auto& [s, b] : stage) {
      if (s == st) return *b;
    }
    stage.emplace_back(st, std::make_unique<DevBuf<float>>());
    return *stage.back().second;
  }
  uint64_t generation = 0;
  uint64_t uid = next_uid();  // process-unique (host-path plan cache key; addresses are reused)
  static uint64_t next_uid() {
    static std::atomic<uint64_t> c{1};
    return c.fetch_add(1);
  }
  bool precise = false;  // keep fp32-faithful factor images (atmm_registry_set_precise)

  ~atmm_registry() {
    DeviceGuard g(device, std::nothrow);
    for (auto& s : slots) free_slot(s);
  }
  void sync_slots() {
    std::vector<SlotDesc> h(slots.size());
    for (size_t i = 0; i < slots.size(); ++i) {
      const Slot& s = slots[i];
      h[i].down_t = s.down_t;
      h[i].up_t = s.up_t;
      h[i].down_layer_stride = d_in_pad * s.r_pad;
      h[i].up_layer_stride = d_out_pad * s.r_pad;
      h[i].rank = static_cast<int32_t>(s.rank);
      h[i].r_pad = static_cast<int32_t>(s.r_pad);
      h[i].scale = s.scale;
      h[i].pad = 0;
    }
    if (d_slots.n < h.size()) d_slots.alloc(std::max<size_t>(h.size(), 2 * d_slots.n));
    if (!h.empty()) CUDA_CHECK(cudaMemcpy(d_slots.p, h.data(), h.size() * sizeof(SlotDesc), cudaMemcpyHostToDevice));
    ++generation;
  }
  const Slot& at(int32_t id) const {
    auto it = slot_of.find(id);
    if (it == slot_of.end()) fail(ATMM_ERR_UNKNOWN_ADAPTER, "unknown adapter id " + std::to_string(id));
    return slots[static_cast<size_t>(it->second)];
  }
  // Adapters above kMaxRank: chunk 0 is slot_of[id], chunks 1.. (ranks
  // [128 c, 128 c + 128)) live in these slots, each applied as its own pass.
  std::map<int32_t, std::vector<int>> extra;
  int num_chunks(int32_t id) const {
    auto it = extra.find(id);
    return 1 + (it == extra.end() ? 0 : static_cast<int>(it->second.size()));
  }
  const Slot& chunk(int32_t id, int c) const { return c == 0 ? at(id) : slots[static_cast<size_t>(extra.at(id)[c - 1])]; }
  void require_unchunked(int32_t id, const char* what) const {
    if (num_chunks(id) > 1) {
      fail(ATMM_ERR_CONFIG, std::string(what) + ": adapter " + std::to_string(id) + " has rank " +
                                std::to_string(at(id).total_rank) + " > " + std::to_string(kMaxRank) +
                                " (rank-chunked adapters are served by BypassPlan / merge / delta_w only)");
    }
  }
  int free_index() {
    for (size_t i = 0; i < slots.size(); ++i) {
      if (!slots[i].live) return static_cast<int>(i);
    }
    slots.emplace_back();
    return static_cast<int>(slots.size()) - 1;
  }
  void drop_extra(int32_t id) {
    auto it = extra.find(id);
    if (it == extra.end()) return;
    for (int idx : it->second) {
      free_slot(slots[static_cast<size_t>(idx)]);
      slots[static_cast<size_t>(idx)] = Slot{};
    }
    extra.erase(it);
  }
};

// =========================================================================
// fp32-faithful factor images (precise registries; precise_kernels.cu)
// =========================================================================
namespace atmm {
cudaError_t launch_split3_rows(const float* src, int64_t lds, const int32_t* rows, int64_t m, int64_t k, int64_t kp,
                               uint16_t* dst, int64_t ldd, cudaStream_t s);
cudaError_t launch_split3_cols(const float* src, int64_t lds, int64_t k, int64_t n, int64_t kp, int64_t np,
                               uint16_t* dst, cudaStream_t s);
cudaError_t launch_rows_out(const float* t, int64_t ldt, const int32_t* rows, int64_t m, int64_t n, float* c,
                            int64_t ldc, float alpha, float beta, cudaStream_t s);
cudaError_t launch_tanh(float* x, int64_t ld, int64_t m, int64_t n, cudaStream_t s);

// Image sizes (elements per layer) of a slot of rank r in registry reg.
struct PreciseDims {
  int64_t kpd, r8, n8, db, ub, da;
  PreciseDims(const atmm_registry* reg, int64_t rank)
      : kpd(round_up(reg->d_in, 8)), r8(round_up(rank, 8)), n8(round_up(reg->d_out, 8)),
        db(kSplitParts * kpd * r8), ub(kSplitParts * r8 * n8), da(reg->d_in * kSplitParts * r8) {}
};

// Builds the slot's images from fp32 factors already on the device
// (down [L][d_in x r], up [L][r x d_out]), stream-ordered on st.
static void build_precise_device(atmm_registry* r, Slot& s, const float* down, const float* up, cudaStream_t st,
                                 bool async) {
  const PreciseDims pd(r, s.rank);
  const size_t L = static_cast<size_t>(r->L);
  void** outs[3] = {reinterpret_cast<void**>(&s.p_down_b), reinterpret_cast<void**>(&s.p_up_b),
                    reinterpret_cast<void**>(&s.p_down_a)};
  const int64_t sizes[3] = {pd.db, pd.ub, pd.da};
  for (int i = 0; i < 3; ++i) {
    const size_t bytes = L * static_cast<size_t>(sizes[i]) * 2;
    if (async) {
      CUDA_CHECK(cudaMallocAsync(outs[i], bytes, st));
    } else {
      CUDA_CHECK(cudaMalloc(outs[i], bytes));
    }
  }
  for (int64_t l = 0; l < r->L; ++l) {
    const float* dn = down + l * r->d_in * s.rank;
    const float* u = up + l * s.rank * r->d_out;
    CUDA_CHECK(launch_split3_cols(dn, s.rank, r->d_in, s.rank, pd.kpd, pd.r8, s.p_down_b + l * pd.db, st));
    CUDA_CHECK(launch_split3_cols(u, r->d_out, s.rank, r->d_out, pd.r8, pd.n8, s.p_up_b + l * pd.ub, st));
    CUDA_CHECK(launch_split3_rows(dn, s.rank, nullptr, r->d_in, s.rank, pd.r8, s.p_down_a + l * pd.da,
                                  kSplitParts * pd.r8, st));
  }
}

// fp32-faithful bypass on a plan (defined with the precise entry points below).
namespace {
void bypass_f32(const atmm_plan* p, int64_t layer, const float* x, int64_t ldx, float* y, int64_t ldy, float scale,
                cudaStream_t st);
}  // namespace

// The same from host fp32 factors (synchronous, atmm_registry_put).
static void build_precise_host(atmm_registry* r, Slot& s, const float* down, const float* up) {
  const size_t fd = static_cast<size_t>(r->L * r->d_in * s.rank), fu = static_cast<size_t>(r->L * s.rank * r->d_out);
  DevBuf<float> tmp(fd + fu);
  CUDA_CHECK(cudaMemcpy(tmp.p, down, fd * 4, cudaMemcpyHostToDevice));
  CUDA_CHECK(cudaMemcpy(tmp.p + fd, up, fu * 4, cudaMemcpyHostToDevice));
  build_precise_device(r, s, tmp.p, tmp.p + fd, nullptr, false);
  CUDA_CHECK(cudaDeviceSynchronize());
}
}  // namespace atmm

// =========================================================================
// Plan: routing tables + launch groups
// =========================================================================
namespace atmm {
// Shared-memory / TMEM layout of one atmm_bypass_a2a_kernel launch.
struct A2aLayout {
  bool ok = false;
  int32_t stages = 0, stage_bytes = 0, a_bytes = 0, ypitch = 0, gcols = 1;
  uint32_t off_up = 0, off_y = 0, off_red = 0, off_mid = 0, off_bar = 0, tmem_cols = 0;
  size_t smem = 0;
};

// Split-path (shrink + expand launches) geometry of one launch group.
struct SplitLayout {
  bool ok = false;
  int32_t stages = 0, estages[2] = {0, 0};
  bool ok_dt[2] = {false, false};  // usable for bf16 / fp32 Y
  int32_t g_bf16 = 2;              // bf16 expand item width: 128 g_bf16 columns
  size_t smem_s = 0, smem_e[2] = {0, 0};
  uint32_t tmem_e[2] = {0, 0};     // expand TMEM columns (two accumulators of G x rows16)
  int32_t rows16 = 0;
};

// Stream-path (atmm_stream_kernel) geometry of a plan, per Y dtype:
//   [shrink ring: SS x (X rows8 x 128 B, 128-byte swizzle | down^T r_pad x 128 B)]
//   [expand ring: ES x (up^T 128 x r_pad bf16 | Y rows x 128 x esz)]
//   [mid: 2 x rows16 x r_pad bf16]
// The shrink MMA (M = 128) reads 16 KiB of A from each stage base; the
// rows past a tile feed TMEM lanes that are never read, so >= 16 KiB of the
// allocation must follow the last shrink stage.
struct StreamLayout {
  bool ok = false;
  int32_t grid = 0, sstages[2] = {0, 0}, estages[2] = {0, 0};
  uint32_t s_stage = 0, s_a = 0, e_stage[2] = {0, 0}, off_e[2] = {0, 0}, off_mid[2] = {0, 0};
  uint32_t mid_bytes = 0, tmem_cols = 0;
  int32_t rows_max = 0, r_pad_max = 16, nsl = 0;
  size_t smem[2] = {0, 0};
};

struct LaunchGroup {
  A2aLayout a2a[2];  // per Y dtype (ATMM_BF16, ATMM_F32)
  SplitLayout split;
  int32_t rows_max = 0;
  int32_t path = 0;  // LaunchCfg::path (0 automatic)
  int32_t cluster = 1, bn = 128, stages = 2, ustages = 1, ny = 2;
  int32_t a_bytes = 0, ustage_bytes = 0, ybuf_bytes = 0, rep = 1, nbuf = 2;
  uint32_t off_up = 0, off_y = 0;
  int32_t r_pad_max = 16;
  int64_t tile_offset = 0, num_tiles = 0;
  int32_t stage_bytes = 0, red_rows = 0;
  uint32_t off_red = 0, off_mid = 0, off_bar = 0, tmem_cols = 0;
  size_t smem = 0;
};

// Shared-memory carve-up and TMEM budget of one fused launch:
//   [shrink ring: stages x (A: round_up(rows,8) x 128 B gathered X | B: 64 x r_pad down^T)]
//   [up^T ring: ustages x bn x r_pad][Y ring: ny x round_up(rows,8) x 128 B]
//   [red: C x red_rows x r_pad fp32][mid: 128 x r_pad bf16][mbarriers]
// The M=128 MMA reads 16 KiB of A from each stage base; rows past the tile
// land in later buffers (never consumed), so >= 16 KiB must follow the last
// stage.  Small tiles (<= 64 rows) are sized for two CTAs per SM so every
// cluster of a latency-bound batch is resident in one wave.
static void resolve_group(LaunchGroup& g, int64_t d_in, int64_t d_out, int32_t tile_rows_max,
                          int32_t want_stages) {
  const int64_t nkb = (d_in + kBK - 1) / kBK;
  const int64_t nun = (d_out + kNUnit - 1) / kNUnit;
  g.cluster = static_cast<int32_t>(std::clamp<int64_t>(g.cluster, 1, std::min<int64_t>({nkb, nun, kMaxCluster})));
  const int32_t rp = g.r_pad_max;
  const int64_t rows8 = round_up(std::max<int32_t>(tile_rows_max, 1), 8);
  const bool small = tile_rows_max <= 64;
  g.a_bytes = static_cast<int32_t>(rows8 * 128);
  const int64_t stage = round_up(rows8 * 128 + int64_t(rp) * kBK * 2, 1024);
  g.stage_bytes = static_cast<int32_t>(stage);
  g.rep = tile_rows_max <= 32 ? 4 : (tile_rows_max <= 64 ? 2 : 1);
  // Small tiles: one 64-column chunk per replica, rep (>= 2) chunks in flight.
  int32_t bn = small ? kNUnit : std::clamp(g.bn / kNUnit * kNUnit, kNUnit, 256);
  g.bn = bn;
  g.nbuf = std::max(2, g.rep);
  const int64_t ustage = round_up(int64_t(bn) * rp * 2, 1024);
  g.ustage_bytes = static_cast<int32_t>(ustage);
  g.red_rows = (tile_rows_max + g.cluster - 1) / g.cluster;
  const int64_t red = g.cluster > 1 ? round_up(int64_t(g.cluster) * g.red_rows * rp * 4, 1024) : 0;
  const int64_t mid = round_up(int64_t(kTileM) * rp * 2, 1024);
  int32_t cols = 32;
  while (cols < std::max<int32_t>(rp, g.nbuf * bn)) cols <<= 1;
  g.tmem_cols = static_cast<uint32_t>(cols);
  const int64_t ybuf = rows8 * 128;
  g.ybuf_bytes = static_cast<int32_t>(ybuf);
  const int64_t slice_cols = (nun + g.cluster - 1) / g.cluster * kNUnit;
  const int kb_per_cta = static_cast<int>((nkb + g.cluster - 1) / g.cluster);
  const int chunks = static_cast<int>((slice_cols + bn - 1) / bn);
  const int ny_all = static_cast<int>(std::min<int64_t>(32, (slice_cols + 31) / 32));  // fp32 sizing
  auto total = [&](int s, int u, int ny) {
    const int64_t bar = round_up((2 * s + 2 * u + 2 * ny + 2 * g.nbuf + 3) * 8 + 8, 16);
    const int64_t after_ring = int64_t(u) * ustage + int64_t(ny) * ybuf + red + mid + bar;
    const int64_t guard = std::max<int64_t>(0, (kTileM * 128) - (stage - 0) - after_ring);
    return size_t(1024 + int64_t(s) * stage + after_ring + guard);
  };
  // Search (stages, up stages, Y buffers) under the shared-memory limit.
  // Targets: small tiles keep every K block, up^T chunk and Y sub-chunk of
  // the CTA in flight; large tiles want ~3 shrink stages (~70 KiB in flight
  // per SM covers HBM latency), 2 up^T stages and >= 4 Y buffers.
  const int s_cap = small ? std::min(kb_per_cta, 8) : std::min(kb_per_cta, 3);
  const int u_cap = small ? std::min(chunks, 16) : std::min(chunks, 2);
  const int ny_cap = small ? ny_all : std::min(ny_all, 4);
  auto search = [&](size_t limit, int& s_out, int& u_out, int& ny_out) {
    const int s_hi = want_stages > 0 ? want_stages : std::min(kb_per_cta, small ? 8 : kMaxStages);
    long best = -1;
    for (int s = std::max(2, std::min(s_hi, kb_per_cta)); s >= 2; --s) {
      for (int u = std::min(16, chunks); u >= 1; --u) {
        for (int ny = ny_all; ny >= std::min(2, ny_all); --ny) {
          if (total(s, u, ny) > limit) continue;
          // lexicographic on capped depths, then on raw depths
          const long score = (long)std::min(s, s_cap) * 1000000 + (long)std::min(u, u_cap) * 10000 +
                             (long)std::min(ny, ny_cap) * 100 + s + u + ny;
          if (score > best) {
            best = score;
            s_out = s;
            u_out = u;
            ny_out = ny;
          }
          break;  // larger ny first: the first fit is the best for (s, u)
        }
      }
    }
    return best >= 0;
  };
  int s = 0, u = 0, ny = 0;
  bool ok = false;
  if (small && cols <= 256) ok = search(kSmemPerSM / 2 - 2048, s, u, ny);
  if (!ok) ok = search(kSmemLimit, s, u, ny);
  if (!ok) fail(ATMM_ERR_CONFIG, "fused bypass does not fit in shared memory (rank too large)");
  g.stages = s;
  g.ustages = u;
  g.ny = ny;
  g.off_up = static_cast<uint32_t>(int64_t(s) * stage);
  g.off_y = static_cast<uint32_t>(g.off_up + int64_t(u) * ustage);
  g.off_red = static_cast<uint32_t>(g.off_y + int64_t(ny) * ybuf);
  g.off_mid = static_cast<uint32_t>(g.off_red + red);
  g.off_bar = static_cast<uint32_t>(g.off_mid + mid);
  g.smem = total(s, u, ny);
  // CTAs of one cluster can share an SM; their TMEM allocations must all fit
  // (512 columns per SM) or the cluster could deadlock.  Pad shared memory
  // so co-residency never exceeds 512 / cols CTAs per SM.
  const int max_co = std::max(1, 512 / cols);
  while (static_cast<int>(kSmemPerSM / (g.smem + 1024)) > max_co) g.smem += 4096;
}
}  // namespace atmm

// All-to-all variant eligibility and layout (kernels.cu atmm_bypass_a2a_kernel):
//   [ring: S x (rows8 x 128 B X | 64 x r_pad down^T)][up^T slice][Y slice: rows x slice x esz]
//   [red: C x rows x r_pad fp32][mid: rows16 x r_pad bf16][mbarriers]
// The shrink (M = 128) over-reads 16 KiB from each stage base and the expand
// (M = 128) 128 up^T rows from each group base; both land inside the
// allocation (guard) and feed TMEM lanes that are never read.
static A2aLayout resolve_a2a(int64_t d_in, int64_t d_out, int32_t cluster, int32_t rows_max, int32_t r_pad,
                             int64_t esz) {
  A2aLayout l;
  if (rows_max > kTileM || d_out % 8 != 0) return l;
  const int64_t nkb = (d_in + kBK - 1) / kBK;
  const int64_t nun = (d_out + kNUnit - 1) / kNUnit;
  const int64_t slice = (nun + cluster - 1) / cluster * kNUnit;
  const int64_t kb_per_cta = (nkb + cluster - 1) / cluster;
  const int64_t rows8 = round_up(std::max<int32_t>(rows_max, 1), 8);
  const int64_t rows16 = round_up(std::max<int32_t>(rows_max, 1), 16);
  // G expand MMAs of 128 output columns; epilogue threads own G adjacent columns.
  int32_t G = 1;
  while (int64_t(G) * kTileM < slice) G <<= 1;
  if (G > 8) return l;
  int32_t cols = 32;
  while (cols < std::max<int64_t>({int64_t(r_pad), int64_t(G) * rows16})) cols <<= 1;
  if (cols > 512) return l;
  l.gcols = G;
  l.a_bytes = static_cast<int32_t>(rows8 * 128);
  const int64_t stage = round_up(rows8 * 128 + int64_t(r_pad) * kBK * 2, 1024);
  l.stage_bytes = static_cast<int32_t>(stage);
  l.ypitch = static_cast<int32_t>(round_up(slice * esz, 16));
  const int64_t up = round_up(int64_t(G) * kTileM * r_pad * 2, 1024);
  const int64_t ybuf = round_up(int64_t(rows_max) * l.ypitch, 1024);
  const int64_t red = round_up(int64_t(cluster) * rows_max * r_pad * 4, 1024);
  // mid (rows16 x r_pad bf16) aliases ring stage 0 (dead once the shrink is done)
  if (rows16 * r_pad * 2 > stage) return l;
  auto total = [&](int64_t S) {
    const int64_t bar = round_up((2 * S + 6) * 8 + 8, 16);
    const int64_t body = S * stage + up + ybuf + red + bar;
    const int64_t guard_a = (S - 1) * stage + kTileM * 128;  // shrink A over-read (M = 128)
    return size_t(1024 + std::max(body, guard_a));
  };
  // Prefer a layout that fits two CTAs per SM (the next launch's prologue
  // overlaps this one under programmatic dependent launch), then depth.
  int64_t s_first = std::min<int64_t>(kb_per_cta, 8);
  if (cols <= 256) {
    for (int64_t S = s_first; S >= std::min<int64_t>(4, kb_per_cta); --S) {
      if (total(S) <= kSmemPerSM / 2 - 1024) {
        s_first = S;
        break;
      }
    }
  }
  for (int64_t S = s_first; S >= std::min<int64_t>(2, kb_per_cta); --S) {
    if (total(S) > kSmemLimit) continue;
    l.stages = static_cast<int32_t>(S);
    l.off_up = static_cast<uint32_t>(S * stage);
    l.off_y = static_cast<uint32_t>(l.off_up + up);
    l.off_red = static_cast<uint32_t>(l.off_y + ybuf);
    l.off_mid = 0;
    l.off_bar = static_cast<uint32_t>(l.off_red + red);
    l.tmem_cols = static_cast<uint32_t>(cols);
    l.smem = total(S);
    const int max_co = std::max(1, 512 / cols);
    while (static_cast<int>(kSmemPerSM / (l.smem + 1024)) > max_co) l.smem += 4096;
    l.ok = true;
    return l;
  }
  return l;
}

// Split path scratch written by the shrink and read by the expand: mid
// partials (fp32, per tile x K slice), bf16 mid per tile and per-tile mid
// readiness counters.  One set per CUDA stream that applies the plan, so
// applies of one plan on different streams never share scratch (the last
// CTA of each expand resets the counters for the next expand on its stream).
struct SplitScratch {
  DevBuf<float> part;
  DevBuf<uint16_t> mid;
  DevBuf<int32_t> counter;
};

// Split path of one plan: the read-only balancing tables (shared by every
// stream) and the per-stream scratch sets, created on a stream's first apply.
struct SplitBufs {
  DevBuf<int32_t> tables;  // [s_begin | e_begin bf16 | e_begin fp32 (P+1 each) | seg_slot0 (P) | nseg | part_off (T) | red_off (T+1) | red_tile0 (P)]
  int32_t grid = 0;
  size_t part_elems = 0, mid_elems = 0, counter_elems = 0;
  std::mutex mu;
  // per stream: two scratch sets (the split path alternates them so that a
  // shrink may run under the previous apply's expand, SplitParams::early);
  // the stream path uses set 0 only
  struct StreamSets {
    cudaStream_t stream = nullptr;
    std::unique_ptr<SplitScratch> set[2];
    int next = 0;
  };
  std::vector<std::unique_ptr<StreamSets>> scratch;
  static constexpr size_t kMaxStreams = 32;

  // Scratch set `k` of `stream`.  A new set is allocated and zeroed outside
  // the caller's stream (relaxed capture mode for this thread, a private
  // non-blocking stream for the zero fill), so the first apply on a stream
  // may happen inside a CUDA graph capture.
  SplitScratch& for_stream(cudaStream_t stream) {
    std::lock_guard<std::mutex> lk(mu);
    return set_of(sets_of(stream), 0);
  }
  // The split path: the set after the one this stream used last.
  SplitScratch& alternate(cudaStream_t stream) {
    std::lock_guard<std::mutex> lk(mu);
    StreamSets& ss = sets_of(stream);
    const int k = ss.next;
    ss.next ^= 1;
    return set_of(ss, k);
  }

 private:
  StreamSets& sets_of(cudaStream_t stream) {
    for (auto& ss : scratch) {
      if (ss->stream == stream) return *ss;
    }
    if (scratch.size() >= kMaxStreams) {
      fail(ATMM_ERR_CONFIG, "split-path plan applied on more than 32 distinct streams");
    }
    scratch.push_back(std::make_unique<StreamSets>());
    scratch.back()->stream = stream;
    return *scratch.back();
  }
  SplitScratch& set_of(StreamSets& ss, int k) {
    if (ss.set[k]) return *ss.set[k];
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    cudaThreadExchangeStreamCaptureMode(&mode);
    auto sc = std::make_unique<SplitScratch>();
    cudaError_t err = cudaSuccess;
    cudaStream_t init = nullptr;
    try {
      sc->part.alloc(part_elems);
      sc->mid.alloc(mid_elems);
      sc->counter.alloc(counter_elems);
      err = cudaStreamCreateWithFlags(&init, cudaStreamNonBlocking);
      if (err == cudaSuccess) err = cudaMemsetAsync(sc->mid.p, 0, mid_elems * sizeof(uint16_t), init);
      if (err == cudaSuccess) err = cudaMemsetAsync(sc->counter.p, 0, counter_elems * sizeof(int32_t), init);
      if (err == cudaSuccess) err = cudaStreamSynchronize(init);
    } catch (...) {
      if (init) cudaStreamDestroy(init);
      cudaThreadExchangeStreamCaptureMode(&mode);
      throw;
    }
    if (init) cudaStreamDestroy(init);
    cudaThreadExchangeStreamCaptureMode(&mode);
    if (err != cudaSuccess) fail(ATMM_ERR_CUDA, std::string("split scratch init failed: ") + cudaGetErrorString(err));
    ss.set[k] = std::move(sc);
    return *ss.set[k];
  }
};

struct atmm_plan {
  atmm_registry* reg = nullptr;
  uint64_t generation = 0;
  int64_t n = 0;         // rows of X / Y
  int64_t n_assign = 0;  // routed rows (== n unless the plan maps rows)
  BatchPlan bp;
  std::vector<LaunchGroup> groups;
  // groups[merged_first ..] all take the split path for bf16 Y: one launch
  // pair over their contiguous tile range (merged.tile_offset, num_tiles).
  int merged_first = -1;
  LaunchGroup merged;
  std::unique_ptr<SplitBufs> merged_bufs;
  // Stream path (atmm_stream_kernel): every tile of the plan in one launch.
  StreamLayout stream;
  int32_t stream_mode = 0;  // 0 never, 1 forced (every segment's launch path is ATMM_PATH_STREAM), 2 automatic
  std::unique_ptr<SplitBufs> stream_bufs;  // tables: [s_begin | e_begin (P+1 each) | seg_slot0 (P) | nseg | part_off | ncons (T)]
  DevBuf<int32_t> d_rows;
  DevBuf<int32_t> d_tile_rows;  // [tile][kTileM] padded row lists (a2a prologue)
  std::vector<int32_t> rows_host;  // routed entry (plan order) -> X / Y row
  bool any_contig = false;         // some tile's rows are consecutive (TileDesc::x_row0)
  DevBuf<TileDesc> d_tiles;
  int64_t total_ctas = 0;
  uint64_t flops = 0;  // algorithmic FLOPs of one apply (flops.hpp accounting)
  uint32_t flags = 0;  // ATMM_PLAN_*
  // Adapters above kMaxRank: pass c (>= 1) applies rank chunk c of every
  // routed row whose adapter has one, as a row-mapped plan over the same X / Y
  // (separate launches: the passes update the same Y rows).
  std::vector<std::unique_ptr<atmm_plan>> passes;
};

namespace atmm {
// Which kernel a launch group runs: the fused all-to-all kernel for small
// (latency-bound) tiles, the split shrink + expand pair for large ones, the
// general fused kernel otherwise.  A launch's `path` (tiling table entry or
// atmm_plan_create_launch) forces one where it is applicable.
enum class BypassPath { kA2a, kSplit, kFused };
static BypassPath choose_path(const LaunchGroup& g, int y_dtype, bool y_vec) {
  const int di = y_dtype == ATMM_BF16 ? 0 : 1;
  const bool a2a = g.a2a[di].ok && y_vec;
  const bool split = g.split.ok_dt[di] && y_vec;
  if (g.path == ATMM_PATH_A2A && a2a) return BypassPath::kA2a;
  if (g.path == ATMM_PATH_SPLIT && split) return BypassPath::kSplit;
  if (g.path == ATMM_PATH_FUSED) return BypassPath::kFused;
  if (a2a && g.rows_max <= 32) return BypassPath::kA2a;
  if (split) return BypassPath::kSplit;  // taken through the plan's merged split range
  if (a2a) return BypassPath::kA2a;
  return BypassPath::kFused;
}

// Expand item width for bf16 Y: 128 G columns, G = 2 adjacent columns per
// epilogue thread (measured: 128-column items 48 vs 36 us at cfg3).
static int expand_g_bf16() { return 2; }

// Split expand output: staged in shared memory and stored by 16-byte
// accesses, or stored straight from the epilogue registers (G x element
// bytes per thread and row).  Measured (tools/path_bench.py, B200): staged
// wins for G = 1 items (bf16: 2-byte direct stores, rank-128 Input2 94.8 ->
// 81.3 us; fp32 cfg3 46.4 -> 43.8, cfg5 118.3 -> 113.5 us) and loses for
// bf16 G = 2, whose direct 4-byte stores already fill a line per warp row
// (cfg3 37.7 vs 40.6, cfg5 89.4 vs 96.7 us: the per-item barrier and the
// extra shared-memory pass).
static int split_out_staged(int g) { return g == 1 ? 1 : 0; }

// Fixed per-item costs (bytes-equivalent: barriers, 4 MMAs) of the split
// kernels' work balancing.
static int64_t shrink_fixed_cost() { return 32768; }
static int64_t expand_fixed_cost() { return 32768; }

static SplitLayout resolve_split(int64_t d_in, int64_t d_out, int32_t rows_max, int32_t r_pad) {
  SplitLayout l;
  (void)d_in;
  if (d_out % 8 != 0 || r_pad > 128 || rows_max > kTileM) return l;
  const int64_t avail = int64_t(kSmemLimit) - 1024 - 512;  // alignment slack + the kernels' static smem
  const int64_t stage = int64_t(kTileM) * 128 + int64_t(r_pad) * kBK * 2;
  l.stages = static_cast<int32_t>(std::min<int64_t>(8, avail / stage));
  l.smem_s = size_t(1024 + l.stages * stage);
  const int64_t rows16 = round_up(rows_max, 16);
  l.rows16 = static_cast<int32_t>(rows16);
  for (int di = 0; di < 2; ++di) {
    const int64_t esz = di == 0 ? 2 : 4;
    // bf16 items are 256 columns wide unless two of them do not fit (large
    // rank x rows): then 128 columns
    for (int g : di == 0 ? std::vector<int>{expand_g_bf16(), 1} : std::vector<int>{1}) {
      const int64_t cols = int64_t(kTileM) * g;  // expand item width (128 G columns)
      const int64_t est = round_up(cols * r_pad * 2 + round_up(rows16 * r_pad * 2, 128) + int64_t(rows_max) * cols * esz + kTileM * 4, 128);
      l.estages[di] = static_cast<int32_t>(std::min<int64_t>(4, (avail + 1024 - 128) / est));  // 128-byte aligned kernel
      l.smem_e[di] = size_t(128 + l.estages[di] * est);
      if (di == 0) l.g_bf16 = g;
      if (l.estages[di] >= 2) break;
    }
    // TMEM: the expand holds two accumulators of G x rows16 columns from its
    // start (before its reduction share, which other CTAs' items wait for):
    // pad shared memory so co-resident expand CTAs always fit in 512 columns.
    {
      const int64_t g = di == 0 ? l.g_bf16 : 1;
      int64_t cols = 32;
      while (cols < 2 * g * rows16) cols <<= 1;
      const int64_t max_co = std::max<int64_t>(1, 512 / cols);
      while (int64_t(kSmemPerSM) / int64_t(l.smem_e[di] + 1024) > max_co) l.smem_e[di] += 4096;
      l.tmem_e[di] = static_cast<uint32_t>(cols);
    }
    l.ok_dt[di] = l.stages >= 2 && l.estages[di] >= 2;
  }
  l.ok = l.ok_dt[0] || l.ok_dt[1];
  return l;
}

// Stream-path ring depths: each ring gets stages until shared memory runs
// out, always extending the ring with fewer bytes in flight (both rings
// stream from HBM at once; ~64 KiB+ in flight per SM covers the latency),
// capped by the units a CTA actually owns.
static void resolve_stream(StreamLayout& l, int32_t rows_max, int32_t r_pad, int s_units_cta, int e_units_cta) {
  l.ok = false;
  if (r_pad > kMaxRank || rows_max > kTileM || rows_max < 1) return;
  l.rows_max = rows_max;
  l.r_pad_max = r_pad;
  const int64_t rows8 = round_up(rows_max, 8), rows16 = round_up(rows_max, 16);
  l.s_a = static_cast<uint32_t>(rows8 * 128);
  l.s_stage = static_cast<uint32_t>(rows8 * 128 + int64_t(r_pad) * 128);
  l.mid_bytes = static_cast<uint32_t>(round_up(rows16 * r_pad * 2, 1024));
  uint32_t cols = 32;
  while (cols < static_cast<uint32_t>(2 * r_pad + 2 * rows16)) cols <<= 1;
  if (cols > 512) return;
  l.tmem_cols = cols;
  const int s_cap = std::clamp(s_units_cta, 1, 16), e_cap = std::clamp(e_units_cta, 1, 16);
  for (int di = 0; di < 2; ++di) {
    const int64_t esz = di == 0 ? 2 : 4;
    const int64_t es = round_up(int64_t(128) * r_pad * 2 + int64_t(rows_max) * 128 * esz, 1024);
    l.e_stage[di] = static_cast<uint32_t>(es);
    const int64_t avail = int64_t(kSmemLimit) - 2048 - 2 * int64_t(l.mid_bytes);
    auto fits = [&](int ss, int e) {
      const int64_t body = int64_t(ss) * l.s_stage + int64_t(e) * es;
      return std::max(body, int64_t(ss - 1) * l.s_stage + 16384) <= avail;
    };
    int ss = 1, e = 1;
    if (!fits(ss, e)) return;
    while (true) {
      const bool can_s = ss < s_cap && fits(ss + 1, e);
      const bool can_e = e < e_cap && fits(ss, e + 1);
      if (!can_s && !can_e) break;
      if (can_s && (!can_e || int64_t(ss) * l.s_stage <= int64_t(e) * es)) ++ss;
      else ++e;
    }
    l.sstages[di] = ss;
    l.estages[di] = e;
    l.off_e[di] = static_cast<uint32_t>(int64_t(ss) * l.s_stage);
    l.off_mid[di] = static_cast<uint32_t>(l.off_e[di] + int64_t(e) * es);
    const int64_t body = int64_t(l.off_mid[di]) + 2 * int64_t(l.mid_bytes);
    l.smem[di] = size_t(1024 + std::max(body, int64_t(ss - 1) * l.s_stage + 16384));
  }
  l.ok = true;
}

// Balanced split of a flattened, weighted work list over `parts` CTAs:
// begin[b] = first item whose cost prefix reaches b * total / parts.
static std::vector<int32_t> balance(const std::vector<int64_t>& cost, int parts) {
  std::vector<int32_t> begin(static_cast<size_t>(parts) + 1, static_cast<int32_t>(cost.size()));
  int64_t total = 0;
  for (int64_t c : cost) total += c;
  int64_t acc = 0;
  int b = 0;
  for (size_t i = 0; i < cost.size() && b < parts; ++i) {
    while (b < parts && acc >= (total * b + parts - 1) / parts) begin[static_cast<size_t>(b++)] = static_cast<int32_t>(i);
    acc += cost[i];
  }
  begin[0] = 0;
  return begin;
}

}  // namespace atmm

namespace atmm {

// Fixed per-unit cost (bytes-equivalent) of the stream kernel's balancing.
static int64_t stream_fixed_cost() { return 4096; }

// Stream path of a plan: every tile in one launch.  Balanced shrink and
// expand ranges over the SMs, the per-tile segment slots of the shrink
// partials (CTA order = fixed reduction order) and consumer counts.
static void build_stream(atmm_plan& plan, const std::vector<TileDesc>& tiles, const atmm_registry* reg) {
  StreamLayout& l = plan.stream;
  l.ok = false;
  const int T = static_cast<int>(tiles.size());
  if (T == 0 || reg->d_out % 8 != 0) return;
  int32_t rows_max = 1, rpm = 16;
  for (const TileDesc& td : tiles) {
    rows_max = std::max(rows_max, td.rows);
    rpm = std::max(rpm, td.r_pad);
  }
  const int nkb = static_cast<int>((reg->d_in + kBK - 1) / kBK);
  const int nsl = static_cast<int>((reg->d_out + 127) / 128);
  std::vector<int64_t> scost, ecost;
  scost.reserve(size_t(T) * nkb);
  ecost.reserve(size_t(T) * nsl);
  for (const TileDesc& td : tiles) {
    for (int k = 0; k < nkb; ++k) scost.push_back(int64_t(td.rows) * 128 + int64_t(td.r_pad) * 128 + stream_fixed_cost());
    for (int k = 0; k < nsl; ++k) ecost.push_back(int64_t(td.rows) * 128 * 2 * 2 + 128 * int64_t(td.r_pad) * 2 + stream_fixed_cost());
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, reg->device);
  const int P = std::max(1, std::min<int>(sms, static_cast<int>(std::max(scost.size(), ecost.size()))));
  std::vector<int32_t> sb = balance(scost, P), eb = balance(ecost, P);
  int s_max = 1, e_max = 1;
  for (int b = 0; b < P; ++b) {
    s_max = std::max(s_max, sb[b + 1] - sb[b]);
    e_max = std::max(e_max, eb[b + 1] - eb[b]);
  }
  resolve_stream(l, rows_max, rpm, s_max, e_max);
  if (!l.ok) return;
  l.grid = P;
  l.nsl = nsl;
  std::vector<int32_t> slot0(static_cast<size_t>(P), 0), nseg(T, 0), off(T), ncons(T, 0);
  for (int b = 0; b < P; ++b) {
    if (sb[b] < sb[b + 1]) {
      const int t0 = sb[b] / nkb, t1 = (sb[b + 1] - 1) / nkb;
      slot0[static_cast<size_t>(b)] = nseg[t0];
      for (int t = t0; t <= t1; ++t) ++nseg[t];
    }
    if (eb[b] < eb[b + 1]) {
      const int t0 = eb[b] / nsl, t1 = (eb[b + 1] - 1) / nsl;
      for (int t = t0; t <= t1; ++t) ++ncons[t];
    }
  }
  int32_t total_seg = 0;
  for (int t = 0; t < T; ++t) {
    off[t] = total_seg;
    total_seg += nseg[t];
  }
  std::vector<int32_t> tables;
  tables.insert(tables.end(), sb.begin(), sb.end());
  tables.insert(tables.end(), eb.begin(), eb.end());
  tables.insert(tables.end(), slot0.begin(), slot0.end());
  tables.insert(tables.end(), nseg.begin(), nseg.end());
  tables.insert(tables.end(), off.begin(), off.end());
  tables.insert(tables.end(), ncons.begin(), ncons.end());
  auto& mb = plan.stream_bufs;
  mb = std::make_unique<SplitBufs>();
  mb->grid = P;
  mb->part_elems = static_cast<size_t>(total_seg) * kTileM * rpm;
  mb->mid_elems = 0;
  mb->counter_elems = 2 * static_cast<size_t>(T);
  mb->tables.alloc(tables.size());
  CUDA_CHECK(cudaMemcpy(mb->tables.p, tables.data(), tables.size() * 4, cudaMemcpyHostToDevice));
}

// Builds routing tables and launch groups.  `forced` (tuner) overrides the
// table for every segment.
// The MMA-ordered up^T copy for G (Slot::up_tg) of the live slot whose up^T
// is `up_t`, made on first use: a permute kernel on a private stream,
// allocated stream-ordered, outside any capture on this thread (relaxed
// mode), waited for before the plan that needs it exists.  G = 1 is the
// registry layout itself.  Null when no slot matches.
static const uint16_t* slot_up_tg(atmm_registry* reg, const uint16_t* up_t, int32_t r_pad, int G) {
  if (G == 1) return up_t;
  const int gi = G == 2 ? 0 : (G == 4 ? 1 : (G == 8 ? 2 : -1));
  if (gi < 0) return nullptr;
  std::lock_guard<std::mutex> lk(reg->up2_mu);
  Slot* sl = nullptr;
  for (Slot& s : reg->slots) {
    if (s.live && s.up_t == up_t && s.r_pad == r_pad) sl = &s;
  }
  // put_async slots: their factors are written stream-ordered on the
  // caller's stream (not necessarily done when a plan is built): no copy,
  // the kernels stage their up^T by 16-byte copies
  if (!sl || sl->async_owned) return nullptr;
  if (sl->up_tg[gi]) return sl->up_tg[gi];
  const int64_t d_out_pad2 = round_up(reg->d_out_pad, 128 * G);
  const size_t elems = static_cast<size_t>(reg->L) * static_cast<size_t>(d_out_pad2) * static_cast<size_t>(r_pad);
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  cudaThreadExchangeStreamCaptureMode(&mode);
  cudaStream_t st = nullptr;
  uint16_t* dst = nullptr;
  cudaError_t err = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (err == cudaSuccess) err = cudaMallocAsync(&dst, elems * 2, st);
  if (err == cudaSuccess) {
    err = launch_permute_up_g2(sl->up_t, reg->d_out_pad * r_pad, dst, d_out_pad2 * r_pad, reg->L, reg->d_out_pad,
                               d_out_pad2, r_pad, G, st);
  }
  if (err == cudaSuccess) err = cudaStreamSynchronize(st);
  if (err != cudaSuccess && dst) {
    cudaFreeAsync(dst, st);
    cudaStreamSynchronize(st);
    dst = nullptr;
  }
  if (st) cudaStreamDestroy(st);
  cudaThreadExchangeStreamCaptureMode(&mode);
  if (err != cudaSuccess) fail(ATMM_ERR_CUDA, std::string("up^T permute failed: ") + cudaGetErrorString(err));
  sl->up_tg[gi] = dst;
  return dst;
}

static std::unique_ptr<atmm_plan> build_plan(atmm_registry* reg, const int32_t* assignment,
                                             int64_t n, const TilingTable* table,
                                             const LaunchCfg* forced, const int32_t* row_map = nullptr,
                                             int64_t n_rows = -1, int chunk = 0) {
  auto plan = std::make_unique<atmm_plan>();
  plan->reg = reg;
  plan->generation = reg->generation;
  plan->n = row_map ? n_rows : n;
  plan->n_assign = n;
  plan->bp = plan_batch(assignment, n);
  if (n > std::numeric_limits<int32_t>::max()) fail(ATMM_ERR_SHAPE, "batch too large");
  struct Pending {
    LaunchCfg cfg;
    std::vector<TileDesc> tiles;
    int32_t r_pad_max = 16;
    int32_t rows_max = 1;
  };
  std::map<std::tuple<int32_t, int32_t, int32_t, int32_t>, Pending> by_launch;
  const size_t S = plan->bp.seg_adapter.size();
  for (size_t s = 0; s < S; ++s) {
    const int32_t id = plan->bp.seg_adapter[s];
    auto it = reg->slot_of.find(id);
    if (it == reg->slot_of.end()) fail(ATMM_ERR_UNKNOWN_ADAPTER, "unknown adapter id " + std::to_string(id));
    const Slot& sl = reg->chunk(id, chunk);
    const int64_t b = plan->bp.seg_offsets[s], e = plan->bp.seg_offsets[s + 1];
    const int64_t ns = e - b;
    plan->flops += 2ull * static_cast<uint64_t>(ns) * static_cast<uint64_t>(sl.alg_rank) *
                   static_cast<uint64_t>(reg->d_in + reg->d_out);
    LaunchCfg lc = forced ? *forced
                          : (table ? table->resolve_launch(ns, reg->d_in, sl.rank, reg->d_out)
                                   : heuristic_launch(ns, reg->d_in, sl.rank, reg->d_out));
    const int64_t tm = std::clamp<int64_t>(lc.tile_m, 1, kTileM);
    const int64_t ntiles = (ns + tm - 1) / tm;
    const int64_t per = (ns + ntiles - 1) / ntiles;  // balanced tiles
    const auto lkey = std::make_tuple(lc.cluster, lc.bn, lc.stages, lc.path);
    auto& pend = by_launch[lkey];
    pend.cfg = lc;
    pend.r_pad_max = std::max<int32_t>(pend.r_pad_max, static_cast<int32_t>(sl.r_pad));
    for (int64_t t = 0; t < ntiles; ++t) {
      const int64_t tb = b + t * per;
      const int64_t te = std::min(e, tb + per);
      if (te <= tb) break;
      TileDesc td{sl.down_t, sl.up_t, reg->d_in_pad * sl.r_pad, reg->d_out_pad * sl.r_pad,
                  static_cast<int32_t>(tb), static_cast<int32_t>(te - tb), static_cast<int32_t>(sl.r_pad),
                  sl.scale};
      pend.rows_max = std::max<int32_t>(pend.rows_max, td.rows);
      pend.tiles.push_back(td);
    }
  }
  std::vector<TileDesc> all_tiles;
  // Groups that run the split path (bf16 Y) go last, so their tiles form one
  // contiguous range launched as a single shrink + expand pair.
  std::vector<std::pair<LaunchGroup, std::vector<TileDesc>>> built;
  for (auto& [key, pend] : by_launch) {
    LaunchGroup g;
    g.cluster = pend.cfg.cluster;
    g.bn = pend.cfg.bn;
    g.path = pend.cfg.path;
    g.r_pad_max = pend.r_pad_max;
    resolve_group(g, reg->d_in, reg->d_out, pend.rows_max, pend.cfg.stages);
    g.a2a[0] = resolve_a2a(reg->d_in, reg->d_out, g.cluster, pend.rows_max, pend.r_pad_max, 2);
    g.a2a[1] = resolve_a2a(reg->d_in, reg->d_out, g.cluster, pend.rows_max, pend.r_pad_max, 4);
    g.split = resolve_split(reg->d_in, reg->d_out, pend.rows_max, pend.r_pad_max);
    g.rows_max = pend.rows_max;
    g.num_tiles = static_cast<int64_t>(pend.tiles.size());
    built.emplace_back(g, std::move(pend.tiles));
  }
  std::stable_partition(built.begin(), built.end(), [](const auto& b) {
    return choose_path(b.first, ATMM_BF16, true) != BypassPath::kSplit;
  });
  for (auto& [g, tiles] : built) {
    g.tile_offset = static_cast<int64_t>(all_tiles.size());
    all_tiles.insert(all_tiles.end(), tiles.begin(), tiles.end());
    plan->total_ctas += g.num_tiles * g.cluster;
    if (choose_path(g, ATMM_BF16, true) == BypassPath::kSplit) {
      if (plan->merged_first < 0) {
        plan->merged_first = static_cast<int>(plan->groups.size());
        plan->merged.tile_offset = g.tile_offset;
      }
      plan->merged.num_tiles += g.num_tiles;
      plan->merged.r_pad_max = std::max(plan->merged.r_pad_max, g.r_pad_max);
      plan->merged.rows_max = std::max(plan->merged.rows_max, g.rows_max);
    }
    plan->groups.push_back(g);
  }
  {
    bool all_stream = true, all_auto = true;
    for (const LaunchGroup& g : plan->groups) {
      all_stream = all_stream && g.path == ATMM_PATH_STREAM;
      all_auto = all_auto && g.path == ATMM_PATH_AUTO;
    }
    plan->stream_mode = all_stream ? 1 : (all_auto ? 2 : 0);
  }
  if (plan->merged_first >= 0) {
    plan->merged.split = resolve_split(reg->d_in, reg->d_out, plan->merged.rows_max, plan->merged.r_pad_max);
    // 256-column expand items (bf16 Y, G = 2) load up^T by one bulk copy
    // from the slot's MMA-ordered copy
    if (plan->merged.split.ok_dt[0] && plan->merged.split.g_bf16 == 2) {
      for (int64_t t = plan->merged.tile_offset; t < plan->merged.tile_offset + plan->merged.num_tiles; ++t) {
        TileDesc& td = all_tiles[static_cast<size_t>(t)];
        td.up_t2 = slot_up_tg(reg, td.up_t, td.r_pad, 2);
        td.up_g = td.up_t2 ? 2 : 0;
      }
    }
    if (!plan->merged.split.ok) plan->merged_first = -1;
  }
  std::vector<int32_t> rows32(plan->bp.row_index.begin(), plan->bp.row_index.end());
  if (row_map) {
    // routed entry i lives in X / Y row row_map[i] (mixture guest rows)
    std::vector<char> seen(static_cast<size_t>(n_rows), 0);
    for (int64_t i = 0; i < n; ++i) {
      if (row_map[i] < 0 || row_map[i] >= n_rows || seen[static_cast<size_t>(row_map[i])]) {
        fail(ATMM_ERR_SHAPE, "row map entries must be distinct rows in [0, n_rows)");
      }
      seen[static_cast<size_t>(row_map[i])] = 1;
    }
    for (auto& v : rows32) v = row_map[v];
  }
  DeviceGuard dg(reg->device);
  if (plan->merged_first >= 0) {
    // Persistent split kernels: balanced work ranges over the SMs.
    const LaunchGroup& g = plan->merged;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, reg->device);
    const int T = static_cast<int>(g.num_tiles);
    const int nkb = static_cast<int>((reg->d_in + kBK - 1) / kBK);
    std::vector<int64_t> scost, ecost[2];
    for (int t = 0; t < T; ++t) {
      const TileDesc& td = all_tiles[static_cast<size_t>(g.tile_offset + t)];
      // bytes moved + a fixed per-item cost (pipeline step: barriers, 4 MMAs)
      for (int k = 0; k < nkb; ++k) scost.push_back(int64_t(td.rows) * 128 + int64_t(td.r_pad) * 128 + shrink_fixed_cost());
      for (int di = 0; di < 2; ++di) {
        const int64_t cols = int64_t(kTileM) * (di == 0 ? g.split.g_bf16 : 1), esz = di == 0 ? 2 : 4;
        const int nsl = static_cast<int>((reg->d_out + cols - 1) / cols);
        for (int k = 0; k < nsl; ++k) ecost[di].push_back(int64_t(td.rows) * cols * esz * 2 + cols * td.r_pad * 2 + expand_fixed_cost());
      }
    }
    const int P = std::max(1, std::min<int>(sms, static_cast<int>(scost.size())));
    std::vector<int32_t> sb = balance(scost, P), eb0 = balance(ecost[0], P), eb1 = balance(ecost[1], P);
    // Segments: the run of one tile inside one non-empty CTA range; slots are
    // numbered per tile in CTA order (fixed reduction order).
    std::vector<int32_t> slot0(static_cast<size_t>(P), 0), nseg(T, 0), off(T);
    for (int b = 0; b < P; ++b) {
      if (sb[b] >= sb[b + 1]) continue;
      const int t0 = sb[b] / nkb, t1 = (sb[b + 1] - 1) / nkb;
      slot0[static_cast<size_t>(b)] = nseg[t0];
      for (int t = t0; t <= t1; ++t) ++nseg[t];
    }
    int32_t total_seg = 0;
    for (int t = 0; t < T; ++t) {
      off[t] = total_seg;
      total_seg += nseg[t];
    }
    std::vector<int32_t> red_off(static_cast<size_t>(T) + 1, 0);
    for (int t = 0; t < T; ++t) {
      const TileDesc& td = all_tiles[static_cast<size_t>(g.tile_offset + t)];
      red_off[static_cast<size_t>(t) + 1] = red_off[static_cast<size_t>(t)] + td.rows * (td.r_pad / 4);
    }
    std::vector<int32_t> tables;
    tables.insert(tables.end(), sb.begin(), sb.end());
    tables.insert(tables.end(), eb0.begin(), eb0.end());
    tables.insert(tables.end(), eb1.begin(), eb1.end());
    tables.insert(tables.end(), slot0.begin(), slot0.end());
    tables.insert(tables.end(), nseg.begin(), nseg.end());
    tables.insert(tables.end(), off.begin(), off.end());
    tables.insert(tables.end(), red_off.begin(), red_off.end());
    {  // tile of each CTA's first reduction item (split_reduce_mid)
      const int64_t total = red_off[static_cast<size_t>(T)];
      for (int b = 0; b < P; ++b) {
        const int32_t i = static_cast<int32_t>((total * b) / P);
        const int t = static_cast<int>(std::upper_bound(red_off.begin(), red_off.end(), i) - red_off.begin()) - 1;
        tables.push_back(std::clamp(t, 0, T - 1));
      }
    }
    auto& mb = plan->merged_bufs;
    mb = std::make_unique<SplitBufs>();
    mb->grid = P;
    mb->part_elems = static_cast<size_t>(total_seg) * kTileM * g.r_pad_max;
    mb->mid_elems = static_cast<size_t>(T) * kTileM * g.r_pad_max;
    mb->counter_elems = 2 + static_cast<size_t>(T);  // [2 reserved][per-tile mid readiness]
    mb->tables.alloc(tables.size());
    CUDA_CHECK(cudaMemcpy(mb->tables.p, tables.data(), tables.size() * 4, cudaMemcpyHostToDevice));
  }
  build_stream(*plan, all_tiles, reg);
  plan->d_rows.alloc(rows32.size());
  CUDA_CHECK(cudaMemcpy(plan->d_rows.p, rows32.data(), rows32.size() * 4, cudaMemcpyHostToDevice));
  plan->rows_host = std::move(rows32);
  {
    std::vector<int32_t> tr(all_tiles.size() * kTileM);
    for (size_t t = 0; t < all_tiles.size(); ++t) {
      TileDesc& td = all_tiles[t];
      for (int i = 0; i < kTileM; ++i) {
        tr[t * kTileM + i] = plan->rows_host[static_cast<size_t>(td.row_begin + std::min(i, std::max(td.rows, 1) - 1))];
      }
      // consecutive rows (a prefill request, a sorted batch): the split
      // kernels move the tile's X / Y by TMA boxes instead of row gathers
      bool contig = td.rows > 0;
      for (int i = 1; contig && i < td.rows; ++i) contig = tr[t * kTileM + i] == tr[t * kTileM] + i;
      td.x_row0 = contig ? tr[t * kTileM] : -1;
      if (contig) plan->any_contig = true;
    }
    plan->d_tile_rows.alloc(std::max<size_t>(tr.size(), 1));
    if (!tr.empty()) CUDA_CHECK(cudaMemcpy(plan->d_tile_rows.p, tr.data(), tr.size() * 4, cudaMemcpyHostToDevice));
  }
  plan->d_tiles.alloc(all_tiles.size());
  CUDA_CHECK(cudaMemcpy(plan->d_tiles.p, all_tiles.data(), all_tiles.size() * sizeof(TileDesc),
                        cudaMemcpyHostToDevice));
  if (chunk == 0 && !reg->extra.empty()) {
    int max_ch = 1;
    for (size_t s = 0; s < S; ++s) max_ch = std::max(max_ch, reg->num_chunks(plan->bp.seg_adapter[s]));
    for (int c = 1; c < max_ch; ++c) {
      std::vector<int32_t> asg, map;
      for (int64_t i = 0; i < n; ++i) {
        if (reg->num_chunks(assignment[i]) > c) {
          asg.push_back(assignment[i]);
          map.push_back(row_map ? row_map[i] : static_cast<int32_t>(i));
        }
      }
      auto ps = build_plan(reg, asg.data(), static_cast<int64_t>(asg.size()), table, forced, map.data(), plan->n, c);
      plan->flops += ps->flops;
      plan->total_ctas += ps->total_ctas;
      plan->passes.push_back(std::move(ps));
    }
  }
  return plan;
}

// =========================================================================
// Programmatic-dependency elision for the all-to-all bypass
// =========================================================================
// Every bypass launch carries the programmatic-stream-serialization
// attribute, and atmm_bypass_a2a_kernel follows a wait-before-trigger
// protocol (kernels.cu): a thread releases the next launch only after its own
// griddepcontrol.wait returned, i.e. once the grid BEFORE it is complete.  So
// when an a2a grid starts, at most one earlier grid can still be running: the
// launch immediately preceding it on the stream.  If that launch is an a2a
// bypass whose X / Y bytes are disjoint from this launch's (no RAW on X or Y,
// no WAW on Y, no WAR on the predecessor's X), nothing this launch reads or
// writes can be touched by a running grid, and it loads X and Y before its
// own griddepcontrol.wait (BypassParams::early): consecutive independent
// batches overlap, dependent ones (Y_i feeds X_i+1) keep the full dependency.
// The record is per (stream, capture sequence); under stream capture the
// predecessor is also checked by graph node identity (cudaStreamGetCaptureInfo),
// so a kernel captured in between can never be mistaken for our launch.
// Other library launches with the PDL attribute invalidate the record
// (pdl_note_other); launches without it serialise fully and only make the
// check conservative.  Limit (documented in include/atmm_b200.h): a foreign
// kernel launched WITH the PDL attribute between two eager library launches
// on one stream is not seen; such callers set ATMM_PLAN_NO_OVERLAP.
namespace {
struct PdlRange {
  uintptr_t lo = 0, hi = 0;
  bool overlaps(const PdlRange& o) const { return lo < o.hi && o.lo < hi; }
};
struct PdlRecord {
  bool valid = false;
  int n = 0;
  PdlRange x[kMaxGroup], y[kMaxGroup];
  cudaGraphNode_t node = nullptr;  // capture: the graph node of the launch
};
struct PdlKey {
  cudaStream_t s;
  unsigned long long capture;
  bool operator<(const PdlKey& o) const { return s != o.s ? s < o.s : capture < o.capture; }
};
std::mutex g_pdl_mu;
std::map<PdlKey, PdlRecord> g_pdl;
std::atomic<int64_t> g_a2a_launches{0}, g_a2a_early{0}, g_split_launches{0}, g_split_early{0};

struct PdlCapture {
  bool capturing = false;
  unsigned long long id = 0;
  cudaGraphNode_t single_dep = nullptr;  // the one current dependency, if exactly one
};
PdlCapture pdl_capture_info(cudaStream_t s) {
  PdlCapture c;
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  if (cudaStreamGetCaptureInfo(s, &st, &c.id, nullptr, &deps, &ndeps) != cudaSuccess) {
    cudaGetLastError();
    c.capturing = true;  // unknown: treat as a capture with no usable record
    c.id = ~0ull;
    return c;
  }
  c.capturing = st == cudaStreamCaptureStatusActive;
  if (!c.capturing) c.id = 0;
  if (c.capturing && ndeps == 1) c.single_dep = deps[0];
  return c;
}
}  // namespace

void pdl_note_other(cudaStream_t s) {
  const PdlCapture c = pdl_capture_info(s);
  std::lock_guard<std::mutex> lk(g_pdl_mu);
  auto it = g_pdl.find(PdlKey{s, c.id});
  if (it != g_pdl.end()) it->second.valid = false;
}

// Whether an a2a launch touching xs / ys may load them before waiting for
// the preceding launch on `s` (see above).
static bool pdl_can_elide(cudaStream_t s, const PdlCapture& c, const PdlRange* xs, const PdlRange* ys, int n) {
  std::lock_guard<std::mutex> lk(g_pdl_mu);
  auto it = g_pdl.find(PdlKey{s, c.id});
  if (it == g_pdl.end() || !it->second.valid) return false;
  const PdlRecord& r = it->second;
  if (c.capturing && (c.single_dep == nullptr || c.single_dep != r.node)) return false;
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < r.n; ++j) {
      if (xs[i].overlaps(r.y[j]) || ys[i].overlaps(r.y[j]) || ys[i].overlaps(r.x[j])) return false;
    }
  }
  return true;
}

// Whether a launch that only READS xs before its own griddepcontrol.wait
// (the split shrink; it writes nothing but private scratch) may start under
// the preceding launch on `s`: that launch is a recorded bypass whose Y
// writes miss xs.
static bool pdl_can_elide_reads(cudaStream_t s, const PdlCapture& c, const PdlRange* xs, int n) {
  std::lock_guard<std::mutex> lk(g_pdl_mu);
  auto it = g_pdl.find(PdlKey{s, c.id});
  if (it == g_pdl.end() || !it->second.valid) return false;
  const PdlRecord& r = it->second;
  if (c.capturing && (c.single_dep == nullptr || c.single_dep != r.node)) return false;
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < r.n; ++j) {
      if (xs[i].overlaps(r.y[j])) return false;
    }
  }
  return true;
}

static void pdl_record_a2a(cudaStream_t s, const PdlRange* xs, const PdlRange* ys, int n) {
  const PdlCapture c = pdl_capture_info(s);  // after the launch: its node is the dependency
  std::lock_guard<std::mutex> lk(g_pdl_mu);
  if (g_pdl.size() > 4096) g_pdl.clear();  // forgetting records only makes the check conservative
  PdlRecord& r = g_pdl[PdlKey{s, c.id}];
  r.valid = !c.capturing || c.single_dep != nullptr;
  r.node = c.single_dep;
  r.n = n;
  for (int i = 0; i < n; ++i) {
    r.x[i] = xs[i];
    r.y[i] = ys[i];
  }
}

static PdlRange byte_range(const void* base, int64_t rows, int64_t cols, int64_t ld, int64_t esz) {
  const uintptr_t lo = reinterpret_cast<uintptr_t>(base);
  const int64_t bytes = rows > 0 ? ((rows - 1) * ld + cols) * esz : 0;
  return PdlRange{lo, lo + static_cast<uintptr_t>(bytes)};
}

// Debug-only phase tracing (tools/profile_trace.py): a device buffer of
// >= ctas * kTraceEvents uint64 filled by the next bypass launches.
static uint64_t* g_trace = nullptr;

// Whether an apply runs as one stream launch (atmm_stream_kernel).
static bool stream_auto(const atmm_plan& p) {
  (void)p;
  return false;
}
static bool use_stream(const atmm_plan& p, bool y_vec) {
  if (!p.stream.ok || !y_vec || !p.stream_bufs) return false;
  return p.stream_mode == 1 || (p.stream_mode == 2 && stream_auto(p));
}

static void launch_stream_plan(const atmm_plan* p, int64_t layer, const void* x, int64_t ldx, void* y, int64_t ldy,
                               int y_dtype, float scale, cudaStream_t stream) {
  const atmm_registry* reg = p->reg;
  const StreamLayout& l = p->stream;
  SplitBufs& sb = *p->stream_bufs;
  SplitScratch& sc = sb.for_stream(stream);
  const int P = sb.grid;
  const int T = static_cast<int>(p->d_tiles.n);
  const int di = y_dtype == ATMM_BF16 ? 0 : 1;
  StreamParams sp{};
  sp.tiles = p->d_tiles.p;
  sp.row_index = p->d_rows.p;
  sp.x = static_cast<const uint16_t*>(x);
  sp.ldx = ldx;
  sp.y = y;
  sp.ldy = ldy;
  sp.d_in = static_cast<int32_t>(reg->d_in);
  sp.d_out = static_cast<int32_t>(reg->d_out);
  sp.layer = static_cast<int32_t>(layer);
  sp.scale = scale;
  sp.num_tiles = T;
  sp.nkb = static_cast<int32_t>((reg->d_in + kBK - 1) / kBK);
  sp.nsl = l.nsl;
  sp.r_pad_max = l.r_pad_max;
  sp.rows_max = l.rows_max;
  sp.sstages = l.sstages[di];
  sp.estages = l.estages[di];
  sp.s_stage_bytes = l.s_stage;
  sp.s_a_bytes = l.s_a;
  sp.e_stage_bytes = l.e_stage[di];
  sp.off_e = l.off_e[di];
  sp.off_mid = l.off_mid[di];
  sp.mid_bytes = l.mid_bytes;
  sp.tmem_cols = l.tmem_cols;
  sp.x_ready = (p->flags & ATMM_PLAN_X_READY) ? 1 : 0;
  sp.s_begin = sb.tables.p;
  sp.e_begin = sp.s_begin + (P + 1);
  sp.seg_slot0 = sp.e_begin + (P + 1);
  sp.nseg = sp.seg_slot0 + P;
  sp.part_off = sp.nseg + T;
  sp.ncons = sp.part_off + T;
  sp.part = sc.part.p;
  sp.counter = sc.counter.p;
  sp.trace = g_trace;
  pdl_note_other(stream);
  const cudaError_t e = launch_stream(di, sp, P, l.smem[di], stream);
  if (e != cudaSuccess) fail(ATMM_ERR_CUDA, std::string("stream bypass launch failed: ") + cudaGetErrorString(e));
}

// count > 1: independent calls (xs[c], ys[c], layers[c]) of one plan; the
// all-to-all kernel runs them as ONE launch, other paths launch per call.
static void apply_pass(const atmm_plan* p, int64_t layer, const void* x, int64_t ldx, void* y,
                       int64_t ldy, int y_dtype, float scale, cudaStream_t stream, int count = 1,
                       const int64_t* layers = nullptr, const void* const* xs = nullptr, void* const* ys = nullptr);
// One apply: the plan, then its rank-chunk passes (atmm_plan::passes) in
// stream order over the same X / Y.
static void apply_plan(const atmm_plan* p, int64_t layer, const void* x, int64_t ldx, void* y,
                       int64_t ldy, int y_dtype, float scale, cudaStream_t stream, int count = 1,
                       const int64_t* layers = nullptr, const void* const* xs = nullptr, void* const* ys = nullptr) {
  apply_pass(p, layer, x, ldx, y, ldy, y_dtype, scale, stream, count, layers, xs, ys);
  for (const auto& ps : p->passes) apply_pass(ps.get(), layer, x, ldx, y, ldy, y_dtype, scale, stream, count, layers, xs, ys);
}

static void apply_pass(const atmm_plan* p, int64_t layer, const void* x, int64_t ldx, void* y,
                       int64_t ldy, int y_dtype, float scale, cudaStream_t stream, int count,
                       const int64_t* layers, const void* const* xs, void* const* ys) {
  const atmm_registry* reg = p->reg;
  if (p->generation != reg->generation) fail(ATMM_ERR_CONFIG, "plan is stale: the registry changed after the plan was built");
  if (layer < 0 || layer >= reg->L) {
    fail(ATMM_ERR_CONFIG, "layer index " + std::to_string(layer) + " out of range (L=" + std::to_string(reg->L) + ")");
  }
  if (y_dtype != ATMM_BF16 && y_dtype != ATMM_F32) fail(ATMM_ERR_CONFIG, "y_dtype must be ATMM_BF16 or ATMM_F32");
  if (!x || !y) fail(ATMM_ERR_SHAPE, "null X or Y");
  if (ldx < reg->d_in || ldx % 8 != 0 || reinterpret_cast<uintptr_t>(x) % 16 != 0) {
    fail(ATMM_ERR_SHAPE, "X must be 16-byte aligned with ldx >= d_in and ldx % 8 == 0");
  }
  const int64_t ysz = y_dtype == ATMM_BF16 ? 2 : 4;
  if (ldy < reg->d_out) fail(ATMM_ERR_SHAPE, "Y row stride ldy must be >= d_out");
  if (reinterpret_cast<uintptr_t>(y) % ysz != 0) fail(ATMM_ERR_SHAPE, "Y is not element aligned");
  int32_t y_vec = ((ldy * ysz) % 16 == 0 && reinterpret_cast<uintptr_t>(y) % 16 == 0) ? 1 : 0;
  if (use_stream(*p, y_vec != 0)) {
    if (count > 1) {
      if (count > kMaxGroup || !layers || !xs || !ys) fail(ATMM_ERR_CONFIG, "grouped apply: 1..8 calls with layers, xs, ys");
      for (int c = 0; c < count; ++c) apply_pass(p, layers[c], xs[c], ldx, ys[c], ldy, y_dtype, scale, stream);
      return;
    }
    launch_stream_plan(p, layer, x, ldx, y, ldy, y_dtype, scale, stream);
    return;
  }
  if (count > 1) {
    if (count > kMaxGroup || !layers || !xs || !ys) fail(ATMM_ERR_CONFIG, "grouped apply: 1..8 calls with layers, xs, ys");
    bool all_a2a = y_vec != 0;
    for (int c = 0; c < count; ++c) {
      if (layers[c] < 0 || layers[c] >= reg->L) fail(ATMM_ERR_CONFIG, "layer index out of range in grouped apply");
      if (!xs[c] || !ys[c] || reinterpret_cast<uintptr_t>(xs[c]) % 16 != 0 || reinterpret_cast<uintptr_t>(ys[c]) % 16 != 0) {
        all_a2a = false;
      }
    }
    for (const LaunchGroup& g : p->groups) all_a2a = all_a2a && choose_path(g, y_dtype, true) == BypassPath::kA2a;
    if (!all_a2a) {
      for (int c = 0; c < count; ++c) apply_pass(p, layers[c], xs[c], ldx, ys[c], ldy, y_dtype, scale, stream);
      return;
    }
  }
  // Tensor maps are encoded on first use only (the split path needs none) and
  // cached per thread by (base, shape, stride): serving loops reuse buffers.
  CUtensorMap tmap_x_v, tmap_y_v;
  bool have_x = false, have_y = false;
  auto tmap_x_get = [&]() -> const CUtensorMap& {
    if (!have_x) {
      tmap_x_v = cached_map(0, x, p->n, reg->d_in, ldx);
      have_x = true;
    }
    return tmap_x_v;
  };
  auto tmap_y_get = [&]() -> const CUtensorMap& {
    if (!have_y) {
      tmap_y_v = y_vec ? cached_map(1 + y_dtype, y, p->n, reg->d_out, ldy) : tmap_x_get();
      have_y = true;
    }
    return tmap_y_v;
  };

  bool merged_ok = p->merged_first >= 0;
  for (size_t gi = merged_ok ? static_cast<size_t>(p->merged_first) : 0; merged_ok && gi < p->groups.size(); ++gi) {
    merged_ok = choose_path(p->groups[gi], y_dtype, y_vec != 0) == BypassPath::kSplit;
  }
  const size_t ng = merged_ok ? static_cast<size_t>(p->merged_first) + 1 : p->groups.size();
  for (size_t gi = 0; gi < ng; ++gi) {
    const bool as_merged = merged_ok && gi == static_cast<size_t>(p->merged_first);
    const LaunchGroup& g = as_merged ? p->merged : p->groups[gi];
    BypassPath path = as_merged ? BypassPath::kSplit : choose_path(g, y_dtype, y_vec != 0);
    if (path == BypassPath::kSplit && !as_merged) path = BypassPath::kFused;  // split runs only as the merged range
    if (path == BypassPath::kSplit) {
      SplitBufs& sb = *p->merged_bufs;
      SplitScratch& sc = sb.alternate(stream);
      const int P = sb.grid;
      const int T = static_cast<int>(g.num_tiles);
      SplitParams sp{};
      sp.tiles = p->d_tiles.p + g.tile_offset;
      sp.row_index = p->d_rows.p;
      sp.x = static_cast<const uint16_t*>(x);
      sp.ldx = ldx;
      sp.y = y;
      sp.ldy = ldy;
      sp.d_in = static_cast<int32_t>(reg->d_in);
      sp.d_out = static_cast<int32_t>(reg->d_out);
      sp.layer = static_cast<int32_t>(layer);
      sp.scale = scale;
      sp.num_tiles = T;
      sp.nkb = static_cast<int32_t>((reg->d_in + kBK - 1) / kBK);
      sp.r_pad_max = g.r_pad_max;
      sp.stages = g.split.stages;
      sp.y_dtype = y_dtype == ATMM_BF16 ? 0 : 1;
      sp.estages = g.split.estages[sp.y_dtype];
      sp.expand_g = sp.y_dtype == 0 ? g.split.g_bf16 : 1;
      sp.e_tmem_cols = g.split.tmem_e[sp.y_dtype];
      sp.out_staged = split_out_staged(sp.expand_g);
      // The shrink may run under the preceding launch (until its own end)
      // when that launch is a recorded bypass whose writes miss X: it reads
      // only X, the factors and its own scratch set (the other set than the
      // preceding apply of this plan on this stream).
      PdlRange xr = byte_range(x, p->n, reg->d_in, ldx, 2), yr = byte_range(y, p->n, reg->d_out, ldy, ysz);
      sp.early = (p->flags & ATMM_PLAN_NO_OVERLAP) ? 0 : (pdl_can_elide_reads(stream, pdl_capture_info(stream), &xr, 1) ? 1 : 0);
      sp.rows_max = g.rows_max;
      sp.s_begin = sb.tables.p;
      sp.e_begin = sb.tables.p + (P + 1) * (sp.y_dtype == 0 ? 1 : 2);
      sp.seg_slot0 = sb.tables.p + 3 * (P + 1);
      sp.nseg = sp.seg_slot0 + P;
      sp.part_off = sp.nseg + T;
      sp.red_off = sp.part_off + T;
      sp.red_tile0 = sp.red_off + T + 1;
      sp.tile_rows = p->d_tile_rows.p + g.tile_offset * kTileM;
      sp.part = sc.part.p;
      sp.mid = sc.mid.p;
      sp.counter = sc.counter.p;
      sp.trace = g_trace;
      pdl_note_other(stream);
      // tiles of consecutive rows load X by 128-row TMA boxes (TileDesc::x_row0)
      CUtensorMap xtile{}, ytile{};
      sp.contig = p->any_contig ? 1 : 0;
      if (p->any_contig) {
        xtile = cached_map(3, x, p->n, reg->d_in, ldx);
        ytile = y_tile_map(y, p->n, reg->d_out, ldy, y_dtype, 128 * sp.expand_g, sp.rows_max);
      }
      const cudaError_t e = launch_split(sp.y_dtype, xtile, ytile, sp, P, g.split.smem_s, g.split.smem_e[sp.y_dtype], stream);
      if (e != cudaSuccess) fail(ATMM_ERR_CUDA, std::string("bypass launch failed: ") + cudaGetErrorString(e));
      pdl_record_a2a(stream, &xr, &yr, 1);  // the expand: reads / writes Y, the shrink read X
      g_split_launches.fetch_add(1, std::memory_order_relaxed);
      if (sp.early) g_split_early.fetch_add(1, std::memory_order_relaxed);
      continue;
    }
    BypassParams bp{};
    bp.tiles = p->d_tiles.p + g.tile_offset;
    bp.row_index = p->d_rows.p;
    bp.tile_rows = p->d_tile_rows.p + g.tile_offset * kTileM;
    bp.x = static_cast<const uint16_t*>(x);
    bp.ldx = ldx;
    bp.y = y;
    bp.ldy = ldy;
    bp.n_rows = static_cast<int32_t>(p->n);
    bp.d_in = static_cast<int32_t>(reg->d_in);
    bp.d_out = static_cast<int32_t>(reg->d_out);
    bp.layer = static_cast<int32_t>(layer);
    bp.scale = scale;
    bp.stages = g.stages;
    bp.stage_bytes = g.stage_bytes;
    bp.a_bytes = g.a_bytes;
    bp.bn = g.bn;
    bp.ustages = g.ustages;
    bp.ustage_bytes = g.ustage_bytes;
    bp.ny = g.ny;
    bp.ycols = y_dtype == ATMM_BF16 ? 64 : 32;
    bp.ybuf_bytes = g.ybuf_bytes;
    bp.x_ready = (p->flags & ATMM_PLAN_X_READY) ? 1 : 0;
    bp.red_rows = g.red_rows;
    bp.r_pad_max = g.r_pad_max;
    bp.off_up = g.off_up;
    bp.off_y = g.off_y;
    bp.off_red = g.off_red;
    bp.off_mid = g.off_mid;
    bp.off_bar = g.off_bar;
    bp.tmem_cols = g.tmem_cols;
    bp.y_vec = y_vec;
    bp.y_ring = y_vec;
    bp.rep = g.rep;
    bp.nbuf = g.nbuf;
    bp.trace = g_trace;
    const A2aLayout& al = g.a2a[y_dtype == ATMM_BF16 ? 0 : 1];
    if (path == BypassPath::kA2a) {
      bp.stages = al.stages;
      bp.stage_bytes = al.stage_bytes;
      bp.a_bytes = al.a_bytes;
      bp.ypitch = al.ypitch;
      bp.gcols = al.gcols;
      bp.off_up = al.off_up;
      bp.off_y = al.off_y;
      bp.off_red = al.off_red;
      bp.off_mid = al.off_mid;
      bp.off_bar = al.off_bar;
      bp.tmem_cols = al.tmem_cols;
      GroupArgs ga{};
      ga.num_tiles = static_cast<int32_t>(g.num_tiles);
      ga.count = count > 1 ? count : 1;
      PdlRange xr[kMaxGroup], yr[kMaxGroup];
      for (int c = 0; c < ga.count; ++c) {
        const void* xc = count > 1 ? xs[c] : x;
        ga.x_map[c] = count > 1 ? cached_map(0, xc, p->n, reg->d_in, ldx) : tmap_x_get();
        ga.x[c] = xc;
        ga.y[c] = count > 1 ? ys[c] : y;
        ga.layer[c] = static_cast<int32_t>(count > 1 ? layers[c] : layer);
        xr[c] = byte_range(xc, p->n, reg->d_in, ldx, 2);
        yr[c] = byte_range(ga.y[c], p->n, reg->d_out, ldy, ysz);
      }
      // X and Y of one call overlapping each other (in-place use) is fine for
      // the predecessor check but not across calls of one grouped launch;
      // the latter is the caller's contract (atmm_bypass_apply_group).
      bp.early = (p->flags & ATMM_PLAN_NO_OVERLAP) ? 0 : (pdl_can_elide(stream, pdl_capture_info(stream), xr, yr, ga.count) ? 1 : 0);
      const cudaError_t e = launch_bypass_a2a(y_dtype, ga, bp, g.cluster, static_cast<int>(g.num_tiles), al.smem, stream);
      if (e != cudaSuccess) fail(ATMM_ERR_CUDA, std::string("bypass launch failed: ") + cudaGetErrorString(e));
      pdl_record_a2a(stream, xr, yr, ga.count);
      g_a2a_launches.fetch_add(1, std::memory_order_relaxed);
      if (bp.early) g_a2a_early.fetch_add(1, std::memory_order_relaxed);
      continue;
    }
    pdl_note_other(stream);
    const cudaError_t e = launch_bypass(y_dtype, tmap_x_get(), tmap_y_get(), bp, g.cluster, static_cast<int>(g.num_tiles), g.smem, stream);
    if (e != cudaSuccess) fail(ATMM_ERR_CUDA, std::string("bypass launch failed: ") + cudaGetErrorString(e));
  }
}

// W = beta*W + alpha * A . B on the merge kernel; A/B in registry layouts.
static void run_merge(const uint16_t* a_t, const uint16_t* b_t, int64_t m, int64_t n,
                      int64_t k_pad, void* w, int64_t ldw, int w_dtype, float alpha, float beta,
                      cudaStream_t stream, int64_t L = 1, int64_t a_ls = 0, int64_t b_ls = 0, int64_t w_ls = 0) {
  MergeParams mp{};
  mp.num_layers = 1;
  mp.a_t = a_t;
  mp.b_t = b_t;
  mp.w = w;
  mp.ldw = ldw;
  mp.m = static_cast<int32_t>(m);
  mp.n = static_cast<int32_t>(n);
  mp.k_pad = static_cast<int32_t>(k_pad);
  mp.bn = k_pad <= 64 ? 256 : 128;
  mp.num_mtiles = static_cast<int32_t>((m + kTileM - 1) / kTileM);
  mp.num_nchunks = static_cast<int32_t>((round_up(n, 32) + mp.bn - 1) / mp.bn);
  mp.alpha = alpha;
  mp.beta = beta;
  const int64_t wsz = w_dtype == ATMM_BF16 ? 2 : 4;
  mp.w_vec = ((ldw * wsz) % 16 == 0 && reinterpret_cast<uintptr_t>(w) % 16 == 0 && (w_ls * wsz) % 16 == 0) ? 1 : 0;
  if (L > 1 && !mp.w_vec) {  // one launch per layer on the direct-epilogue kernel
    for (int64_t l = 0; l < L; ++l) {
      run_merge(a_t + l * a_ls, b_t + l * b_ls, m, n, k_pad, static_cast<uint8_t*>(w) + l * w_ls * wsz, ldw, w_dtype,
                alpha, beta, stream);
    }
    return;
  }
  const int64_t a_bytes = int64_t(kTileM) * k_pad * 2;
  int sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (mp.w_vec) {
    // TMA-staged W: 128-column chunks (two TMEM accumulators of 128 columns),
    // two B stages, and every remaining byte of shared memory as W slabs.
    mp.bn = 128;
    mp.num_nchunks = static_cast<int32_t>((round_up(n, 32) + mp.bn - 1) / mp.bn);
    mp.slab_cols = static_cast<int32_t>(128 / wsz);
    mp.b_stage_bytes = static_cast<uint32_t>(round_up(int64_t(mp.bn) * k_pad * 2, 1024));
    mp.stages = 2;
    mp.off_b = static_cast<uint32_t>(round_up(a_bytes, 1024));
    mp.off_w = static_cast<uint32_t>(mp.off_b + int64_t(mp.stages) * mp.b_stage_bytes);
    const int64_t slab = int64_t(kTileM) * 128;
    auto total_w = [&](int sw) {
      return size_t(1024 + mp.off_w + int64_t(sw) * slab + round_up((2 * mp.stages + 6 + 2 * sw) * 8 + 8, 16));
    };
    int sw = 12;
    while (sw > 2 && total_w(sw) > kSmemLimit) --sw;
    mp.w_stages = sw;
    mp.off_bar = static_cast<uint32_t>(mp.off_w + int64_t(sw) * slab);
    mp.tmem_cols = 256;
    mp.num_layers = static_cast<int32_t>(L);
    mp.a_layer_stride = a_ls;
    mp.b_layer_stride = b_ls;
    const int64_t tiles = L * int64_t(mp.num_mtiles) * mp.num_nchunks;
    const int grid = static_cast<int>(std::min<int64_t>(tiles, sms));
    const CUtensorMap tmap_w = make_w_map(w, m, n, ldw, w_dtype, L, w_ls);
    const cudaError_t e = launch_merge_tma(w_dtype, tmap_w, mp, grid, total_w(sw), stream);
    if (e != cudaSuccess) fail(ATMM_ERR_CUDA, std::string("merge launch failed: ") + cudaGetErrorString(e));
    return;
  }
  mp.b_stage_bytes = static_cast<uint32_t>(round_up(int64_t(mp.bn) * k_pad * 2, 1024));
  int stages = 4;
  auto total = [&](int s) {
    return size_t(1024 + a_bytes + int64_t(s) * mp.b_stage_bytes + round_up((2 * s + 6) * 8 + 8, 16));
  };
  while (stages > 2 && total(stages) > kSmemLimit) --stages;
  mp.stages = stages;
  mp.off_b = static_cast<uint32_t>(a_bytes);
  mp.off_bar = static_cast<uint32_t>(a_bytes + int64_t(stages) * mp.b_stage_bytes);
  int32_t cols = 32;
  while (cols < 2 * mp.bn) cols <<= 1;
  mp.tmem_cols = static_cast<uint32_t>(cols);
  size_t smem = total(stages);
  const int max_co = std::max(1, 512 / cols);
  while (static_cast<int>(kSmemPerSM / (smem + 1024)) > max_co) smem += 4096;
  const int64_t tiles = int64_t(mp.num_mtiles) * mp.num_nchunks;
  const int grid = static_cast<int>(std::min<int64_t>(tiles, sms));
  const cudaError_t e = launch_merge(w_dtype, mp, grid, smem, stream);
  if (e != cudaSuccess) fail(ATMM_ERR_CUDA, std::string("merge launch failed: ") + cudaGetErrorString(e));
}

}  // namespace atmm

extern "C" {

int atmm_debug_set_trace(void* device_buffer) {
  g_trace = static_cast<uint64_t*>(device_buffer);
  return ATMM_OK;
}

int atmm_device_count(void) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int ok = 0;
  for (int d = 0; d < count; ++d) {
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, d) == cudaSuccess && prop.major == 10) ++ok;
  }
  return ok;
}

int atmm_registry_create(int device, int64_t num_layers, int64_t d_in, int64_t d_out,
                         atmm_registry** out) {
  return guarded([&] {
    if (!out) fail(ATMM_ERR_CONFIG, "null output");
    if (num_layers < 1 || d_in < 1 || d_out < 1) fail(ATMM_ERR_SHAPE, "registry dimensions must be >= 1");
    require_device(device);
    auto r = std::make_unique<atmm_registry>();
    r->device = device;
    r->L = num_layers;
    r->d_in = d_in;
    r->d_out = d_out;
    r->d_in_pad = round_up(d_in, 128);
    r->d_out_pad = round_up(d_out, 128);  // every kernel may read up^T rows up to a 128-row boundary
    *out = r.release();
  });
}

void atmm_registry_destroy(atmm_registry* r) { delete r; }

int atmm_registry_put(atmm_registry* r, int32_t adapter_id, int64_t rank, const float* down,
                      const float* up, float scale) {
  return guarded([&] {
    if (!r) fail(ATMM_ERR_CONFIG, "null registry");
    // The reference accepts any rank below the hidden size (adapter.hpp:30-31);
    // ranks above kMaxRank are stored as 128-rank chunk slots.
    if (rank < 1 || (rank > kMaxRank && rank >= std::min(r->d_in, r->d_out))) {
      fail(ATMM_ERR_CONFIG, "adapter rank must be >= 1 and < the hidden size");
    }
    if (!down || !up) fail(ATMM_ERR_SHAPE, "null factors");
    const int nch = static_cast<int>((rank + kMaxRank - 1) / kMaxRank);
    if (nch > 1 && r->precise) fail(ATMM_ERR_CONFIG, "a precise registry takes ranks <= 128");
    DeviceGuard g(r->device);
    // One slot per 128-rank chunk (columns [128 c, ..) of down, rows of up).
    std::vector<Slot> made;
    for (int c = 0; c < nch; ++c) {
      const int64_t r0 = int64_t(c) * kMaxRank, rc = std::min<int64_t>(kMaxRank, rank - r0);
      const int64_t r_pad = round_up(rc, 16);
      const size_t dn = static_cast<size_t>(r->d_in_pad * r_pad);
      const size_t un = static_cast<size_t>(r->d_out_pad * r_pad);
      std::vector<uint16_t> hd(dn * static_cast<size_t>(r->L)), hu(un * static_cast<size_t>(r->L));
      for (int64_t l = 0; l < r->L; ++l) {
        pack_down_t(down + l * r->d_in * rank + r0, r->d_in, rc, rank, r->d_in_pad, r_pad, hd.data() + l * dn);
        pack_up_t(up + l * rank * r->d_out + r0 * r->d_out, rc, r->d_out, r->d_out, r->d_out_pad, r_pad,
                  hu.data() + l * un);
      }
      Slot s;
      s.id = adapter_id;
      s.rank = rc;
      s.r_pad = r_pad;
      s.alg_rank = rc;
      s.total_rank = rank;
      s.scale = scale;
      s.live = true;
      CUDA_CHECK(cudaMalloc(&s.down_t, hd.size() * 2));
      CUDA_CHECK(cudaMalloc(&s.up_t, hu.size() * 2));
      CUDA_CHECK(cudaMemcpy(s.down_t, hd.data(), hd.size() * 2, cudaMemcpyHostToDevice));
      CUDA_CHECK(cudaMemcpy(s.up_t, hu.data(), hu.size() * 2, cudaMemcpyHostToDevice));
      made.push_back(s);
    }
    Slot s = made[0];
    if (r->precise) build_precise_host(r, s, down, up);
    r->drop_extra(adapter_id);
    if (nch > 1) {
      std::vector<int> idx;
      for (int c = 1; c < nch; ++c) {
        const int i = r->free_index();
        r->slots[static_cast<size_t>(i)] = made[static_cast<size_t>(c)];
        idx.push_back(i);
      }
      r->extra[adapter_id] = idx;
    }
    auto it = r->slot_of.find(adapter_id);
    if (it != r->slot_of.end()) {
      Slot& old = r->slots[static_cast<size_t>(it->second)];
      free_slot(old);
      old = s;
    } else {
      int idx = -1;
      for (size_t i = 0; i < r->slots.size(); ++i) {
        if (!r->slots[i].live) {
          idx = static_cast<int>(i);
          break;
        }
      }
      if (idx < 0) {
        idx = static_cast<int>(r->slots.size());
        r->slots.push_back(s);
      } else {
        r->slots[static_cast<size_t>(idx)] = s;
      }
      r->slot_of[adapter_id] = idx;
    }
    r->sync_slots();
  });
}

int atmm_registry_put_combined(atmm_registry* r, int32_t new_id, int64_t n_parts, const int32_t* part_ids,
                               const float* part_signs) {
  return guarded([&] {
    if (!r || !part_ids || !part_signs || n_parts < 1) fail(ATMM_ERR_CONFIG, "null registry or empty part list");
    if (r->precise) fail(ATMM_ERR_CONFIG, "combined slots are not built on a precise registry (apply the parts)");
    std::vector<Slot> parts;
    int64_t r_c = 0, alg = 0;
    for (int64_t i = 0; i < n_parts; ++i) {
      r->require_unchunked(part_ids[i], "combined slot");
      parts.push_back(r->at(part_ids[i]));
      r_c += parts.back().r_pad;
      alg += parts.back().alg_rank;
    }
    if (r_c > kMaxRank) fail(ATMM_ERR_CONFIG, "combined rank " + std::to_string(r_c) + " exceeds 128");
    DeviceGuard g(r->device);
    r->drop_extra(new_id);
    Slot s;
    s.id = new_id;
    s.rank = r_c;
    s.r_pad = r_c;
    s.alg_rank = alg;
    s.total_rank = r_c;
    s.scale = 1.0f;
    s.live = true;
    const size_t dn = static_cast<size_t>(r->d_in_pad * r_c), un = static_cast<size_t>(r->d_out_pad * r_c);
    CUDA_CHECK(cudaMalloc(&s.down_t, dn * static_cast<size_t>(r->L) * 2));
    CUDA_CHECK(cudaMalloc(&s.up_t, un * static_cast<size_t>(r->L) * 2));
    int64_t off = 0;
    for (size_t i = 0; i < parts.size(); ++i) {
      const Slot& ps = parts[i];
      const float f = part_signs[i] * ps.scale;
      for (int64_t l = 0; l < r->L; ++l) {
        // down^T: per 64-wide K block r_pad x 64 contiguous -> rank rows off ..
        CUDA_CHECK(cudaMemcpy2D(s.down_t + l * dn + off * kBK, static_cast<size_t>(r_c * kBK * 2),
                                ps.down_t + l * r->d_in_pad * ps.r_pad, static_cast<size_t>(ps.r_pad * kBK * 2),
                                static_cast<size_t>(ps.r_pad * kBK * 2), static_cast<size_t>(r->d_in_pad / kBK),
                                cudaMemcpyDeviceToDevice));
        // up^T: per 8 output columns r_pad x 8 contiguous -> rank columns off ..
        uint16_t* ud = s.up_t + l * un + off * 8;
        CUDA_CHECK(cudaMemcpy2D(ud, static_cast<size_t>(r_c * 16), ps.up_t + l * r->d_out_pad * ps.r_pad,
                                static_cast<size_t>(ps.r_pad * 16), static_cast<size_t>(ps.r_pad * 16),
                                static_cast<size_t>(r->d_out_pad / 8), cudaMemcpyDeviceToDevice));
        if (f != 1.0f) {
          CUDA_CHECK(launch_scale_bf16_2d(ud, r->d_out_pad / 8, ps.r_pad * 8, r_c * 8, f, nullptr));
        }
      }
      off += ps.r_pad;
    }
    CUDA_CHECK(cudaDeviceSynchronize());
    auto it = r->slot_of.find(new_id);
    if (it != r->slot_of.end()) {
      Slot& old = r->slots[static_cast<size_t>(it->second)];
      free_slot(old);
      old = s;
    } else {
      int idx = -1;
      for (size_t i = 0; i < r->slots.size(); ++i) {
        if (!r->slots[i].live) {
          idx = static_cast<int>(i);
          break;
        }
      }
      if (idx < 0) {
        idx = static_cast<int>(r->slots.size());
        r->slots.push_back(s);
      } else {
        r->slots[static_cast<size_t>(idx)] = s;
      }
      r->slot_of[new_id] = idx;
    }
    r->sync_slots();
  });
}

int atmm_registry_put_async(atmm_registry* r, int32_t adapter_id, int64_t rank, const float* down,
                            const float* up, float scale, void* stream) {
  return guarded([&] {
    if (!r) fail(ATMM_ERR_CONFIG, "null registry");
    if (rank < 1 || rank > kMaxRank) fail(ATMM_ERR_CONFIG, "put_async takes ranks in [1, 128] (larger ranks: put)");
    if (!down || !up) fail(ATMM_ERR_SHAPE, "null factors");
    DeviceGuard g(r->device);
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t r_pad = round_up(rank, 16);
    const size_t dn = static_cast<size_t>(r->d_in_pad * r_pad) * static_cast<size_t>(r->L);
    const size_t un = static_cast<size_t>(r->d_out_pad * r_pad) * static_cast<size_t>(r->L);
    const size_t fd = static_cast<size_t>(r->L * r->d_in * rank), fu = static_cast<size_t>(r->L * rank * r->d_out);
    Slot s;
    s.id = adapter_id;
    s.rank = rank;
    s.r_pad = r_pad;
    s.alg_rank = rank;
    s.total_rank = rank;
    s.scale = scale;
    s.live = true;
    // A swap of the same shape overwrites the slot's buffers in place (stream
    // order: after every earlier use on this stream); the fp32 staging buffer
    // is the registry's, grow-only -- no allocation on the swap path.
    auto it = r->slot_of.find(adapter_id);
    Slot* same = nullptr;
    if (it != r->slot_of.end() && r->slots[static_cast<size_t>(it->second)].r_pad == r_pad &&
        r->slots[static_cast<size_t>(it->second)].async_owned) {
      same = &r->slots[static_cast<size_t>(it->second)];
      s.down_t = same->down_t;
      s.up_t = same->up_t;
    } else {
      CUDA_CHECK(cudaMallocAsync(&s.down_t, dn * 2, st));
      CUDA_CHECK(cudaMallocAsync(&s.up_t, un * 2, st));
    }
    s.async_owned = true;
    DevBuf<float>& stage_buf = r->stage_for(st);
    if (stage_buf.n < fd + fu) {
      CUDA_CHECK(cudaStreamSynchronize(st));  // the old staging buffer may still be read on this stream
      stage_buf.alloc(fd + fu);
    }
    float* stage = stage_buf.p;
    CUDA_CHECK(cudaMemcpyAsync(stage, down, fd * 4, cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaMemcpyAsync(stage + fd, up, fu * 4, cudaMemcpyHostToDevice, st));
    CUDA_CHECK(launch_pack_factors(stage, stage + fd, r->L, r->d_in, r->d_out, rank, r->d_in_pad, r->d_out_pad, r_pad,
                                   s.down_t, s.up_t, st));
    if (r->precise) {
      if (same) {  // a same-shape swap reuses the bf16 buffers; the images are rebuilt
        for (uint16_t* p : {same->p_down_b, same->p_up_b, same->p_down_a}) {
          if (p) CUDA_CHECK(cudaFreeAsync(p, st));
        }
      }
      build_precise_device(r, s, stage, stage + fd, st, true);
    }
    if (r->extra.count(adapter_id)) {  // replacing a rank-chunked adapter: its extra chunks go
      CUDA_CHECK(cudaStreamSynchronize(st));
      r->drop_extra(adapter_id);
    }
    if (same) {
      *same = s;
    } else if (it != r->slot_of.end()) {
      Slot& old = r->slots[static_cast<size_t>(it->second)];
      if (old.async_owned) {
        free_slot(old, st, true);  // stream order: after every earlier use on this stream
      } else {
        CUDA_CHECK(cudaStreamSynchronize(st));
        free_slot(old);
      }
      old = s;
    } else {
      int idx = -1;
      for (size_t i = 0; i < r->slots.size(); ++i) {
        if (!r->slots[i].live) {
          idx = static_cast<int>(i);
          break;
        }
      }
      if (idx < 0) {
        idx = static_cast<int>(r->slots.size());
        r->slots.push_back(s);
      } else {
        r->slots[static_cast<size_t>(idx)] = s;
      }
      r->slot_of[adapter_id] = idx;
    }
    r->sync_slots();
  });
}

int atmm_registry_load_fixture(atmm_registry* r, const char* dir, int64_t* num_adapters) {
  return guarded([&] {
    if (!r || !dir) fail(ATMM_ERR_CONFIG, "null registry or directory");
    const FixtureManifest m = read_fixture_manifest(dir);
    if (m.num_layers != r->L || m.hidden_dim != r->d_in || m.hidden_dim != r->d_out) {
      fail(ATMM_ERR_SHAPE, "fixture (L=" + std::to_string(m.num_layers) + ", d=" + std::to_string(m.hidden_dim) +
                               ") does not match the registry (L=" + std::to_string(r->L) + ", d_in=" +
                               std::to_string(r->d_in) + ", d_out=" + std::to_string(r->d_out) + ")");
    }
    const std::string base(dir);
    for (const FixtureAdapter& a : m.adapters) {
      std::vector<float> down, up;
      for (int64_t l = 0; l < m.num_layers; ++l) {
        int64_t rr = 0, cc = 0;
        std::vector<float> dm = load_matrix_f32(base + "/" + a.down[static_cast<size_t>(l)], rr, cc);
        if (rr != r->d_in || cc != a.rank) fail(ATMM_ERR_SHAPE, "adapter " + std::to_string(a.id) + " down factor must be d x r");
        down.insert(down.end(), dm.begin(), dm.end());
        std::vector<float> um = load_matrix_f32(base + "/" + a.up[static_cast<size_t>(l)], rr, cc);
        if (rr != a.rank || cc != r->d_out) fail(ATMM_ERR_SHAPE, "adapter " + std::to_string(a.id) + " up factor must be r x d");
        up.insert(up.end(), um.begin(), um.end());
      }
      const int st = atmm_registry_put(r, a.id, a.rank, down.data(), up.data(), 1.0f);
      if (st != ATMM_OK) fail(st, atmm_last_error());
    }
    if (num_adapters) *num_adapters = static_cast<int64_t>(m.adapters.size());
  });
}

int atmm_registry_remove(atmm_registry* r, int32_t adapter_id) {
  return guarded([&] {
    if (!r) fail(ATMM_ERR_CONFIG, "null registry");
    auto it = r->slot_of.find(adapter_id);
    if (it == r->slot_of.end()) fail(ATMM_ERR_UNKNOWN_ADAPTER, "unknown adapter id " + std::to_string(adapter_id));
    DeviceGuard g(r->device);
    Slot& s = r->slots[static_cast<size_t>(it->second)];
    free_slot(s);
    s = Slot{};
    r->slot_of.erase(it);
    r->drop_extra(adapter_id);
    r->sync_slots();
  });
}

int atmm_registry_contains(const atmm_registry* r, int32_t adapter_id) {
  return r && r->slot_of.count(adapter_id) ? 1 : 0;
}

int atmm_registry_rank(const atmm_registry* r, int32_t adapter_id, int64_t* rank) {
  return guarded([&] {
    if (!r || !rank) fail(ATMM_ERR_CONFIG, "null registry or output");
    *rank = r->at(adapter_id).total_rank;
  });
}

int atmm_registry_bytes(const atmm_registry* r, int64_t* bytes) {
  return guarded([&] {
    if (!r || !bytes) fail(ATMM_ERR_CONFIG, "null registry or output");
    int64_t b = 0;
    for (const auto& s : r->slots) {
      if (s.live) b += r->L * (r->d_in_pad + r->d_out_pad) * s.r_pad * 2;
    }
    *bytes = b;
  });
}

int atmm_plan_create(atmm_registry* r, const int32_t* assignment, int64_t n, const atmm_table* table,
                     atmm_plan** out) {
  return guarded([&] {
    if (!r || !out) fail(ATMM_ERR_CONFIG, "null registry or output");
    const TilingTable* t = table ? &table->t : nullptr;
    *out = build_plan(r, assignment, n, t, nullptr).release();
  });
}

int atmm_plan_create_mapped(atmm_registry* r, const int32_t* assignment, const int32_t* rows, int64_t n,
                            int64_t n_rows, const atmm_table* table, atmm_plan** out) {
  return guarded([&] {
    if (!r || !out) fail(ATMM_ERR_CONFIG, "null registry or output");
    if (!rows) fail(ATMM_ERR_SHAPE, "null row map");
    if (n_rows < n) fail(ATMM_ERR_SHAPE, "n_rows must be >= the number of routed rows");
    const TilingTable* t = table ? &table->t : nullptr;
    *out = build_plan(r, assignment, n, t, nullptr, rows, n_rows).release();
  });
}

int atmm_plan_create_launch(atmm_registry* r, const int32_t* assignment, int64_t n, const int32_t launch[5],
                            atmm_plan** out) {
  return guarded([&] {
    if (!r || !out || !launch) fail(ATMM_ERR_CONFIG, "null registry, launch or output");
    const LaunchCfg lc = launch_from_ints(launch);
    validate_launch(lc);
    *out = build_plan(r, assignment, n, nullptr, &lc).release();
  });
}

int atmm_overlap_stats(int64_t* a2a_launches, int64_t* early_launches) {
  if (a2a_launches) *a2a_launches = g_a2a_launches.load();
  if (early_launches) *early_launches = g_a2a_early.load();
  return ATMM_OK;
}

int atmm_split_overlap_stats(int64_t* split_launches, int64_t* early_launches) {
  if (split_launches) *split_launches = g_split_launches.load();
  if (early_launches) *early_launches = g_split_early.load();
  return ATMM_OK;
}

int atmm_plan_set_flags(atmm_plan* p, uint32_t flags) {
  return guarded([&] {
    if (!p) fail(ATMM_ERR_CONFIG, "null plan");
    if (flags & ~(ATMM_PLAN_X_READY | ATMM_PLAN_NO_OVERLAP)) fail(ATMM_ERR_CONFIG, "unknown plan flag");
    p->flags = flags;
  });
}

void atmm_plan_destroy(atmm_plan* p) {
  if (!p) return;
  DeviceGuard g(p->reg->device, std::nothrow);
  delete p;
}

int atmm_plan_routing(const atmm_plan* p, int32_t* seg_adapter, int64_t* seg_offsets,
                      int64_t* row_index, int64_t* num_segments) {
  return guarded([&] {
    if (!p) fail(ATMM_ERR_CONFIG, "null plan");
    // Read back what the kernels index with (row_index from HBM).
    DeviceGuard g(p->reg->device);
    std::vector<int32_t> rows(static_cast<size_t>(p->n_assign));
    CUDA_CHECK(cudaMemcpy(rows.data(), p->d_rows.p, rows.size() * 4, cudaMemcpyDeviceToHost));
    if (seg_adapter) std::copy(p->bp.seg_adapter.begin(), p->bp.seg_adapter.end(), seg_adapter);
    if (seg_offsets) std::copy(p->bp.seg_offsets.begin(), p->bp.seg_offsets.end(), seg_offsets);
    if (row_index) std::copy(rows.begin(), rows.end(), row_index);
    if (num_segments) *num_segments = static_cast<int64_t>(p->bp.seg_adapter.size());
  });
}

int atmm_plan_describe(const atmm_plan* p, char* buf, size_t cap) {
  return guarded([&] {
    if (!p || !buf || cap == 0) fail(ATMM_ERR_CONFIG, "null plan or buffer");
    std::string s = "[";
    std::vector<const atmm_plan*> all{p};
    for (const auto& ps : p->passes) all.push_back(ps.get());
    bool firstg = true;
    for (size_t pi = 0; pi < all.size(); ++pi) {
    const atmm_plan* pp = all[pi];
    for (size_t i = 0; i < pp->groups.size(); ++i) {
      const LaunchGroup& g = pp->groups[i];
      s += (firstg ? "" : ", ") + std::string("{\"pass\": ") + std::to_string(pi) + ", \"cluster\": " + std::to_string(g.cluster) +
           ", \"tiles\": " + std::to_string(g.num_tiles) + ", \"bn\": " + std::to_string(g.bn) +
           ", \"stages\": " + std::to_string(g.stages) + ", \"ustages\": " + std::to_string(g.ustages) +
           ", \"ny\": " + std::to_string(g.ny) + ", \"rep\": " + std::to_string(g.rep) +
           ", \"nbuf\": " + std::to_string(g.nbuf) + ", \"r_pad\": " + std::to_string(g.r_pad_max) +
           ", \"tmem_cols\": " + std::to_string(g.tmem_cols) + ", \"smem\": " + std::to_string(g.smem) +
           ", \"path_bf16\": \"" +
           std::string(use_stream(*pp, true) ? "stream" : choose_path(g, ATMM_BF16, true) == BypassPath::kA2a ? "a2a" : (choose_path(g, ATMM_BF16, true) == BypassPath::kSplit ? "split" : "fused")) +
           "\", \"split\": " + (g.split.ok ? std::string("{\"stages\": ") + std::to_string(g.split.stages) +
                                                   ", \"estages_bf16\": " + std::to_string(g.split.estages[0]) +
                                                   ", \"g_bf16\": " + std::to_string(g.split.g_bf16) +
                                                   ", \"rows16\": " + std::to_string(g.split.rows16) +
                                                   ", \"etmem\": [" + std::to_string(g.split.tmem_e[0]) + ", " +
                                                   std::to_string(g.split.tmem_e[1]) + "], \"smem_e\": [" +
                                                   std::to_string(g.split.smem_e[0]) + ", " + std::to_string(g.split.smem_e[1]) + "]}"
                                             : std::string("null")) +
           ", \"a2a_bf16\": " + (g.a2a[0].ok ? std::string("{\"stages\": ") + std::to_string(g.a2a[0].stages) +
                                                  ", \"tmem_cols\": " + std::to_string(g.a2a[0].tmem_cols) +
                                                  ", \"smem\": " + std::to_string(g.a2a[0].smem) + "}"
                                            : std::string("null")) +
           ", \"stream\": " +
           (pp->stream.ok ? std::string("{\"grid\": ") + std::to_string(pp->stream.grid) +
                               ", \"sstages_bf16\": " + std::to_string(pp->stream.sstages[0]) +
                               ", \"estages_bf16\": " + std::to_string(pp->stream.estages[0]) +
                               ", \"smem_bf16\": " + std::to_string(pp->stream.smem[0]) +
                               ", \"tmem_cols\": " + std::to_string(pp->stream.tmem_cols) + "}"
                         : std::string("null")) +
           "}";
      firstg = false;
    }
    }
    s += "]";
    std::strncpy(buf, s.c_str(), cap - 1);
    buf[cap - 1] = 0;
  });
}

int atmm_plan_stats(const atmm_plan* p, int64_t* launches, int64_t* tiles, int64_t* ctas) {
  return guarded([&] {
    if (!p) fail(ATMM_ERR_CONFIG, "null plan");
    int64_t t = 0, nl = 0;
    std::vector<const atmm_plan*> all{p};
    for (const auto& ps : p->passes) all.push_back(ps.get());
    for (const atmm_plan* pp : all) {
      int64_t l = 0;
      for (const auto& g : pp->groups) {
        t += g.num_tiles;
        l += choose_path(g, ATMM_BF16, true) == BypassPath::kSplit ? 0 : 1;  // bf16 Y, aligned
      }
      if (pp->merged_first >= 0) l += 2;  // one shrink + expand pair for all split groups
      if (use_stream(*pp, true)) l = 1;   // one stream launch for the whole plan
      nl += l;
    }
    if (launches) *launches = nl;
    if (tiles) *tiles = t;
    if (ctas) *ctas = p->total_ctas;
  });
}

int atmm_bypass_apply(const atmm_plan* p, int64_t layer, const void* x, int64_t ldx, void* y,
                      int64_t ldy, int y_dtype, float scale, void* stream) {
  return guarded([&] {
    if (!p) fail(ATMM_ERR_CONFIG, "null plan");
    DeviceGuard g(p->reg->device);
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (x && ldx >= p->reg->d_in && (ldx % 8 != 0 || reinterpret_cast<uintptr_t>(x) % 16 != 0)) {
      // Any hidden size / row stride (the reference takes any): X rows that
      // are not 16-byte aligned are staged once into a padded copy (stream
      // ordered, capturable); the kernels then read it by TMA / 16-byte loads.
      const int64_t lds = round_up(p->reg->d_in, 8);
      void* xs = nullptr;
      CUDA_CHECK(cudaMallocAsync(&xs, static_cast<size_t>(std::max<int64_t>(p->n, 1) * lds * 2), st));
      CUDA_CHECK(cudaMemsetAsync(xs, 0, static_cast<size_t>(std::max<int64_t>(p->n, 1) * lds * 2), st));
      CUDA_CHECK(cudaMemcpy2DAsync(xs, lds * 2, x, ldx * 2, p->reg->d_in * 2, p->n, cudaMemcpyDeviceToDevice, st));
      pdl_note_other(st);
      apply_plan(p, layer, xs, lds, y, ldy, y_dtype, scale, st);
      CUDA_CHECK(cudaFreeAsync(xs, st));
    } else {
      apply_plan(p, layer, x, ldx, y, ldy, y_dtype, scale, st);
    }
    flops_add(p->flops);
  });
}

int atmm_bypass_apply_group(const atmm_plan* p, int64_t count, const int64_t* layers, const void* const* xs,
                            int64_t ldx, void* const* ys, int64_t ldy, int y_dtype, float scale, void* stream) {
  return guarded([&] {
    if (!p) fail(ATMM_ERR_CONFIG, "null plan");
    if (count < 1 || count > kMaxGroup || !layers || !xs || !ys) fail(ATMM_ERR_CONFIG, "grouped apply: 1..8 calls");
    DeviceGuard g(p->reg->device);
    apply_plan(p, layers[0], xs[0], ldx, ys[0], ldy, y_dtype, scale, static_cast<cudaStream_t>(stream),
               static_cast<int>(count), layers, xs, ys);
    flops_add(p->flops * static_cast<uint64_t>(count));
  });
}

}  // extern "C"

// run_bypass's host-buffer entry (batch.hpp:48, the reference-signature shim
// calls it once per layer): plans are cached per thread (registry uid and
// generation, table, assignment; LRU of 8) and the device buffers are
// grow-only per thread, so a steady serving loop allocates nothing and
// rebuilds no routing tables.
namespace {
struct HostBypassCache {
  struct Entry {
    uint64_t uid = 0, gen = 0;
    const void* table = nullptr;
    std::vector<int32_t> asg;
    std::unique_ptr<atmm_plan> plan;
    uint64_t used = 0;
  };
  std::vector<Entry> e;
  uint64_t tick = 0;
  int dev = -1;
  DevBuf<float> xf, y;
  DevBuf<uint16_t> xb;
  template <typename T>
  static T* grow(DevBuf<T>& b, size_t n) {
    if (b.n < n) b.alloc(n);
    return b.p;
  }
  atmm_plan* get(atmm_registry* r, const int32_t* asg, int64_t n, const TilingTable* t) {
    if (dev != r->device) {  // buffers and plans belong to one device
      e.clear();
      xf.release();
      y.release();
      xb.release();
      dev = r->device;
    }
    for (Entry& en : e) {
      if (en.uid == r->uid && en.gen == r->generation && en.table == t && int64_t(en.asg.size()) == n &&
          std::equal(en.asg.begin(), en.asg.end(), asg)) {
        en.used = ++tick;
        return en.plan.get();
      }
    }
    Entry en;
    en.uid = r->uid;
    en.gen = r->generation;
    en.table = t;
    en.asg.assign(asg, asg + n);
    en.plan = build_plan(r, asg, n, t, nullptr);
    en.used = ++tick;
    if (e.size() >= 8) {
      auto lru = std::min_element(e.begin(), e.end(), [](const Entry& a, const Entry& b) { return a.used < b.used; });
      *lru = std::move(en);
      return lru->plan.get();
    }
    e.push_back(std::move(en));
    return e.back().plan.get();
  }
};
thread_local HostBypassCache g_host_bypass;
}  // namespace

extern "C" {

int atmm_run_bypass_host(atmm_registry* r, const float* x, int64_t n, const int32_t* assignment,
                         int64_t layer, const atmm_table* table, float* out) {
  return guarded([&] {
    if (!r || !x || !out) fail(ATMM_ERR_CONFIG, "null registry or buffer");
    DeviceGuard g(r->device);
    const TilingTable* t = table ? &table->t : nullptr;
    HostBypassCache& c = g_host_bypass;
    atmm_plan* plan = c.get(r, assignment, n, t);
    if (r->precise) {  // fp32-faithful: fp32 X / out, split-bf16 tensor-core products
      float* xd = HostBypassCache::grow(c.xf, static_cast<size_t>(n * r->d_in));
      float* yd = HostBypassCache::grow(c.y, static_cast<size_t>(n * r->d_out));
      CUDA_CHECK(cudaMemcpy(xd, x, static_cast<size_t>(n * r->d_in) * 4, cudaMemcpyHostToDevice));
      CUDA_CHECK(cudaMemset(yd, 0, static_cast<size_t>(n * r->d_out) * 4));
      bypass_f32(plan, layer, xd, r->d_in, yd, r->d_out, 1.0f, nullptr);
      CUDA_CHECK(cudaMemcpy(out, yd, static_cast<size_t>(n * r->d_out) * 4, cudaMemcpyDeviceToHost));
      flops_add(plan->flops);
      return;
    }
    const int64_t ldx = round_up(r->d_in, 8), ldy = round_up(r->d_out, 8);
    float* xf = HostBypassCache::grow(c.xf, static_cast<size_t>(n * r->d_in));
    uint16_t* xb = HostBypassCache::grow(c.xb, static_cast<size_t>(n * ldx));
    float* y = HostBypassCache::grow(c.y, static_cast<size_t>(n * ldy));
    CUDA_CHECK(cudaMemcpy(xf, x, static_cast<size_t>(n * r->d_in) * 4, cudaMemcpyHostToDevice));
    if (ldx != r->d_in) CUDA_CHECK(cudaMemset(xb, 0, static_cast<size_t>(n * ldx) * 2));
    CUDA_CHECK(cudaMemset(y, 0, static_cast<size_t>(n * ldy) * 4));
    CUDA_CHECK(launch_f32_to_bf16(xf, xb, n, r->d_in, r->d_in, ldx, nullptr));
    pdl_note_other(nullptr);
    apply_plan(plan, layer, xb, ldx, y, ldy, ATMM_F32, 1.0f, nullptr);
    CUDA_CHECK(cudaMemcpy2D(out, r->d_out * 4, y, ldy * 4, r->d_out * 4, n, cudaMemcpyDeviceToHost));
    flops_add(plan->flops);
  });
}

int atmm_bypass_residual_host_bf16(const atmm_plan* p, int64_t layer, const uint16_t* x_host,
                                   uint16_t* y_host, float scale, void* stream) {
  return guarded([&] {
    if (!p || !x_host || !y_host) fail(ATMM_ERR_CONFIG, "null plan or buffer");
    const atmm_registry* r = p->reg;
    DeviceGuard g(r->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // Device staging owned by the plan's registry device; sized per call.
    thread_local DevBuf<uint16_t> xs, ys;
    thread_local int dev_of_bufs = -1;
    const int64_t ldx = round_up(r->d_in, 8), ldy = round_up(r->d_out, 8);
    const size_t nx = static_cast<size_t>(p->n * ldx), ny = static_cast<size_t>(p->n * ldy);
    if (dev_of_bufs != r->device || xs.n < nx) xs.alloc(nx);
    if (dev_of_bufs != r->device || ys.n < ny) ys.alloc(ny);
    dev_of_bufs = r->device;
    CUDA_CHECK(cudaMemcpy2DAsync(xs.p, ldx * 2, x_host, r->d_in * 2, r->d_in * 2, p->n, cudaMemcpyHostToDevice, s));
    CUDA_CHECK(cudaMemcpy2DAsync(ys.p, ldy * 2, y_host, r->d_out * 2, r->d_out * 2, p->n, cudaMemcpyHostToDevice, s));
    apply_plan(p, layer, xs.p, ldx, ys.p, ldy, ATMM_BF16, scale, s);
    CUDA_CHECK(cudaMemcpy2DAsync(y_host, r->d_out * 2, ys.p, ldy * 2, r->d_out * 2, p->n, cudaMemcpyDeviceToHost, s));
    CUDA_CHECK(cudaStreamSynchronize(s));
    flops_add(p->flops);
  });
}

}  // extern "C"

// Host-buffer pipelines (atmm_run_bypass_host_bf16_pipelined,
// atmm_bypass_residual_host_bf16_pipelined): one H2D stream, one compute
// stream, one D2H stream per thread and device, kSlots device buffer pairs,
// events between them.  Each copy engine direction sees one FIFO of copies
// that never waits behind the other direction or a kernel of another batch
// (measured cfg2: 112 vs 124 us per batch with four streams each running
// H2D -> kernel -> D2H; raw duplex copies alone 101 us).
struct HostPipe {
  static constexpr int kSlots = 4;
  cudaStream_t s_in = nullptr, s_c = nullptr, s_out = nullptr;
  DevBuf<uint16_t> x[kSlots], y[kSlots];
  cudaEvent_t ev_in[kSlots] = {}, ev_c[kSlots] = {}, ev_out[kSlots] = {};
  HostPipe() {
    CUDA_CHECK(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
    CUDA_CHECK(cudaStreamCreateWithFlags(&s_c, cudaStreamNonBlocking));
    CUDA_CHECK(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));
    for (int k = 0; k < kSlots; ++k) {
      CUDA_CHECK(cudaEventCreateWithFlags(&ev_in[k], cudaEventDisableTiming));
      CUDA_CHECK(cudaEventCreateWithFlags(&ev_c[k], cudaEventDisableTiming));
      CUDA_CHECK(cudaEventCreateWithFlags(&ev_out[k], cudaEventDisableTiming));
    }
  }
  ~HostPipe() {  // errors ignored: may run after the context is gone (thread / process exit)
    for (int k = 0; k < kSlots; ++k) {
      cudaEventDestroy(ev_in[k]);
      cudaEventDestroy(ev_c[k]);
      cudaEventDestroy(ev_out[k]);
    }
    cudaStreamDestroy(s_in);
    cudaStreamDestroy(s_c);
    cudaStreamDestroy(s_out);
  }
  HostPipe(const HostPipe&) = delete;
  HostPipe& operator=(const HostPipe&) = delete;
  void sync() {
    CUDA_CHECK(cudaStreamSynchronize(s_in));
    CUDA_CHECK(cudaStreamSynchronize(s_c));
    CUDA_CHECK(cudaStreamSynchronize(s_out));
  }
};

// The calling thread's pipeline on `dev` (the current device), buffers grown
// to nx / ny elements.  The previous call on this thread synchronised all
// three streams, so slots carry no hazard into the next call.
static HostPipe& host_pipe(int dev, size_t nx, size_t ny) {
  thread_local std::vector<std::pair<int, std::unique_ptr<HostPipe>>> pipes;
  HostPipe* hp = nullptr;
  for (auto& [d, q] : pipes) {
    if (d == dev) hp = q.get();
  }
  if (!hp) {
    pipes.emplace_back(dev, std::make_unique<HostPipe>());
    hp = pipes.back().second.get();
  }
  for (int k = 0; k < HostPipe::kSlots; ++k) {
    if (hp->x[k].n < nx) hp->x[k].alloc(nx);
    if (hp->y[k].n < ny) hp->y[k].alloc(ny);
  }
  return *hp;
}

extern "C" {

int atmm_bypass_residual_host_bf16_pipelined(const atmm_plan* p, const int64_t* layers,
                                             const uint16_t* const* x_hosts, uint16_t* const* y_hosts,
                                             int64_t count, float scale) {
  return guarded([&] {
    if (!p || !layers || !x_hosts || !y_hosts || count < 0) fail(ATMM_ERR_CONFIG, "null plan or buffers");
    const atmm_registry* r = p->reg;
    DeviceGuard g(r->device);
    const int64_t ldx = round_up(r->d_in, 8), ldy = round_up(r->d_out, 8);
    HostPipe& hp = host_pipe(r->device, static_cast<size_t>(p->n * ldx), static_cast<size_t>(p->n * ldy));
    for (int64_t i = 0; i < count; ++i) {
      const int k = static_cast<int>(i % HostPipe::kSlots);
      if (i >= HostPipe::kSlots) {  // slot k's buffers: the kernel and the D2H of batch i - kSlots are done
        CUDA_CHECK(cudaStreamWaitEvent(hp.s_in, hp.ev_c[k], 0));
        CUDA_CHECK(cudaStreamWaitEvent(hp.s_in, hp.ev_out[k], 0));
      }
      CUDA_CHECK(cudaMemcpy2DAsync(hp.x[k].p, ldx * 2, x_hosts[i], r->d_in * 2, r->d_in * 2, p->n, cudaMemcpyHostToDevice, hp.s_in));
      CUDA_CHECK(cudaMemcpy2DAsync(hp.y[k].p, ldy * 2, y_hosts[i], r->d_out * 2, r->d_out * 2, p->n, cudaMemcpyHostToDevice, hp.s_in));
      CUDA_CHECK(cudaEventRecord(hp.ev_in[k], hp.s_in));
      CUDA_CHECK(cudaStreamWaitEvent(hp.s_c, hp.ev_in[k], 0));
      apply_plan(p, layers[i], hp.x[k].p, ldx, hp.y[k].p, ldy, ATMM_BF16, scale, hp.s_c);
      CUDA_CHECK(cudaEventRecord(hp.ev_c[k], hp.s_c));
      CUDA_CHECK(cudaStreamWaitEvent(hp.s_out, hp.ev_c[k], 0));
      CUDA_CHECK(cudaMemcpy2DAsync(y_hosts[i], r->d_out * 2, hp.y[k].p, ldy * 2, r->d_out * 2, p->n, cudaMemcpyDeviceToHost, hp.s_out));
      CUDA_CHECK(cudaEventRecord(hp.ev_out[k], hp.s_out));
    }
    hp.sync();
    flops_add(p->flops * static_cast<uint64_t>(count));
  });
}

int atmm_run_bypass_host_bf16_pipelined(const atmm_plan* p, const int64_t* layers, const uint16_t* const* x_hosts,
                                        uint16_t* const* out_hosts, int64_t count) {
  return guarded([&] {
    if (!p || !layers || !x_hosts || !out_hosts || count < 0) fail(ATMM_ERR_CONFIG, "null plan or buffers");
    const atmm_registry* r = p->reg;
    DeviceGuard g(r->device);
    const int64_t ldx = round_up(r->d_in, 8), ldy = round_up(r->d_out, 8);
    const size_t nx = static_cast<size_t>(p->n * ldx), ny = static_cast<size_t>(p->n * ldy);
    HostPipe& hp = host_pipe(r->device, nx, ny);
    for (int64_t i = 0; i < count; ++i) {
      const int k = static_cast<int>(i % HostPipe::kSlots);
      // H2D stream: X of batch i into slot k once the kernel of i - kSlots read it
      if (i >= HostPipe::kSlots) CUDA_CHECK(cudaStreamWaitEvent(hp.s_in, hp.ev_c[k], 0));
      if (ldx == r->d_in) {
        CUDA_CHECK(cudaMemcpyAsync(hp.x[k].p, x_hosts[i], nx * 2, cudaMemcpyHostToDevice, hp.s_in));
      } else {
        CUDA_CHECK(cudaMemcpy2DAsync(hp.x[k].p, ldx * 2, x_hosts[i], r->d_in * 2, r->d_in * 2, p->n, cudaMemcpyHostToDevice, hp.s_in));
      }
      CUDA_CHECK(cudaEventRecord(hp.ev_in[k], hp.s_in));
      // compute stream: the bypass into a fresh output once X landed and the
      // D2H of i - kSlots released the output slot
      CUDA_CHECK(cudaStreamWaitEvent(hp.s_c, hp.ev_in[k], 0));
      if (i >= HostPipe::kSlots) CUDA_CHECK(cudaStreamWaitEvent(hp.s_c, hp.ev_out[k], 0));
      CUDA_CHECK(cudaMemsetAsync(hp.y[k].p, 0, ny * 2, hp.s_c));  // fresh output: out = 0 + bypass
      apply_plan(p, layers[i], hp.x[k].p, ldx, hp.y[k].p, ldy, ATMM_BF16, 1.0f, hp.s_c);
      CUDA_CHECK(cudaEventRecord(hp.ev_c[k], hp.s_c));
      // D2H stream
      CUDA_CHECK(cudaStreamWaitEvent(hp.s_out, hp.ev_c[k], 0));
      if (ldy == r->d_out) {
        CUDA_CHECK(cudaMemcpyAsync(out_hosts[i], hp.y[k].p, ny * 2, cudaMemcpyDeviceToHost, hp.s_out));
      } else {
        CUDA_CHECK(cudaMemcpy2DAsync(out_hosts[i], r->d_out * 2, hp.y[k].p, ldy * 2, r->d_out * 2, p->n, cudaMemcpyDeviceToHost, hp.s_out));
      }
      CUDA_CHECK(cudaEventRecord(hp.ev_out[k], hp.s_out));
    }
    hp.sync();
    flops_add(p->flops * static_cast<uint64_t>(count));
  });
}

int atmm_merge_apply(atmm_registry* r, int32_t adapter_id, int64_t layer, void* w, int64_t ldw,
                     int w_dtype, float sign, void* stream) {
  return guarded([&] {
    if (!r || !w) fail(ATMM_ERR_CONFIG, "null registry or W");
    if (layer < 0 || layer >= r->L) {
      fail(ATMM_ERR_CONFIG, "layer index " + std::to_string(layer) + " out of range (L=" + std::to_string(r->L) + ")");
    }
    if (w_dtype != ATMM_BF16 && w_dtype != ATMM_F32) fail(ATMM_ERR_CONFIG, "w_dtype must be ATMM_BF16 or ATMM_F32");
    const int64_t wsz = w_dtype == ATMM_BF16 ? 2 : 4;
    if (ldw < r->d_out) fail(ATMM_ERR_SHAPE, "W row stride ldw must be >= d_out");
    if (reinterpret_cast<uintptr_t>(w) % wsz != 0) fail(ATMM_ERR_SHAPE, "W is not element aligned");
    DeviceGuard g(r->device);
    for (int c = 0; c < r->num_chunks(adapter_id); ++c) {  // rank-chunked adapters: one update per chunk
      const Slot& s = r->chunk(adapter_id, c);
      run_merge(s.down_t + layer * r->d_in_pad * s.r_pad, s.up_t + layer * r->d_out_pad * s.r_pad, r->d_in,
                r->d_out, s.r_pad, w, ldw, w_dtype, sign * s.scale, 1.0f, static_cast<cudaStream_t>(stream));
      flops_add(2ull * static_cast<uint64_t>(r->d_in * r->d_out * s.alg_rank));  // delta_w_into (model.hpp:124)
    }
  });
}

int atmm_merge_apply_layers(atmm_registry* r, int32_t adapter_id, int64_t layer0, int64_t num_layers, void* w,
                            int64_t ldw, int64_t w_layer_stride, int w_dtype, float sign, void* stream) {
  return guarded([&] {
    if (!r || !w) fail(ATMM_ERR_CONFIG, "null registry or W");
    if (num_layers < 1 || layer0 < 0 || layer0 + num_layers > r->L) {
      fail(ATMM_ERR_CONFIG, "layer range [" + std::to_string(layer0) + ", " + std::to_string(layer0 + num_layers) +
                                ") out of range (L=" + std::to_string(r->L) + ")");
    }
    if (w_dtype != ATMM_BF16 && w_dtype != ATMM_F32) fail(ATMM_ERR_CONFIG, "w_dtype must be ATMM_BF16 or ATMM_F32");
    const int64_t wsz = w_dtype == ATMM_BF16 ? 2 : 4;
    if (ldw < r->d_out) fail(ATMM_ERR_SHAPE, "W row stride ldw must be >= d_out");
    if (num_layers > 1 && w_layer_stride < ldw * r->d_in) fail(ATMM_ERR_SHAPE, "W layer stride must be >= ldw * d_in");
    if (reinterpret_cast<uintptr_t>(w) % wsz != 0) fail(ATMM_ERR_SHAPE, "W is not element aligned");
    DeviceGuard g(r->device);
    for (int c = 0; c < r->num_chunks(adapter_id); ++c) {  // rank-chunked adapters: one update per chunk
      const Slot& s = r->chunk(adapter_id, c);
      run_merge(s.down_t + layer0 * r->d_in_pad * s.r_pad, s.up_t + layer0 * r->d_out_pad * s.r_pad, r->d_in,
                r->d_out, s.r_pad, w, ldw, w_dtype, sign * s.scale, 1.0f, static_cast<cudaStream_t>(stream), num_layers,
                r->d_in_pad * s.r_pad, r->d_out_pad * s.r_pad, w_layer_stride);
      flops_add(2ull * static_cast<uint64_t>(num_layers * r->d_in * r->d_out * s.alg_rank));
    }
  });
}

}  // extern "C"

// ModelState (model.hpp:104-112) bound to the device weights of one model:
// which adapter is folded into W, the inference mode, and the weight binding
// (every layer of W is rewritten in ONE merge launch).
struct atmm_model_state {
  atmm_registry* reg = nullptr;
  void* w = nullptr;
  int64_t ldw = 0, w_layer_stride = 0;
  int w_dtype = ATMM_BF16;
  int mode = ATMM_MODE_UNMERGED;
  int32_t merged_adapter = -1;
  int64_t weight_writes = 0;  // merge/unmerge launches issued so far
};

namespace atmm {
namespace {
const char* mode_name(int m) {
  return m == ATMM_MODE_UNMERGED ? "unmerged" : (m == ATMM_MODE_MERGED ? "merged" : "mixture");
}
// One-shot all-layer W +-= s.down.up for the state's weights.
void state_merge_launch(atmm_model_state* st, int32_t adapter_id, float sign, cudaStream_t stream) {
  // fp32 weights of a precise registry take the fp32-faithful merge
  const int rc = st->reg->precise && st->w_dtype == ATMM_F32
                     ? atmm_merge_apply_f32(st->reg, adapter_id, 0, st->reg->L, static_cast<float*>(st->w), st->ldw,
                                            st->w_layer_stride, sign, stream)
                     : atmm_merge_apply_layers(st->reg, adapter_id, 0, st->reg->L, st->w, st->ldw, st->w_layer_stride,
                                               st->w_dtype, sign, stream);
  if (rc != ATMM_OK) fail(rc, atmm_last_error());
  ++st->weight_writes;
}
// merge (model.hpp:144-165): requires the unmerged state.
void state_merge(atmm_model_state* st, int32_t adapter_id, cudaStream_t stream) {
  if (st->mode != ATMM_MODE_UNMERGED) {
    fail(ATMM_ERR_MODE, std::string("merge requires unmerged state (currently ") + mode_name(st->mode) + ")");
  }
  state_merge_launch(st, adapter_id, +1.0f, stream);
  st->mode = ATMM_MODE_MERGED;
  st->merged_adapter = adapter_id;
}
// unmerge (model.hpp:167-188): requires merged / mixture state of this adapter.
void state_unmerge(atmm_model_state* st, int32_t adapter_id, cudaStream_t stream) {
  if (st->mode == ATMM_MODE_UNMERGED) fail(ATMM_ERR_MODE, "unmerge requires merged or mixture state");
  if (st->merged_adapter != adapter_id) {
    fail(ATMM_ERR_MODE, "unmerge of adapter " + std::to_string(adapter_id) + " but adapter " +
                            std::to_string(st->merged_adapter) + " is merged");
  }
  state_merge_launch(st, adapter_id, -1.0f, stream);
  st->mode = ATMM_MODE_UNMERGED;
  st->merged_adapter = -1;
}
}  // namespace
}  // namespace atmm

extern "C" {

int atmm_state_create(atmm_registry* r, void* w, int64_t ldw, int64_t w_layer_stride, int w_dtype,
                      atmm_model_state** out) {
  return guarded([&] {
    if (!r || !w || !out) fail(ATMM_ERR_CONFIG, "null registry, W or output");
    if (w_dtype != ATMM_BF16 && w_dtype != ATMM_F32) fail(ATMM_ERR_CONFIG, "w_dtype must be ATMM_BF16 or ATMM_F32");
    if (ldw < r->d_out) fail(ATMM_ERR_SHAPE, "W row stride ldw must be >= d_out");
    if (r->L > 1 && w_layer_stride < ldw * r->d_in) fail(ATMM_ERR_SHAPE, "W layer stride must be >= ldw * d_in");
    auto st = std::make_unique<atmm_model_state>();
    st->reg = r;
    st->w = w;
    st->ldw = ldw;
    st->w_layer_stride = r->L > 1 ? w_layer_stride : ldw * r->d_in;
    st->w_dtype = w_dtype;
    *out = st.release();
  });
}

void atmm_state_destroy(atmm_model_state* st) { delete st; }

int atmm_state_get(const atmm_model_state* st, int* mode, int32_t* merged_adapter, int64_t* weight_writes) {
  return guarded([&] {
    if (!st) fail(ATMM_ERR_CONFIG, "null state");
    if (mode) *mode = st->mode;
    if (merged_adapter) *merged_adapter = st->merged_adapter;
    if (weight_writes) *weight_writes = st->weight_writes;
  });
}

int atmm_state_merge(atmm_model_state* st, int32_t adapter_id, void* stream) {
  return guarded([&] {
    if (!st) fail(ATMM_ERR_CONFIG, "null state");
    state_merge(st, adapter_id, static_cast<cudaStream_t>(stream));
  });
}

int atmm_state_unmerge(atmm_model_state* st, int32_t adapter_id, void* stream) {
  return guarded([&] {
    if (!st) fail(ATMM_ERR_CONFIG, "null state");
    state_unmerge(st, adapter_id, static_cast<cudaStream_t>(stream));
  });
}

int atmm_state_set_mixture(atmm_model_state* st, int32_t adapter_id) {
  return guarded([&] {
    if (!st) fail(ATMM_ERR_CONFIG, "null state");
    // init_delora (serving.hpp:24-33): the subtraction branch is the merged adapter
    if (st->mode == ATMM_MODE_UNMERGED) fail(ATMM_ERR_MODE, "mixture requires a merged adapter");
    if (st->merged_adapter != adapter_id) {
      fail(ATMM_ERR_MODE, "delora branch must be the merged adapter " + std::to_string(st->merged_adapter));
    }
    if (!atmm_registry_contains(st->reg, adapter_id)) {
      fail(ATMM_ERR_MODE, "mixture integrity: subtraction branch missing");
    }
    st->mode = ATMM_MODE_MIXTURE;
  });
}

int atmm_state_mode_switch(atmm_model_state* st, int to_mode, int32_t target_adapter, void* stream,
                           int64_t* launches) {
  return guarded([&] {
    if (!st) fail(ATMM_ERR_CONFIG, "null state");
    if (to_mode != ATMM_MODE_UNMERGED && to_mode != ATMM_MODE_MERGED && to_mode != ATMM_MODE_MIXTURE) {
      fail(ATMM_ERR_CONFIG, "unknown inference mode");
    }
    const auto s = static_cast<cudaStream_t>(stream);
    const int64_t before = st->weight_writes;
    if (to_mode == ATMM_MODE_UNMERGED) {
      if (st->mode != ATMM_MODE_UNMERGED) state_unmerge(st, st->merged_adapter, s);
    } else {
      if (target_adapter < 0) fail(ATMM_ERR_MODE, "merged/mixture transition needs a target adapter");
      if (!atmm_registry_contains(st->reg, target_adapter)) {
        fail(ATMM_ERR_UNKNOWN_ADAPTER, "unknown adapter id " + std::to_string(target_adapter));
      }
      if (st->mode != ATMM_MODE_UNMERGED && st->merged_adapter != target_adapter) {
        state_unmerge(st, st->merged_adapter, s);
      }
      if (st->mode == ATMM_MODE_UNMERGED) state_merge(st, target_adapter, s);
      st->mode = to_mode;  // merged <-> mixture of the same adapter touches no weights
    }
    if (launches) *launches = st->weight_writes - before;
  });
}

int atmm_delta_w_host(atmm_registry* r, int32_t adapter_id, int64_t layer, float* out) {
  return guarded([&] {
    if (!r || !out) fail(ATMM_ERR_CONFIG, "null registry or output");
    if (layer < 0 || layer >= r->L) {
      fail(ATMM_ERR_CONFIG, "layer index " + std::to_string(layer) + " out of range (L=" + std::to_string(r->L) + ")");
    }
    const Slot& s = r->at(adapter_id);
    DeviceGuard g(r->device);
    if (r->precise) {
      DevBuf<float> wd(static_cast<size_t>(r->d_in * r->d_out));
      const int rc = atmm_delta_w_f32(r, adapter_id, layer, wd.p, r->d_out, nullptr);
      if (rc != ATMM_OK) fail(rc, atmm_last_error());
      CUDA_CHECK(cudaMemcpy(out, wd.p, wd.n * 4, cudaMemcpyDeviceToHost));
      return;
    }
    const int64_t ldw = round_up(r->d_out, 8);
    DevBuf<float> w(static_cast<size_t>(r->d_in * ldw));
    for (int c = 0; c < r->num_chunks(adapter_id); ++c) {  // sum of the chunks' products (fp32)
      const Slot& sc = r->chunk(adapter_id, c);
      run_merge(sc.down_t + layer * r->d_in_pad * sc.r_pad, sc.up_t + layer * r->d_out_pad * sc.r_pad, r->d_in,
                r->d_out, sc.r_pad, w.p, ldw, ATMM_F32, sc.scale, c == 0 ? 0.0f : 1.0f, nullptr);
      flops_add(2ull * static_cast<uint64_t>(r->d_in * r->d_out * sc.alg_rank));
    }
    (void)s;
    CUDA_CHECK(cudaMemcpy2D(out, r->d_out * 4, w.p, ldw * 4, r->d_out * 4, r->d_in, cudaMemcpyDeviceToHost));
  });
}

int atmm_multiply_host(const float* a, int64_t m, int64_t k, const float* b, int64_t n, float* c,
                       const int32_t cfg[6]) {
  return guarded([&] {
    if (!cfg) fail(ATMM_ERR_CONFIG, "null config");
    TilingConfig tc;
    std::copy(cfg, cfg + 6, tc.e.begin());
    if (m < 1 || k < 1 || n < 1) fail(ATMM_ERR_SHAPE, "atmm_multiply: matrix dimensions must be >= 1");
    if (!tc.structurally_valid()) fail(ATMM_ERR_CONFIG, "invalid tiling config " + tc.str());
    if (!a || !b || !c) fail(ATMM_ERR_SHAPE, "null operand");
    int dev = 0;
    cudaGetDevice(&dev);
    require_device(dev);
    // The reference's fp32 GEMM (atmm.hpp:111-142) kept fp32-faithful on the
    // tensor cores: one split-bf16 tcgen05 product (atmm_gemm_f32).  The
    // config is validated like the reference's; the B200 tiles are the GEMM's.
    DevBuf<float> ad(static_cast<size_t>(m * k)), bd(static_cast<size_t>(k * n)), cd(static_cast<size_t>(m * n));
    CUDA_CHECK(cudaMemcpy(ad.p, a, ad.n * 4, cudaMemcpyHostToDevice));
    CUDA_CHECK(cudaMemcpy(bd.p, b, bd.n * 4, cudaMemcpyHostToDevice));
    const int rc = atmm_gemm_f32(ad.p, k, bd.p, n, cd.p, n, m, k, n, 0.0f, nullptr);
    if (rc != ATMM_OK) fail(rc, atmm_last_error());
    CUDA_CHECK(cudaMemcpy(c, cd.p, cd.n * 4, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"

// =========================================================================
// Offline tiling search on B200 (atmm.hpp:188-355): benchmark_config,
// grid_bench_ns, tiling_search, default_shape_grid, re-read for the fused
// bypass.  A tuning shape is a batch of `segments` segments of `m` rows, each
// its own adapter of rank `rank`, rows shuffled; a candidate is a B200 launch
// {tile_m, cluster, bn, stages, path} forced for every segment.
// =========================================================================
namespace atmm {
namespace {

struct TuneBench {
  int device = 0;
  atmm_tune_shape shape{};
  std::unique_ptr<atmm_registry> reg;
  std::vector<int32_t> assignment;
  int64_t ldx = 0, ldy = 0;
  static constexpr int kSets = 4;  // applies per trial, each on its own X / Y (cold after the L2 flush)
  DevBuf<uint16_t> x[kSets], y[kSets];
  DevBuf<uint8_t> flush;
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;

  TuneBench(int dev, const atmm_tune_shape& sh, uint64_t seed) : device(dev), shape(sh) {
    if (sh.m < 1 || sh.d_in < 1 || sh.d_out < 1 || sh.rank < 1 || sh.segments < 1) {
      fail(ATMM_ERR_SHAPE, "tuning shape dimensions must be >= 1");
    }
    reg.reset(new atmm_registry());
    reg->device = dev;
    reg->L = 1;
    reg->d_in = sh.d_in;
    reg->d_out = sh.d_out;
    reg->d_in_pad = round_up(sh.d_in, 128);
    reg->d_out_pad = round_up(sh.d_out, 128);
    // Synthetic factors: values do not change the timing.
    std::vector<float> dn(static_cast<size_t>(sh.d_in * sh.rank)), up(static_cast<size_t>(sh.rank * sh.d_out));
    for (size_t i = 0; i < dn.size(); ++i) dn[i] = 0.001f * static_cast<float>((i * 7919) % 61) - 0.03f;
    for (size_t i = 0; i < up.size(); ++i) up[i] = 0.001f * static_cast<float>((i * 104729) % 53) - 0.026f;
    for (int64_t a = 0; a < sh.segments; ++a) {
      const int st = atmm_registry_put(reg.get(), static_cast<int32_t>(a), sh.rank, dn.data(), up.data(), 1.0f);
      if (st != ATMM_OK) fail(st, atmm_last_error());
    }
    const int64_t n = sh.m * sh.segments;
    assignment.resize(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) assignment[static_cast<size_t>(i)] = static_cast<int32_t>(i / sh.m);
    uint64_t st = seed | 1;  // xorshift Fisher-Yates: the rows of a segment are scattered
    for (int64_t i = n - 1; i > 0; --i) {
      st ^= st << 13;
      st ^= st >> 7;
      st ^= st << 17;
      std::swap(assignment[static_cast<size_t>(i)], assignment[static_cast<size_t>(st % static_cast<uint64_t>(i + 1))]);
    }
    ldx = round_up(sh.d_in, 8);
    ldy = round_up(sh.d_out, 8);
    for (int k = 0; k < kSets; ++k) {
      x[k].alloc(static_cast<size_t>(n * ldx));
      y[k].alloc(static_cast<size_t>(n * ldy));
      CUDA_CHECK(cudaMemset(x[k].p, 0, x[k].n * 2));
      CUDA_CHECK(cudaMemset(y[k].p, 0, y[k].n * 2));
    }
    flush.alloc(size_t(256) << 20);  // > 2x the 126 MB L2
    CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CUDA_CHECK(cudaEventCreate(&e0));
    CUDA_CHECK(cudaEventCreate(&e1));
  }
  ~TuneBench() {
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (s) cudaStreamDestroy(s);
  }

  // benchmark_config (atmm.hpp:188-216): median of `trials` after one
  // warm-up; each trial flushes L2, then times kSets back-to-back applies
  // (bf16 Y, each on its own buffers) with CUDA events on the launch stream
  // and records the per-apply time.
  int64_t median_ns(const LaunchCfg& lc, int trials) {
    auto plan = build_plan(reg.get(), assignment.data(), static_cast<int64_t>(assignment.size()), nullptr, &lc);
    std::vector<int64_t> samples;
    for (int t = 0; t < trials + 1; ++t) {
      CUDA_CHECK(cudaMemsetAsync(flush.p, t & 0xff, flush.n, s));
      CUDA_CHECK(cudaEventRecord(e0, s));
      for (int k = 0; k < kSets; ++k) apply_plan(plan.get(), 0, x[k].p, ldx, y[k].p, ldy, ATMM_BF16, 1.0f, s);
      CUDA_CHECK(cudaEventRecord(e1, s));
      CUDA_CHECK(cudaEventSynchronize(e1));
      float ms = 0.f;
      CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
      if (t > 0) samples.push_back(static_cast<int64_t>(static_cast<double>(ms) * 1e6 / kSets));
    }
    std::sort(samples.begin(), samples.end());
    return samples[samples.size() / 2];
  }
};

std::string shape_str(const atmm_tune_shape& s) {
  return std::to_string(s.segments) + "x" + std::to_string(s.m) + " rows, d " + std::to_string(s.d_in) + "->" +
         std::to_string(s.d_out) + ", r " + std::to_string(s.rank);
}
std::string launch_str(const LaunchCfg& l) {
  return "{" + std::to_string(l.tile_m) + "," + std::to_string(l.cluster) + "," + std::to_string(l.bn) + "," +
         std::to_string(l.stages) + "," + std::to_string(l.path) + "}";
}

// grid_bench_ns (atmm.hpp:229-270): every round sweeps the whole grid before
// any point is sampled again; a point's score is the median of its round
// medians; points that fail score INT64_MAX (reported, never fatal).
std::vector<std::vector<int64_t>> grid_bench(int device, const atmm_tune_shape* shapes, int64_t ns,
                                             const std::vector<LaunchCfg>& cands, int trials, int rounds,
                                             std::vector<std::string>& failures) {
  std::vector<std::vector<std::vector<int64_t>>> samples(static_cast<size_t>(ns),
                                                         std::vector<std::vector<int64_t>>(cands.size()));
  std::vector<std::vector<char>> failed(static_cast<size_t>(ns), std::vector<char>(cands.size(), 0));
  std::vector<std::unique_ptr<TuneBench>> benches(static_cast<size_t>(ns));
  for (int round = 0; round < rounds; ++round) {
    for (int64_t si = 0; si < ns; ++si) {
      auto& b = benches[static_cast<size_t>(si)];
      if (!b) b.reset(new TuneBench(device, shapes[si], 0x5eedbeefull + static_cast<uint64_t>(si)));
      for (size_t ci = 0; ci < cands.size(); ++ci) {
        if (failed[static_cast<size_t>(si)][ci]) continue;
        try {
          samples[static_cast<size_t>(si)][ci].push_back(b->median_ns(cands[ci], trials));
        } catch (const Failure& e) {
          cudaGetLastError();
          failed[static_cast<size_t>(si)][ci] = 1;
          failures.push_back("shape " + shape_str(shapes[si]) + " launch " + launch_str(cands[ci]) + ": " + e.what());
        }
      }
      if (round + 1 == rounds) b.reset();  // bound device memory: one shape's buffers at a time at the end
    }
  }
  std::vector<std::vector<int64_t>> scores(static_cast<size_t>(ns),
                                           std::vector<int64_t>(cands.size(), std::numeric_limits<int64_t>::max()));
  for (int64_t si = 0; si < ns; ++si) {
    for (size_t ci = 0; ci < cands.size(); ++ci) {
      auto& v = samples[static_cast<size_t>(si)][ci];
      if (failed[static_cast<size_t>(si)][ci] || v.empty()) continue;
      std::sort(v.begin(), v.end());
      scores[static_cast<size_t>(si)][ci] = v[v.size() / 2];
    }
  }
  return scores;
}

std::vector<LaunchCfg> launches_from(const int32_t* v, int64_t count) {
  std::vector<LaunchCfg> out;
  for (int64_t i = 0; i < count; ++i) {
    out.push_back(launch_from_ints(v + 5 * i));
    validate_launch(out.back());
  }
  return out;
}

void write_failures(const std::vector<std::string>& f, char* buf, size_t cap) {
  if (!buf || cap == 0) return;
  std::string all;
  for (const auto& s : f) all += s + "\n";
  std::strncpy(buf, all.c_str(), cap - 1);
  buf[cap - 1] = 0;
}

}  // namespace
}  // namespace atmm

extern "C" {

int atmm_benchmark_launch(int device, const atmm_tune_shape* shape, const int32_t launch[5], int trials,
                          uint64_t seed, int64_t* median_ns) {
  return guarded([&] {
    if (!shape || !launch || !median_ns) fail(ATMM_ERR_CONFIG, "null shape, launch or output");
    if (trials < 3) fail(ATMM_ERR_CONFIG, "benchmark_config needs trials >= 3");
    require_device(device);
    DeviceGuard g(device);
    const LaunchCfg lc = launch_from_ints(launch);
    validate_launch(lc);
    TuneBench b(device, *shape, seed);
    *median_ns = b.median_ns(lc, trials);
  });
}

int atmm_grid_bench_ns(int device, const atmm_tune_shape* shapes, int64_t num_shapes, const int32_t* launches,
                       int64_t num_launches, int trials, int rounds, int64_t* scores, char* failures,
                       size_t failures_cap) {
  return guarded([&] {
    if (!shapes || !launches || !scores || num_shapes < 1 || num_launches < 1) {
      fail(ATMM_ERR_CONFIG, "grid_bench needs a nonempty grid and candidates");
    }
    if (trials < 3 || rounds < 1) fail(ATMM_ERR_CONFIG, "grid_bench needs trials >= 3 and rounds >= 1");
    require_device(device);
    DeviceGuard g(device);
    std::vector<std::string> fails;
    const auto cands = launches_from(launches, num_launches);
    const auto sc = grid_bench(device, shapes, num_shapes, cands, trials, rounds, fails);
    for (int64_t si = 0; si < num_shapes; ++si) {
      for (int64_t ci = 0; ci < num_launches; ++ci) {
        scores[si * num_launches + ci] = sc[static_cast<size_t>(si)][static_cast<size_t>(ci)];
      }
    }
    write_failures(fails, failures, failures_cap);
  });
}

int atmm_tiling_search(int device, const atmm_tune_shape* shapes, int64_t num_shapes, const int32_t* launches,
                       int64_t num_launches, int trials, atmm_table** out, char* failures, size_t failures_cap) {
  return guarded([&] {
    if (!out) fail(ATMM_ERR_CONFIG, "null output");
    if (!shapes || !launches || num_shapes < 1 || num_launches < 1) {
      fail(ATMM_ERR_CONFIG, "tiling_search needs a nonempty grid and candidates");
    }
    if (trials < 3) fail(ATMM_ERR_CONFIG, "tiling_search needs trials >= 3");
    require_device(device);
    DeviceGuard g(device);
    std::vector<std::string> fails;
    const auto cands = launches_from(launches, num_launches);
    const auto scores = grid_bench(device, shapes, num_shapes, cands, trials, 3, fails);
    std::vector<int64_t> flat;
    for (const auto& row : scores) flat.insert(flat.end(), row.begin(), row.end());
    std::string sel_fail(failures_cap > 0 ? failures_cap : 1, '\0');
    const int st = atmm_table_from_scores(shapes, num_shapes, launches, num_launches, flat.data(), out,
                                          sel_fail.data(), sel_fail.size());
    if (st != ATMM_OK) fail(st, atmm_last_error());
    if (sel_fail[0]) fails.push_back(sel_fail.c_str());
    write_failures(fails, failures, failures_cap);
  });
}

int atmm_default_shape_grid(int64_t d_in, int64_t d_out, const int64_t* ranks, int64_t num_ranks, atmm_tune_shape* out,
                            int64_t cap, int64_t* count) {
  return guarded([&] {
    if (!count || (num_ranks > 0 && !ranks)) fail(ATMM_ERR_CONFIG, "null argument");
    if (d_in < 1 || d_out < 1) fail(ATMM_ERR_SHAPE, "dimensions must be >= 1");
    static const int64_t kDefaultRanks[] = {8, 16, 32, 64, 128};
    const int64_t* rs = num_ranks > 0 ? ranks : kDefaultRanks;
    const int64_t nr = num_ranks > 0 ? num_ranks : 5;
    // atmm.hpp:341-355 re-read for the bypass: segment rows from single
    // tokens (decode) to whole prompts, each batch ~1-2k tokens of
    // concurrent segments (the serving batch sizes of BASELINE.json).
    static const int64_t kRows[] = {8, 16, 32, 64, 96, 128, 256, 512};
    std::vector<atmm_tune_shape> grid;
    for (int64_t r = 0; r < nr; ++r) {
      for (int64_t m : kRows) {
        const int64_t segs = std::clamp<int64_t>(1024 / m, 4, 64);
        { atmm_tune_shape t; t.m=m; t.d_in=d_in; t.rank=rs[r]; t.d_out=d_out; t.segments=segs; grid.push_back(t); }
      }
    }
    *count = static_cast<int64_t>(grid.size());
    if (out) std::copy(grid.begin(), grid.begin() + std::min<int64_t>(cap, *count), out);
  });
}

int atmm_default_launch_candidates(int32_t* out, int64_t cap, int64_t* count) {
  return guarded([&] {
    if (!count) fail(ATMM_ERR_CONFIG, "null count");
    std::vector<LaunchCfg> c;
    for (int32_t tm : {16, 32, 64, 128}) {
      for (int32_t cl : {4, 8, 16}) {
        c.push_back(LaunchCfg{tm, cl, tm <= 64 ? 128 : 256, 0, 0});
      }
    }
    c.push_back(LaunchCfg{128, 8, 128, 0, 0});
    c.push_back(LaunchCfg{32, 8, 128, 0, ATMM_PATH_SPLIT});
    c.push_back(LaunchCfg{64, 8, 128, 0, ATMM_PATH_A2A});
    c.push_back(LaunchCfg{128, 8, 128, 0, ATMM_PATH_A2A});
    *count = static_cast<int64_t>(c.size());
    if (out) {
      for (int64_t i = 0; i < std::min<int64_t>(cap, *count); ++i) launch_to_ints(c[static_cast<size_t>(i)], out + 5 * i);
    }
  });
}

}  // extern "C"

// =========================================================================
// Layer forward (model.hpp:192-328): cur <- tanh(cur . W_l + bypass_l(cur))
// over L layers; two launches per layer (forward_kernels.cu).
// =========================================================================
struct atmm_forward {
  atmm_registry* reg = nullptr;  // null: forward_merged (no bypass)
  uint64_t generation = 0;
  uint64_t bypass_flops = 0;     // algorithmic FLOPs of one layer's bypass (the plan's)
  int device = 0;
  int64_t n = 0, d = 0;
  bool sorted = false;  // rows run in plan order (gathered in, scattered out)
  int32_t row_tiles = 0, bn = 128, ntn = 0, num_tiles = 0, nkb = 0, ks = 1, num_items = 0, num_ext = 0;
  int32_t stages_g = 0, stages_s = 0, grid = 0, sbytes = 0;
  bool pair = false;  // GEMM as 2-SM CTA pairs (fwd_gemm_pair_kernel)
  int32_t kz = 1;     // 1-SM GEMM split-K cluster
  bool bk2 = false;   // 1-SM GEMM with 128-deep K stages (A as 64-wide atoms)
  int64_t zero_off = 0;
  CUtensorMap amap;            // pair GEMM: the A images, 16 KB slots
  DevBuf<CUtensorMap> umaps;   // pair GEMM: per-slot up^T maps
  DevBuf<int32_t> pext, pext_begin;
  size_t smem_g = 0, smem_s = 0;
  DevBuf<uint16_t> buf[2];
  DevBuf<uint8_t> ext;
  DevBuf<FwdExt> exts;
  DevBuf<int32_t> ext_begin, order;
  DevBuf<FwdItem> items;
  CUtensorMap bmap[2];
  CUtensorMap bmap2[2];  // bk2: the same buffers as 64-wide K atoms (GEMM A operand)
};

namespace atmm {
namespace {
// Activations (rows x d bf16, row stride ld): box = 128 rows x one 64-wide K block, 128-byte swizzle.
CUtensorMap make_act_map(const void* x, int64_t rows, int64_t d, int64_t ld, int box_rows = kTileM) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  const cuuint32_t box[2] = {kBK, static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x), dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(ATMM_ERR_CUDA, "cuTensorMapEncodeTiled(activations) failed: " + std::to_string(r));
  return m;
}
// Layer weights W_l (k x n bf16, [k][n], row stride ldw, layer stride w_ls):
// box = 64 K rows x 64 N columns, 128-byte swizzle = the MN-major B operand.
CUtensorMap make_layer_w_map(const void* w, int64_t k, int64_t n, int64_t ldw, int64_t L, int64_t w_ls,
                             int box_k = kBK) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(L)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(ldw) * 2, static_cast<cuuint64_t>(L > 1 ? w_ls : ldw * k) * 2};
  const cuuint32_t box[3] = {kBK, static_cast<cuuint32_t>(box_k), 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(w), dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(ATMM_ERR_CUDA, "cuTensorMapEncodeTiled(layer W) failed: " + std::to_string(r));
  return m;
}
// Activations as 64-wide K atoms (K % 64 == 0): dims {64, rows, K / 64},
// box {64, 128 rows, 2 atoms} = two 128-byte-swizzled K-major blocks.
CUtensorMap make_act_map_atoms(const void* x, int64_t rows, int64_t k, int64_t ld) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(kBK), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(k / kBK)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 2, static_cast<cuuint64_t>(kBK) * 2};
  const cuuint32_t box[3] = {kBK, kTileM, 2};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(x), dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(ATMM_ERR_CUDA, "cuTensorMapEncodeTiled(activation atoms) failed: " + std::to_string(r));
  return m;
}
void require_aligned16(const void* p, const char* what) {
  if (reinterpret_cast<uintptr_t>(p) % 16 != 0) fail(ATMM_ERR_SHAPE, std::string(what) + " must be 16-byte aligned");
}

// Tile shape of the base GEMM (m rows x n columns, nkb K blocks) on `sms` SMs
// given the 1-SM / 2-SM choice: N tile width, persistent grid, ring depth and
// the 1-SM split-K cluster size.
struct GemmTiling {
  int32_t bn = 128, ntn = 1, num_tiles = 1, stages = 1, grid = 1, kz = 1, mc = 1;
  bool bk2 = false;  // 128-deep K stages (1-SM, bn 128, no split-K / multicast, K % 64 == 0)
  size_t smem = 0;
};
// Tile options of the GEMM / layer forward (atmm_gemm_opts; all zero =
// automatic): the explicit form of what the heuristics below choose, for the
// tile sweeps and the path-coverage tests.
atmm_gemm_opts opts_or_auto(const atmm_gemm_opts* o) {
  atmm_gemm_opts a{};
  a.pair = -1;
  if (!o) return a;
  if (o->pair < -1 || o->pair > 1 || (o->bn != 0 && o->bn != 128 && o->bn != 256) ||
      (o->kz != 0 && o->kz != 1 && o->kz != 2 && o->kz != 4 && o->kz != 8) || o->ks < 0 || o->ks > 16 ||
      (o->mc != 0 && o->mc != 1 && o->mc != 2 && o->mc != 4) || o->stages < 0 || o->stages == 1 || o->stages > 8) {
    fail(ATMM_ERR_CONFIG, "invalid GEMM tile options");
  }
  return *o;
}
// Without a bypass: 2-SM pairs unless one wave of 1-SM 128 x 128 tiles with
// 128-deep K stages covers the GEMM (measured m = 512, n = k = 4096: 19.1 us
// vs 22.9 us for pairs; m = 1024 needs two waves and pairs win, 26 vs 34 us).
bool pair_without_bypass(int64_t m, int64_t n, int64_t k, int sms, const atmm_gemm_opts& o) {
  const int64_t row_tiles = (m + kTileM - 1) / kTileM;
  if (row_tiles < 2) return false;
  if (o.pair >= 0) return o.pair != 0;
  return !(k % kBK == 0 && row_tiles * ((n + 127) / 128) <= sms);
}
GemmTiling gemm_tiling(int64_t m, int64_t n, int64_t k, int sms, bool pair, const atmm_gemm_opts& o,
                       bool allow_mc = false) {
  const int32_t nkb = static_cast<int32_t>((k + kBK - 1) / kBK);
  GemmTiling t;
  const int64_t row_tiles = (m + kTileM - 1) / kTileM;
  const int64_t mtiles = pair ? (row_tiles + 1) / 2 : row_tiles;
  const int64_t units = pair ? sms / 2 : sms;
  // 256-wide N tiles once they alone fill the SMs, or when 128-wide ones
  // would need more waves (measured: m = 1024, n = 4096 pair tiles 41 -> 26 us)
  const int64_t t128 = mtiles * ((n + 127) / 128), t256 = mtiles * ((n + 255) / 256);
  t.bn = t256 >= units || (t128 + units - 1) / units > (t256 + units - 1) / units ? 256 : 128;
  if (o.bn) t.bn = o.bn;
  t.ntn = static_cast<int32_t>((n + t.bn - 1) / t.bn);
  t.num_tiles = static_cast<int32_t>(mtiles) * t.ntn;
  const size_t gstage = 16384 + static_cast<size_t>(pair ? t.bn / 2 : t.bn) * 128;
  t.stages = static_cast<int32_t>(std::min<size_t>(8, (kSmemLimit - 2048) / gstage));
  if (o.stages) t.stages = std::clamp<int32_t>(o.stages, 2, t.stages);
  t.smem = 1024 + t.stages * gstage;
  if (pair) {
    if (k % kBK == 0) {  // 128-deep K stages
      t.bk2 = true;
      const size_t gstage2 = 2 * 16384 + static_cast<size_t>(t.bn / 2) * 256;
      t.stages = static_cast<int32_t>(std::min<size_t>(8, (kSmemLimit - 2048) / gstage2));
      t.smem = 1024 + t.stages * gstage2;
    }
    int clusters = fwd_gemm_pair_max_clusters(t.smem);
    if (clusters <= 0) clusters = sms / 2;
    t.grid = std::min(t.num_tiles, clusters) * 2;
  } else {
    // Split-K for small batches: clusters of kz CTAs per tile while every
    // tile still gets its own cluster on the SMs and each rank >= 8 K blocks.
    if (t.bn == 128) {
      while (t.kz < 8 && int64_t(t.num_tiles) * t.kz * 2 <= sms && nkb / (t.kz * 2) >= 8) t.kz *= 2;
    }
    if (o.kz) t.kz = (o.kz > 1 && t.bn == 128 && nkb / o.kz >= 1) ? o.kz : 1;
    if (t.kz > 1) {
      // the split-K epilogue stages the 128-row fp32 partial and the kz
      // receive slots in the idle ring: 2 x 128 x (bn + 4) x 4 bytes
      const size_t need = 2 * size_t(kTileM) * (t.bn + 4) * 4;
      while (size_t(t.stages) * gstage < need) ++t.stages;
      t.smem = 1024 + t.stages * gstage;
    }
    t.grid = t.kz > 1 ? t.num_tiles * t.kz : std::min(t.num_tiles, sms);
    // A multicast across mc adjacent N tiles (plain GEMM; replaces split-K)
    if (allow_mc) {
      if ((o.mc == 2 || o.mc == 4) && t.ntn % o.mc == 0) t.mc = o.mc;
      if (t.mc > 1) {
        t.kz = 1;
        int clusters = fwd_gemm_max_clusters(t.smem, t.mc);
        if (clusters <= 0) clusters = sms / t.mc;
        t.grid = std::min(t.num_tiles / t.mc, clusters) * t.mc;
      }
    }
    // 128-deep K stages: half the TMA instructions and barrier round trips
    // (measured m = 512, n = k = 4096: 25.2 -> 19.1 us; 256-wide tiles lose,
    // two stages only).
    if (t.mc == 1 && t.bn == 128 && k % kBK == 0 && (k / kBK + 1) / 2 >= t.kz) {
      t.bk2 = true;
      const size_t gstage2 = 2 * 16384 + static_cast<size_t>(t.bn) * 256;
      t.stages = static_cast<int32_t>(std::min<size_t>(8, (kSmemLimit - 2048) / gstage2));
      t.smem = 1024 + t.stages * gstage2;
    }
  }
  return t;
}
}  // namespace
}  // namespace atmm

int atmm_forward_create(const atmm_plan* plan, int device, int64_t n, int64_t hidden_dim, atmm_forward** out) {
  return atmm_forward_create_opts(plan, device, n, hidden_dim, nullptr, out);
}

int atmm_forward_create_opts(const atmm_plan* plan, int device, int64_t n, int64_t hidden_dim,
                             const atmm_gemm_opts* opts, atmm_forward** out) {
  return guarded([&] {
    if (!out) fail(ATMM_ERR_CONFIG, "null output");
    const atmm_gemm_opts o = opts_or_auto(opts);
    auto f = std::make_unique<atmm_forward>();
    if (plan) {
      atmm_registry* reg = plan->reg;
      if (plan->generation != reg->generation) fail(ATMM_ERR_CONFIG, "plan is stale: the registry changed since it was built");
      if (reg->d_in != reg->d_out) fail(ATMM_ERR_SHAPE, "the layer forward needs square layers (d_in == d_out)");
      if (hidden_dim > 0 && hidden_dim != reg->d_in) fail(ATMM_ERR_SHAPE, "hidden_dim does not match the registry");
      if (n > 0 && n != plan->n) fail(ATMM_ERR_SHAPE, "row count does not match the plan");
      if (!plan->passes.empty()) {
        fail(ATMM_ERR_CONFIG, "the fused layer forward takes adapters of rank <= 128 (rank-chunked adapters: "
                              "BypassPlan.apply after the base GEMM)");
      }
      f->reg = reg;
      f->generation = reg->generation;
      f->bypass_flops = plan->flops;
      f->device = reg->device;
      f->n = plan->n;
      f->d = reg->d_in;
    } else {
      f->device = device;
      f->n = n;
      f->d = hidden_dim;
    }
    if (f->n < 1 || f->d < 1) fail(ATMM_ERR_SHAPE, "rows and hidden_dim must be >= 1");
    if (f->d % 8 != 0) fail(ATMM_ERR_SHAPE, "hidden_dim must be a multiple of 8 (16-byte activation rows)");
    if (f->n > std::numeric_limits<int32_t>::max() / 2) fail(ATMM_ERR_SHAPE, "batch too large");
    require_device(f->device);
    DeviceGuard g(f->device);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, f->device);
    const int64_t n_ = f->n, d = f->d;
    f->nkb = static_cast<int32_t>((d + kBK - 1) / kBK);
    f->row_tiles = static_cast<int32_t>((n_ + kTileM - 1) / kTileM);
    // 2-SM CTA pairs (cta_group::2, M = 256) whenever there are two row tiles:
    // each SM then stages half of every W block (without a bypass,
    // atmm_gemm_opts::pair forces either).
    // With a bypass, pairs pay for the union of two row tiles' extension
    // chunks; they are taken when the GEMM is large enough to amortise it
    // (measured: cfg5-sized batches win, cfg2/cfg3-sized ones lose).
    const bool bypass_plan = plan && !plan->bp.seg_adapter.empty();
    const int64_t pair_tiles = int64_t((f->row_tiles + 1) / 2) * ((d + 255) / 256);
    f->pair = bypass_plan ? f->row_tiles >= 2 && pair_tiles >= 2 * sms : pair_without_bypass(n_, d, d, sms, o);
    if (o.pair >= 0) f->pair = f->row_tiles >= 2 && o.pair != 0;
    GemmTiling gt = gemm_tiling(n_, d, d, sms, f->pair, o);
    // With a bypass, the shrink launch (a cluster of up to 16 K slices per
    // item) runs beside the GEMM: a split-K grid that leaves less than two
    // such clusters of SMs free has clusters that only start once the shrink
    // is done and then set the layer's end (tools/fwd_trace.py --graph, cfg1:
    // kz 4 -> 2 measured 20.2 -> 19.2 us per layer).
    if (bypass_plan && !f->pair && o.kz == 0 && gt.kz > 1 && gt.grid + 32 > sms) {
      atmm_gemm_opts o2 = o;
      o2.kz = gt.kz / 2;
      gt = gemm_tiling(n_, d, d, sms, f->pair, o2);
    }
    f->bk2 = gt.bk2;
    f->bn = gt.bn;
    f->ntn = gt.ntn;
    f->num_tiles = gt.num_tiles;
    f->stages_g = gt.stages;
    f->smem_g = gt.smem;
    f->grid = gt.grid;
    f->kz = gt.kz;

    std::vector<int32_t> order;
    std::vector<FwdExt> exts;
    std::vector<int32_t> ext_begin{0};
    std::vector<FwdItem> items;
    std::vector<int64_t> ext_key;  // (segment, chunk) of each ext, for the pair unions
    std::map<const uint16_t*, int32_t> umap_of;
    std::vector<const Slot*> umap_slots;
    if (plan && !plan->bp.seg_adapter.empty()) {
      atmm_registry* reg = plan->reg;
      f->sorted = true;
      order = plan->rows_host;
      std::vector<char> covered(static_cast<size_t>(n_), 0);
      for (int32_t r : order) covered[static_cast<size_t>(r)] = 1;
      for (int64_t r = 0; r < n_; ++r)
        if (!covered[static_cast<size_t>(r)]) order.push_back(static_cast<int32_t>(r));
      const auto& off = plan->bp.seg_offsets;
      const size_t S = plan->bp.seg_adapter.size();
      int64_t a_off = 0;
      for (int32_t t = 0; t < f->row_tiles; ++t) {
        const int64_t t0 = int64_t(t) * kTileM, t1 = std::min<int64_t>(t0 + kTileM, n_);
        const size_t first = exts.size();
        for (size_t s = 0; s < S; ++s) {
          const int64_t b = std::max<int64_t>(off[s], t0), e = std::min<int64_t>(off[s + 1], t1);
          if (e <= b) continue;
          const Slot& sl = reg->at(plan->bp.seg_adapter[s]);
          for (int32_t kc = 0; kc * 32 < sl.r_pad; ++kc) {
            FwdExt x{};
            x.down_t = sl.down_t;
            x.up_t = sl.up_t;
            x.down_ls = reg->d_in_pad * sl.r_pad;
            x.up_ls = reg->d_out_pad * sl.r_pad;
            x.a_off = a_off;
            x.r_pad = static_cast<int32_t>(sl.r_pad);
            x.kc = kc;
            x.kk = static_cast<int32_t>(std::min<int64_t>(32, sl.r_pad - 32 * kc));
            x.lo = static_cast<int32_t>(b - t0);
            x.hi = static_cast<int32_t>(e - t0);
            x.scale = sl.scale;
            a_off += 16384;  // one 16 KB slot per image: 128 rows x [mid_hi | mid_lo] (<= 64 columns)
            auto um = umap_of.find(sl.up_t);
            if (um == umap_of.end()) {
              um = umap_of.emplace(sl.up_t, static_cast<int32_t>(umap_slots.size())).first;
              umap_slots.push_back(&sl);
            }
            x.umap = um->second;
            exts.push_back(x);
            ext_key.push_back(int64_t(s) * 16 + kc);
          }
        }
        // shrink items: consecutive chunks of the tile, <= 64 rank columns each
        // (keeps >= 4 pipeline stages beside the two reduction buffers)
        for (size_t i = first; i < exts.size();) {
          FwdItem it{t, static_cast<int32_t>(i), static_cast<int32_t>(i), 0};
          while (i < exts.size() && it.ncols + exts[i].kk <= 64) {
            exts[i].col = it.ncols;
            it.ncols += exts[i].kk;
            ++i;
          }
          it.e_end = static_cast<int32_t>(i);
          items.push_back(it);
        }
        ext_begin.push_back(static_cast<int32_t>(exts.size()));
      }
      f->num_ext = static_cast<int32_t>(exts.size());
      f->num_items = static_cast<int32_t>(items.size());
      // K split of the shrink: when the GEMM grid leaves room, keep shrink +
      // GEMM co-resident (the GEMM's main loop then hides the shrink, which
      // only gates its final K-extension blocks); otherwise fill the SMs.
      // Otherwise the shrink's CTAs delay the GEMM CTAs that get their SMs
      // last: size it to the CTAs that own one tile fewer (they start late at
      // no cost), with K split 1 when even that does not fit.
      f->ks = 1;
      const int64_t room = sms - f->grid;
      const int64_t units = f->pair ? f->grid / 2 : f->grid;
      const int64_t per = units > 0 ? (f->num_tiles + units - 1) / units : 1;
      const int64_t slack = (units * per - f->num_tiles) * (f->pair ? 2 : 1);
      const int64_t cap = room >= f->num_items ? room : slack;
      while (f->ks < 16 && int64_t(f->num_items) * f->ks * 2 <= cap && f->ks * 2 <= f->nkb) f->ks *= 2;
      if (o.ks) f->ks = o.ks;
      while (f->ks > 1 && f->ks > f->nkb) f->ks /= 2;  // every K slice gets >= 1 K block
      int32_t max_cols = 16;
      for (const FwdItem& it : items) max_cols = std::max(max_cols, it.ncols);
      f->sbytes = max_cols * 128;
      const size_t red = f->ks > 1 ? 2 * size_t(kTileM) * (max_cols + 4) * 4 : 0;  // partial + receive slots
      const size_t sstage = 16384 + static_cast<size_t>(f->sbytes);
      f->stages_s = static_cast<int32_t>(std::min<size_t>(8, (kSmemLimit - 2048 - red) / sstage));  // 1 KiB static
      f->smem_s = 1024 + f->stages_s * sstage + red;
      if (f->pair) {  // per pair: the union of both row tiles' chunks, in (segment, chunk) order
        std::vector<int32_t> pe, pb{0};
        for (int32_t pi = 0; pi < (f->row_tiles + 1) / 2; ++pi) {
          const int32_t t0 = 2 * pi, t1 = 2 * pi + 1;
          int32_t i0 = ext_begin[static_cast<size_t>(t0)], e0 = ext_begin[static_cast<size_t>(t0) + 1];
          int32_t i1 = t1 < f->row_tiles ? ext_begin[static_cast<size_t>(t1)] : 0;
          const int32_t e1 = t1 < f->row_tiles ? ext_begin[static_cast<size_t>(t1) + 1] : 0;
          while (i0 < e0 || i1 < e1) {
            const int64_t k0 = i0 < e0 ? ext_key[static_cast<size_t>(i0)] : INT64_MAX;
            const int64_t k1 = i1 < e1 ? ext_key[static_cast<size_t>(i1)] : INT64_MAX;
            pe.push_back(k0 <= k1 ? i0 : -1);
            pe.push_back(k1 <= k0 ? i1 : -1);
            if (k0 <= k1) ++i0;
            if (k1 <= k0) ++i1;
          }
          pb.push_back(static_cast<int32_t>(pe.size() / 2));
        }
        f->pext.alloc(std::max<size_t>(pe.size(), 2));
        f->pext_begin.alloc(pb.size());
        if (!pe.empty()) CUDA_CHECK(cudaMemcpy(f->pext.p, pe.data(), pe.size() * 4, cudaMemcpyHostToDevice));
        CUDA_CHECK(cudaMemcpy(f->pext_begin.p, pb.data(), pb.size() * 4, cudaMemcpyHostToDevice));
      }
      f->zero_off = a_off;
      a_off += 16384;  // a zero A image for pair members without rows in a chunk
      f->ext.alloc(static_cast<size_t>(a_off));
      if (f->pair) {
        const int64_t images = a_off / 16384;
        const cuuint64_t adims[2] = {64, static_cast<cuuint64_t>(images * kTileM)};
        const cuuint64_t astr[1] = {128};
        const cuuint32_t abox[2] = {64, static_cast<cuuint32_t>(kTileM)};
        const cuuint32_t ones[3] = {1, 1, 1};
        CUresult r = encode_fn()(&f->amap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, f->ext.p, adims, astr, abox, ones,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) fail(ATMM_ERR_CUDA, "cuTensorMapEncodeTiled(A images) failed: " + std::to_string(r));
        std::vector<CUtensorMap> um(umap_slots.size());
        const int64_t hb = f->bn / 2;
        for (size_t i = 0; i < umap_slots.size(); ++i) {
          const Slot& sl = *umap_slots[i];
          const cuuint64_t udims[3] = {64, static_cast<cuuint64_t>(sl.r_pad / 8),
                                       static_cast<cuuint64_t>(reg->L * reg->d_out_pad / 8)};
          const cuuint64_t ustr[2] = {128, static_cast<cuuint64_t>(sl.r_pad) * 16};
          const cuuint32_t ubox[3] = {64, static_cast<cuuint32_t>(std::min<int64_t>(4, sl.r_pad / 8)),
                                      static_cast<cuuint32_t>(hb / 8)};
          r = encode_fn()(&um[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, sl.up_t, udims, ustr, ubox, ones,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          if (r != CUDA_SUCCESS) fail(ATMM_ERR_CUDA, "cuTensorMapEncodeTiled(up^T) failed: " + std::to_string(r));
        }
        f->umaps.alloc(std::max<size_t>(um.size(), 1));
        if (!um.empty()) CUDA_CHECK(cudaMemcpy(f->umaps.p, um.data(), um.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice));
      }
      f->exts.alloc(exts.size());
      f->ext_begin.alloc(ext_begin.size());
      f->items.alloc(items.size());
      f->order.alloc(order.size());
      CUDA_CHECK(cudaMemset(f->ext.p, 0, f->ext.n));
      CUDA_CHECK(cudaMemcpy(f->exts.p, exts.data(), exts.size() * sizeof(FwdExt), cudaMemcpyHostToDevice));
      CUDA_CHECK(cudaMemcpy(f->ext_begin.p, ext_begin.data(), ext_begin.size() * 4, cudaMemcpyHostToDevice));
      CUDA_CHECK(cudaMemcpy(f->items.p, items.data(), items.size() * sizeof(FwdItem), cudaMemcpyHostToDevice));
      CUDA_CHECK(cudaMemcpy(f->order.p, order.data(), order.size() * 4, cudaMemcpyHostToDevice));
    }
    for (int b = 0; b < 2; ++b) {
      f->buf[b].alloc(static_cast<size_t>(n_ * d));
      f->bmap[b] = make_act_map(f->buf[b].p, n_, d, d);
      if (f->bk2) f->bmap2[b] = make_act_map_atoms(f->buf[b].p, n_, d, d);
    }
    *out = f.release();
  });
}

void atmm_forward_destroy(atmm_forward* f) {
  if (!f) return;
  DeviceGuard g(f->device, std::nothrow);
  delete f;
}

int atmm_forward_stats(const atmm_forward* f, int64_t* out, int64_t cap) {
  return guarded([&] {
    if (!f || !out) fail(ATMM_ERR_CONFIG, "null forward or output");
    const int64_t v[] = {f->n, f->d, f->bn, f->num_tiles, f->grid, f->num_ext, f->num_items, f->ks, f->sorted ? 1 : 0,
                         f->stages_g, f->stages_s, f->pair ? 2 : 1, f->kz};
    const int64_t k = std::min<int64_t>(cap, static_cast<int64_t>(sizeof(v) / sizeof(v[0])));
    for (int64_t i = 0; i < k; ++i) out[i] = v[i];
  });
}

int atmm_forward_run(atmm_forward* f, const void* w, int64_t ldw, int64_t w_layer_stride, int64_t num_layers,
                     const void* x, int64_t ldx, void* out, int64_t ldo, void* stream) {
  return guarded([&] {
    if (!f || !w || !x || !out) fail(ATMM_ERR_CONFIG, "null forward, W, X or output");
    if (f->reg && f->reg->generation != f->generation) {
      fail(ATMM_ERR_CONFIG, "forward is stale: the registry changed since it was created");
    }
    const int64_t d = f->d, n = f->n;
    if (num_layers < 0) fail(ATMM_ERR_SHAPE, "num_layers must be >= 0");
    if (f->reg && num_layers > f->reg->L) fail(ATMM_ERR_SHAPE, "more layers than the adapters carry");
    if (ldw < d || ldw % 8 != 0) fail(ATMM_ERR_SHAPE, "W row stride must be >= hidden_dim and a multiple of 8");
    if (num_layers > 1 && (w_layer_stride < ldw * d || w_layer_stride % 8 != 0)) {
      fail(ATMM_ERR_SHAPE, "W layer stride must be >= ldw * hidden_dim and a multiple of 8");
    }
    if (ldx < d || ldx % 8 != 0) fail(ATMM_ERR_SHAPE, "X row stride must be >= hidden_dim and a multiple of 8");
    if (ldo < d || ldo % 8 != 0) fail(ATMM_ERR_SHAPE, "output row stride must be >= hidden_dim and a multiple of 8");
    require_aligned16(w, "W");
    require_aligned16(x, "X");
    require_aligned16(out, "the output");
    DeviceGuard g(f->device);
    const auto st = static_cast<cudaStream_t>(stream);
    if (num_layers == 0) {
      CUDA_CHECK(cudaMemcpy2DAsync(out, ldo * 2, x, ldx * 2, d * 2, n, cudaMemcpyDeviceToDevice, st));
      return;
    }
    const CUtensorMap wmap = make_layer_w_map(w, d, d, ldw, num_layers, w_layer_stride, f->bk2 ? 2 * kBK : kBK);
    CUtensorMap xm, xg;  // activations for the shrink / for the GEMM (64-wide K atoms under bk2)
    int cur = -1;  // -1: the caller's X
    if (f->sorted) {
      pdl_note_other(st);
      CUDA_CHECK(launch_fwd_gather(static_cast<const uint16_t*>(x), ldx, f->buf[0].p, d, f->order.p, n, d, st));
      cur = 0;
      xm = f->bmap[0];
      xg = f->bk2 ? f->bmap2[0] : xm;
    } else {
      xm = make_act_map(x, n, d, ldx);
      xg = f->bk2 ? make_act_map_atoms(x, n, d, ldx) : xm;
    }
    FwdParams p{};
    const bool bypass = f->num_ext > 0;
    p.ext = f->ext.p;
    p.exts = bypass ? f->exts.p : nullptr;
    p.ext_begin = f->ext_begin.p;
    p.items = f->items.p;
    p.n = n;
    p.d = d;
    p.bn = f->bn;
    p.ntn = f->ntn;
    p.num_tiles = f->num_tiles;
    p.nkb = f->nkb;
    p.ks = f->ks;
    p.num_items = f->num_items;
    p.sbytes = f->sbytes;
    p.pair = f->pair ? 1 : 0;
    p.kz = f->kz;
    p.pext = f->pext.p;
    p.pext_begin = f->pext_begin.p;
    p.zero_a = f->ext.p ? f->ext.p + f->zero_off : nullptr;
    p.umaps = f->umaps.p;
    p.zero_img = static_cast<int32_t>(f->zero_off / 16384);
    p.trace = g_trace;
    // natural K order: forward_mixture's host rows stay bit-identical to
    // forward_merged across the 1-SM / pair kernels (rotation was neutral here)
    p.krot = 0;
    p.mc = 1;
    p.bk2 = f->bk2 ? 1 : 0;
    for (int64_t l = 0; l < num_layers; ++l) {
      const bool last = l + 1 == num_layers;
      const int nxt = cur == 0 ? 1 : 0;
      p.layer = static_cast<int32_t>(l);
      p.out = last ? static_cast<uint16_t*>(out) : f->buf[nxt].p;
      p.ldo = last ? ldo : d;
      p.out_rows = last && f->sorted ? f->order.p : nullptr;
      if (bypass) {
        p.stages = f->stages_s;
        pdl_note_other(st);
        CUDA_CHECK(launch_fwd_shrink(xm, p, f->smem_s, st));
      }
      p.stages = f->stages_g;
      if (f->pair) {
        pdl_note_other(st);
        CUDA_CHECK(launch_fwd_gemm_pair(xg, wmap, f->amap, p, f->grid, f->smem_g, st));
      } else {
        pdl_note_other(st);
        CUDA_CHECK(launch_fwd_gemm(xg, wmap, p, f->grid, f->smem_g, st));
      }
      cur = nxt;
      xm = f->bmap[nxt];
      xg = f->bk2 ? f->bmap2[nxt] : xm;
    }
    // model.hpp:238 (2 n d^2 per layer) + run_bypass per layer (batch.hpp:70-73)
    flops_add(static_cast<uint64_t>(num_layers) * (2ull * static_cast<uint64_t>(n * d * d) + f->bypass_flops));
  });
}

// Plain device GEMM C = A . B (atmm.hpp:111-154 atmm_multiply_into with a
// dense right operand; the base GEMM of model.hpp:238): the layer-forward
// GEMM kernels without the bypass extension and with an identity epilogue.
int atmm_gemm(const void* a, int64_t lda, const void* b, int64_t ldb, void* c, int64_t ldc, int c_dtype, int64_t m,
              int64_t k, int64_t n, void* stream) {
  return atmm_gemm_ex(a, lda, b, ldb, c, ldc, c_dtype, m, k, n, nullptr, stream);
}

namespace atmm {
// The plain GEMM launch behind atmm_gemm_ex (no FLOP accounting: the
// fp32-faithful path calls it on split operands and counts the algorithmic
// product itself).
void gemm_launch(const void* a, int64_t lda, const void* b, int64_t ldb, void* c, int64_t ldc, int c_dtype, int64_t m,
                 int64_t k, int64_t n, const atmm_gemm_opts* opts, void* stream) {
  {
    const atmm_gemm_opts o = opts_or_auto(opts);
    if (m < 0 || k < 0 || n < 0) fail(ATMM_ERR_SHAPE, "negative GEMM shape");
    if (c_dtype != ATMM_BF16 && c_dtype != ATMM_F32) fail(ATMM_ERR_CONFIG, "c_dtype must be ATMM_BF16 or ATMM_F32");
    if (n % 8 != 0) fail(ATMM_ERR_SHAPE, "n must be a multiple of 8 (16-byte output rows)");
    if (m == 0 || n == 0) return;
    if (!c || (k > 0 && (!a || !b))) fail(ATMM_ERR_CONFIG, "null A, B or C");
    if (k > 0 && (lda < k || lda % 8 != 0)) fail(ATMM_ERR_SHAPE, "A row stride must be >= k and a multiple of 8");
    if (k > 0 && (ldb < n || ldb % 8 != 0)) fail(ATMM_ERR_SHAPE, "B row stride must be >= n and a multiple of 8");
    if (ldc < n || ldc % (c_dtype == ATMM_F32 ? 4 : 8) != 0) fail(ATMM_ERR_SHAPE, "C row stride must be >= n and 16-byte aligned");
    if (m > std::numeric_limits<int32_t>::max() / 2 || n > (int64_t(1) << 31) || k > (int64_t(1) << 31)) {
      fail(ATMM_ERR_SHAPE, "GEMM too large");
    }
    require_aligned16(a, "A");
    require_aligned16(b, "B");
    require_aligned16(c, "C");
    int dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    require_device(dev);
    const auto st = static_cast<cudaStream_t>(stream);
    const size_t esz = c_dtype == ATMM_F32 ? 4 : 2;
    if (k == 0) {
      CUDA_CHECK(cudaMemset2DAsync(c, ldc * esz, 0, n * esz, m, st));
      return;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int32_t nkb = static_cast<int32_t>((k + kBK - 1) / kBK);
    const bool pair = pair_without_bypass(m, n, k, sms, o);
    const GemmTiling gt = gemm_tiling(m, n, k, sms, pair, o, true);
    const bool bk2 = gt.bk2;
    const CUtensorMap amap = bk2 ? make_act_map_atoms(a, m, k, lda) : make_act_map(a, m, k, lda, kTileM / gt.mc);
    const CUtensorMap bmap = make_layer_w_map(b, k, n, ldb, 1, 0, bk2 ? 2 * kBK : kBK);
    FwdParams p{};
    p.out = static_cast<uint16_t*>(c);
    p.ldo = ldc;
    p.n = m;
    p.d = n;
    p.bn = gt.bn;
    p.ntn = gt.ntn;
    p.num_tiles = gt.num_tiles;
    p.nkb = nkb;
    p.ks = 1;
    p.stages = gt.stages;
    p.pair = pair ? 1 : 0;
    p.kz = gt.kz;
    p.act_none = 1;
    p.krot = pair ? 1 : 0;  // measured: helps pairs (m = 256: 32 -> 23 us), costs 1-SM 256-wide tiles
    p.mc = gt.mc;
    p.bk2 = bk2 ? 1 : 0;
    p.out_f32 = c_dtype == ATMM_F32 ? 1 : 0;
    p.trace = g_trace;
    if (pair) {
      pdl_note_other(st);
      CUDA_CHECK(launch_fwd_gemm_pair(amap, bmap, amap, p, gt.grid, gt.smem, st));
    } else {
      pdl_note_other(st);
      CUDA_CHECK(launch_fwd_gemm(amap, bmap, p, gt.grid, gt.smem, st));
    }
  }
}
}  // namespace atmm

int atmm_gemm_ex(const void* a, int64_t lda, const void* b, int64_t ldb, void* c, int64_t ldc, int c_dtype, int64_t m,
                 int64_t k, int64_t n, const atmm_gemm_opts* opts, void* stream) {
  return guarded([&] {
    gemm_launch(a, lda, b, ldb, c, ldc, c_dtype, m, k, n, opts, stream);
    flops_add(2ull * static_cast<uint64_t>(m * n * k));  // atmm.hpp:123
  });
}

// =========================================================================
// fp32-faithful path (the reference's fp32 contract on bf16 tensor cores):
// every product is ONE tcgen05 GEMM over the K-concatenation of the
// operands' three-part bf16 splits (six partial products, fp32
// accumulation; precise_kernels.cu).  Used by the reference-signature C++ shim
// (include/loraserve_compat.hpp), whose callers expect 1e-4 agreement with
// their fp32 CPU results (acceptance.cpp:62-101, 107-211).
// =========================================================================
namespace atmm {
namespace {

// Stream-ordered scratch: allocated on `s`, released on `s` after use.
struct AsyncScratch {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  AsyncScratch(size_t bytes, cudaStream_t st) : s(st) {
    if (bytes) CUDA_CHECK(cudaMallocAsync(&p, bytes, st));
  }
  ~AsyncScratch() {
    if (p) cudaFreeAsync(p, s);
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
  AsyncScratch(const AsyncScratch&) = delete;
  AsyncScratch& operator=(const AsyncScratch&) = delete;
};

// T (m x np fp32, row stride np) = A' (m x 6kp bf16) . B' (6kp x np bf16).
void gemm_split(const uint16_t* a3, const uint16_t* b3, float* t, int64_t m, int64_t kp, int64_t np, cudaStream_t st) {
  gemm_launch(a3, kSplitParts * kp, b3, np, t, np, ATMM_F32, m, kSplitParts * kp, np, nullptr, st);
}

void require_precise(const atmm_registry* r) {
  if (!r->precise) {
    fail(ATMM_ERR_CONFIG, "the fp32-faithful path needs a precise registry (atmm_registry_set_precise)");
  }
}

// y[row] += scale * s_a * (x[row] . down_a) . up_a for every routed row of the
// plan, fp32-faithful, per segment: gather + split the rows, x . down, split
// mid, mid . up, scatter-add.
void bypass_f32(const atmm_plan* p, int64_t layer, const float* x, int64_t ldx, float* y, int64_t ldy, float scale,
                cudaStream_t st) {
  const atmm_registry* reg = p->reg;
  require_precise(reg);
  if (p->generation != reg->generation) fail(ATMM_ERR_CONFIG, "plan is stale: the registry changed after the plan was built");
  if (layer < 0 || layer >= reg->L) fail(ATMM_ERR_CONFIG, "layer index " + std::to_string(layer) + " out of range");
  if (!x || !y) fail(ATMM_ERR_SHAPE, "null X or Y");
  if (ldx < reg->d_in || ldy < reg->d_out) fail(ATMM_ERR_SHAPE, "row strides must be >= d_in / d_out");
  const size_t S = p->bp.seg_adapter.size();
  int64_t ns_max = 0, r8_max = 8;
  for (size_t s = 0; s < S; ++s) {
    ns_max = std::max(ns_max, p->bp.seg_offsets[s + 1] - p->bp.seg_offsets[s]);
    r8_max = std::max(r8_max, round_up(reg->at(p->bp.seg_adapter[s]).rank, 8));
  }
  const int64_t kpd = round_up(reg->d_in, 8), n8 = round_up(reg->d_out, 8);
  AsyncScratch xa(size_t(ns_max) * kSplitParts * kpd * 2, st), t1(size_t(ns_max) * r8_max * 4, st),
      ma(size_t(ns_max) * kSplitParts * r8_max * 2, st), t2(size_t(ns_max) * n8 * 4, st);
  for (size_t s = 0; s < S; ++s) {
    const Slot& sl = reg->at(p->bp.seg_adapter[s]);
    const PreciseDims pd(reg, sl.rank);
    const int64_t off = p->bp.seg_offsets[s], ns = p->bp.seg_offsets[s + 1] - off;
    const int32_t* rows = p->d_rows.p + off;
    CUDA_CHECK(launch_split3_rows(x, ldx, rows, ns, reg->d_in, kpd, xa.as<uint16_t>(), kSplitParts * kpd, st));
    gemm_split(xa.as<uint16_t>(), sl.p_down_b + layer * pd.db, t1.as<float>(), ns, kpd, pd.r8, st);
    CUDA_CHECK(launch_split3_rows(t1.as<float>(), pd.r8, nullptr, ns, sl.rank, pd.r8, ma.as<uint16_t>(),
                                  kSplitParts * pd.r8, st));
    gemm_split(ma.as<uint16_t>(), sl.p_up_b + layer * pd.ub, t2.as<float>(), ns, pd.r8, n8, st);
    CUDA_CHECK(launch_rows_out(t2.as<float>(), n8, rows, ns, reg->d_out, y, ldy, scale * sl.scale, 1.0f, st));
  }
}

}  // namespace
}  // namespace atmm

int atmm_registry_set_precise(atmm_registry* r, int on) {
  return guarded([&] {
    if (!r) fail(ATMM_ERR_CONFIG, "null registry");
    if (!r->slot_of.empty() && (on != 0) != r->precise) {
      fail(ATMM_ERR_CONFIG, "set the precision of a registry before putting adapters");
    }
    r->precise = on != 0;
  });
}

int atmm_gemm_f32(const float* a, int64_t lda, const float* b, int64_t ldb, float* c, int64_t ldc, int64_t m,
                  int64_t k, int64_t n, float beta, void* stream) {
  return guarded([&] {
    if (m < 0 || k < 0 || n < 0) fail(ATMM_ERR_SHAPE, "negative GEMM shape");
    if (m == 0 || n == 0) return;
    if (!c || (k > 0 && (!a || !b))) fail(ATMM_ERR_CONFIG, "null A, B or C");
    if ((k > 0 && (lda < k || ldb < n)) || ldc < n) fail(ATMM_ERR_SHAPE, "row strides must cover the matrices");
    if (beta != 0.0f && beta != 1.0f) fail(ATMM_ERR_CONFIG, "beta must be 0 or 1");
    int dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    require_device(dev);
    const auto st = static_cast<cudaStream_t>(stream);
    const int64_t kp = round_up(k, 8), np = round_up(n, 8);
    AsyncScratch a3(size_t(m) * kSplitParts * kp * 2, st), b3(size_t(kSplitParts) * kp * np * 2, st),
        t(size_t(m) * np * 4, st);
    CUDA_CHECK(launch_split3_rows(a, lda, nullptr, m, k, kp, a3.as<uint16_t>(), kSplitParts * kp, st));
    CUDA_CHECK(launch_split3_cols(b, ldb, k, n, kp, np, b3.as<uint16_t>(), st));
    gemm_split(a3.as<uint16_t>(), b3.as<uint16_t>(), t.as<float>(), m, kp, np, st);
    CUDA_CHECK(launch_rows_out(t.as<float>(), np, nullptr, m, n, c, ldc, 1.0f, beta, st));
    flops_add(2ull * static_cast<uint64_t>(m * n * k));
  });
}

int atmm_bypass_apply_f32(const atmm_plan* p, int64_t layer, const float* x, int64_t ldx, float* y, int64_t ldy,
                          float scale, void* stream) {
  return guarded([&] {
    if (!p) fail(ATMM_ERR_CONFIG, "null plan");
    DeviceGuard g(p->reg->device);
    bypass_f32(p, layer, x, ldx, y, ldy, scale, static_cast<cudaStream_t>(stream));
    flops_add(p->flops);
  });
}

int atmm_merge_apply_f32(atmm_registry* r, int32_t adapter_id, int64_t layer0, int64_t num_layers, float* w, int64_t ldw,
                         int64_t w_layer_stride, float sign, void* stream) {
  return guarded([&] {
    if (!r || !w) fail(ATMM_ERR_CONFIG, "null registry or W");
    require_precise(r);
    if (num_layers < 1 || layer0 < 0 || layer0 + num_layers > r->L) fail(ATMM_ERR_CONFIG, "layer range out of range");
    if (ldw < r->d_out || (num_layers > 1 && w_layer_stride < ldw * r->d_in)) fail(ATMM_ERR_SHAPE, "W strides too small");
    const Slot& s = r->at(adapter_id);
    DeviceGuard g(r->device);
    const auto st = static_cast<cudaStream_t>(stream);
    const PreciseDims pd(r, s.rank);
    AsyncScratch t(size_t(r->d_in) * pd.n8 * 4, st);
    for (int64_t l = layer0; l < layer0 + num_layers; ++l) {
      // delta_w_into (model.hpp:120-125) into scratch, then add / sub_inplace (model.hpp:157-158, 180-181)
      gemm_split(s.p_down_a + l * pd.da, s.p_up_b + l * pd.ub, t.as<float>(), r->d_in, pd.r8, pd.n8, st);
      CUDA_CHECK(launch_rows_out(t.as<float>(), pd.n8, nullptr, r->d_in, r->d_out, w + (l - layer0) * w_layer_stride,
                                 ldw, sign * s.scale, 1.0f, st));
    }
    flops_add(2ull * static_cast<uint64_t>(num_layers * r->d_in * r->d_out * s.alg_rank));
  });
}

int atmm_delta_w_f32(atmm_registry* r, int32_t adapter_id, int64_t layer, float* out, int64_t ldo, void* stream) {
  return guarded([&] {
    if (!r || !out) fail(ATMM_ERR_CONFIG, "null registry or output");
    require_precise(r);
    if (layer < 0 || layer >= r->L) {
      fail(ATMM_ERR_CONFIG, "layer index " + std::to_string(layer) + " out of range (L=" + std::to_string(r->L) + ")");
    }
    if (ldo < r->d_out) fail(ATMM_ERR_SHAPE, "output row stride must be >= d_out");
    const Slot& s = r->at(adapter_id);
    DeviceGuard g(r->device);
    const auto st = static_cast<cudaStream_t>(stream);
    const PreciseDims pd(r, s.rank);
    AsyncScratch t(size_t(r->d_in) * pd.n8 * 4, st);
    gemm_split(s.p_down_a + layer * pd.da, s.p_up_b + layer * pd.ub, t.as<float>(), r->d_in, pd.r8, pd.n8, st);
    CUDA_CHECK(launch_rows_out(t.as<float>(), pd.n8, nullptr, r->d_in, r->d_out, out, ldo, s.scale, 0.0f, st));
    flops_add(2ull * static_cast<uint64_t>(r->d_in * r->d_out * s.alg_rank));
  });
}

int atmm_forward_f32(const float* w, int64_t ldw, int64_t w_layer_stride, int64_t num_layers, int64_t n, int64_t d,
                     const float* x, int64_t ldx, float* out, int64_t ldo, const atmm_plan* const* plans,
                     const float* scales, int64_t num_plans, void* stream) {
  return guarded([&] {
    if (!w || !x || !out || (num_plans > 0 && (!plans || !scales))) fail(ATMM_ERR_CONFIG, "null argument");
    if (n < 1 || d < 1 || num_layers < 0) fail(ATMM_ERR_SHAPE, "rows and hidden_dim must be >= 1");
    if (ldw < d || ldx < d || ldo < d || (num_layers > 1 && w_layer_stride < ldw * d)) {
      fail(ATMM_ERR_SHAPE, "row / layer strides must cover the matrices");
    }
    uint64_t bypass_flops = 0;
    for (int64_t i = 0; i < num_plans; ++i) {
      const atmm_plan* p = plans[i];
      if (!p) fail(ATMM_ERR_CONFIG, "null plan");
      require_precise(p->reg);
      if (p->reg->d_in != d || p->reg->d_out != d || p->n != n) fail(ATMM_ERR_SHAPE, "plan does not match the forward");
      if (p->reg->L < num_layers) fail(ATMM_ERR_SHAPE, "more layers than the adapters carry");
      bypass_flops += p->flops;
    }
    int dev = 0;
    CUDA_CHECK(cudaGetDevice(&dev));
    require_device(dev);
    const auto st = static_cast<cudaStream_t>(stream);
    const int64_t kp = round_up(d, 8), d8 = round_up(d, 8);
    AsyncScratch cur(size_t(n) * d8 * 4, st), nxt(size_t(n) * d8 * 4, st), w3(size_t(kSplitParts) * kp * d8 * 2, st),
        a3(size_t(n) * kSplitParts * kp * 2, st);
    float* c = cur.as<float>();
    float* nx = nxt.as<float>();
    CUDA_CHECK(launch_rows_out(x, ldx, nullptr, n, d, c, d8, 1.0f, 0.0f, st));
    for (int64_t l = 0; l < num_layers; ++l) {
      // next = cur . W_l (model.hpp:238) + bypass_l(cur) (model.hpp:239-241, 315-322), tanh
      CUDA_CHECK(launch_split3_cols(w + l * w_layer_stride, ldw, d, d, kp, d8, w3.as<uint16_t>(), st));
      CUDA_CHECK(launch_split3_rows(c, d8, nullptr, n, d, kp, a3.as<uint16_t>(), kSplitParts * kp, st));
      gemm_split(a3.as<uint16_t>(), w3.as<uint16_t>(), nx, n, kp, d8, st);
      for (int64_t i = 0; i < num_plans; ++i) bypass_f32(plans[i], l, c, d8, nx, d8, scales[i], st);
      CUDA_CHECK(launch_tanh(nx, d8, n, d, st));
      std::swap(c, nx);
    }
    CUDA_CHECK(launch_rows_out(c, d8, nullptr, n, d, out, ldo, 1.0f, 0.0f, st));
    flops_add(static_cast<uint64_t>(num_layers) * (2ull * static_cast<uint64_t>(n * d * d) + bypass_flops));
  });
}

// ---- host-buffer forms of the fp32-faithful path (the C++ shim's calls) ----
// Device staging is a per-thread, per-device grow-only workspace (no
// allocation per call once warm); copies and kernels run on one private
// stream per thread, synchronized before returning.
namespace atmm {
namespace {
struct HostStage {
  int device = -1;
  DevBuf<uint8_t> buf;
  cudaStream_t s = nullptr;
  uint8_t* get(int dev, size_t bytes) {
    if (device != dev) {
      buf.release();
      if (s) cudaStreamDestroy(s);
      s = nullptr;
      device = dev;
    }
    if (!s) CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    if (buf.n < bytes) buf.alloc(std::max(bytes, buf.n * 2));
    return buf.p;
  }
};
HostStage& host_stage() {
  thread_local HostStage hs;
  return hs;
}
size_t align256(size_t b) { return (b + 255) / 256 * 256; }
}  // namespace
}  // namespace atmm

int atmm_forward_f32_host(const float* w, int64_t num_layers, int64_t n, int64_t d, const float* x, float* out,
                          const atmm_plan* const* plans, const float* scales, int64_t num_plans) {
  return guarded([&] {
    if (!w || !x || !out) fail(ATMM_ERR_CONFIG, "null argument");
    if (n < 1 || d < 1 || num_layers < 0) fail(ATMM_ERR_SHAPE, "rows and hidden_dim must be >= 1");
    int dev = 0;
    if (num_plans > 0 && plans && plans[0]) dev = plans[0]->reg->device;
    else CUDA_CHECK(cudaGetDevice(&dev));
    require_device(dev);
    DeviceGuard g(dev);
    const size_t wb = align256(size_t(num_layers) * d * d * 4), xb = align256(size_t(n) * d * 4);
    HostStage& hs = host_stage();
    uint8_t* base = hs.get(dev, wb + 2 * xb);
    float* wd = reinterpret_cast<float*>(base);
    float* xd = reinterpret_cast<float*>(base + wb);
    float* od = reinterpret_cast<float*>(base + wb + xb);
    if (num_layers) CUDA_CHECK(cudaMemcpyAsync(wd, w, size_t(num_layers) * d * d * 4, cudaMemcpyHostToDevice, hs.s));
    CUDA_CHECK(cudaMemcpyAsync(xd, x, size_t(n) * d * 4, cudaMemcpyHostToDevice, hs.s));
    const int rc = atmm_forward_f32(wd, d, d * d, num_layers, n, d, xd, d, od, d, plans, scales, num_plans, hs.s);
    if (rc != ATMM_OK) fail(rc, atmm_last_error());
    CUDA_CHECK(cudaMemcpyAsync(out, od, size_t(n) * d * 4, cudaMemcpyDeviceToHost, hs.s));
    CUDA_CHECK(cudaStreamSynchronize(hs.s));
  });
}

int atmm_merge_f32_host(atmm_registry* r, int32_t adapter_id, float* w, float sign) {
  return guarded([&] {
    if (!r || !w) fail(ATMM_ERR_CONFIG, "null registry or W");
    DeviceGuard g(r->device);
    const size_t wb = size_t(r->L) * r->d_in * r->d_out * 4;
    HostStage& hs = host_stage();
    float* wd = reinterpret_cast<float*>(hs.get(r->device, wb));
    CUDA_CHECK(cudaMemcpyAsync(wd, w, wb, cudaMemcpyHostToDevice, hs.s));
    const int rc = atmm_merge_apply_f32(r, adapter_id, 0, r->L, wd, r->d_out, r->d_in * r->d_out, sign, hs.s);
    if (rc != ATMM_OK) fail(rc, atmm_last_error());
    CUDA_CHECK(cudaMemcpyAsync(w, wd, wb, cudaMemcpyDeviceToHost, hs.s));  // in place: the caller's W stays put
    CUDA_CHECK(cudaStreamSynchronize(hs.s));
  });
}
