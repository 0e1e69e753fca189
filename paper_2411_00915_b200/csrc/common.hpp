// common.hpp -- host-side internals shared by host.cpp (pure C++) and
// device.cu (CUDA runtime).  Not part of the public ABI.
#pragma once

#include <array>
#include <compare>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/atmm_b200.h"

namespace atmm {

// Internal exception; every extern "C" entry point converts it to a status
// code + thread-local message (the loraserve exception classes are restored
// by the C++ shim, include/loraserve_b200.hpp).
struct Failure : std::runtime_error {
  int code;
  Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Failure(code, msg); }

void set_last_error(const std::string& msg);

// flops.hpp:10-24: thread-local algorithmic FLOP counter (one multiply-add =
// 2 FLOPs, padding never counted).  Every compute entry point adds what the
// reference's GEMMs would have counted for the same call.
void flops_add(uint64_t n);

// Runs f, mapping exceptions to ATMM status codes.
template <typename F>
int guarded(F&& f) noexcept {
  try {
    f();
    set_last_error("");
    return ATMM_OK;
  } catch (const Failure& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return ATMM_ERR_INTERNAL;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return ATMM_ERR_INTERNAL;
  } catch (...) {
    set_last_error("unknown exception");
    return ATMM_ERR_INTERNAL;
  }
}

// ------------------------------------------------------------ tiling ----
// TilingConfig (tiling.hpp:22-65): {outer_m, outer_n, outer_k, inner_m,
// inner_n, inner_k}.
struct TilingConfig {
  std::array<int32_t, 6> e{};
  auto operator<=>(const TilingConfig&) const = default;
  bool structurally_valid() const;
  std::string str() const;
  int64_t footprint_elems() const {
    return int64_t(e[0]) * e[2] + int64_t(e[2]) * e[1] + int64_t(e[0]) * e[1];
  }
};
TilingConfig reference_default_config();  // {64,32,32,32,32,32} (tiling.hpp:160)

struct ShapeKey {
  int32_t m_bucket = 32, k = 0, n = 0;
  auto operator<=>(const ShapeKey&) const = default;
};
int32_t m_bucket_of(int64_t m);

// Launch parameters of the fused bypass kernel for one segment shape.
struct LaunchCfg {
  int32_t tile_m = 128;  // rows per cluster tile
  int32_t cluster = 8;   // CTAs per cluster (K / N split)
  int32_t bn = 128;      // expand N chunk
  int32_t stages = 0;    // 0 = as many as shared memory allows (<= 6)
  int32_t path = 0;      // kernel: 0 automatic, 1 all-to-all fused, 2 split pair, 3 general fused, 4 stream
  auto operator<=>(const LaunchCfg&) const = default;
};
// A launch as the 5 ints of the C ABI ({tile_m, cluster, bn, stages, path}).
void validate_launch(const LaunchCfg& l);
inline LaunchCfg launch_from_ints(const int32_t* v) { return LaunchCfg{v[0], v[1], v[2], v[3], v[4]}; }
inline void launch_to_ints(const LaunchCfg& l, int32_t* v) {
  v[0] = l.tile_m;
  v[1] = l.cluster;
  v[2] = l.bn;
  v[3] = l.stages;
  v[4] = l.path;
}

// ---- reference fixture I/O (matrix.hpp:183-218, model_io.hpp:25-114) ----
// Binary matrix: little-endian u32 rows, u32 cols, u8 scalar width, row-major payload.
std::vector<float> load_matrix_f32(const std::string& path, int64_t& rows, int64_t& cols);
void save_matrix_f32(const std::string& path, int64_t rows, int64_t cols, const float* data);
struct FixtureAdapter {
  int32_t id = 0;
  int64_t rank = 0;
  std::vector<std::string> down, up;  // per-layer matrix files (relative to the fixture dir)
};
struct FixtureManifest {
  int64_t num_layers = 0, hidden_dim = 0;
  std::vector<FixtureAdapter> adapters;
};
FixtureManifest read_fixture_manifest(const std::string& dir);

struct TableEntry {
  TilingConfig config;
  int64_t measured_ns = 0;
  bool has_sm100 = false;
  LaunchCfg sm100;
};

class TilingTable {
 public:
  TilingTable();  // reference default config, heuristic B200 resolution
  explicit TilingTable(const TilingConfig& dflt);
  void insert(ShapeKey key, const TilingConfig& cfg, int64_t ns, const LaunchCfg* sm100);
  void set_default(const TilingConfig& cfg, const LaunchCfg* sm100 = nullptr);
  const TilingConfig& default_config() const { return default_; }
  const LaunchCfg* default_launch() const { return has_default_sm100_ ? &default_sm100_ : nullptr; }
  const std::map<ShapeKey, TableEntry>& entries() const { return entries_; }
  // tiling.hpp:181-199
  const TableEntry* find(int64_t m, int64_t k, int64_t n) const;
  TilingConfig lookup(int64_t m, int64_t k, int64_t n) const;
  // B200 launch for a segment of m rows at (d_in, rank, d_out).
  LaunchCfg resolve_launch(int64_t m, int64_t d_in, int64_t rank, int64_t d_out) const;
  std::string to_json() const;
  static TilingTable from_json(const std::string& text);
  bool heuristic_default() const { return heuristic_default_; }

 private:
  std::map<ShapeKey, TableEntry> entries_;
  TilingConfig default_;
  bool heuristic_default_ = true;
  bool has_default_sm100_ = false;  // the default's B200 launch (JSON "default_sm100")
  LaunchCfg default_sm100_;
};

LaunchCfg heuristic_launch(int64_t m, int64_t d_in, int64_t rank, int64_t d_out);
LaunchCfg launch_from_config(const TilingConfig& cfg, int64_t d_in);
std::vector<TilingConfig> candidate_configs(size_t budget, size_t width);
std::vector<TilingConfig> default_candidates(size_t budget, size_t width);

// ----------------------------------------------------------- planner ----
struct BatchPlan {
  std::vector<int32_t> seg_adapter;   // ascending ids
  std::vector<int64_t> seg_offsets;   // S + 1
  std::vector<int64_t> row_index;     // n, stable within a segment
};
BatchPlan plan_batch(const int32_t* assignment, int64_t n);

// bf16 round-to-nearest-even (NaN preserved).
inline uint16_t f32_to_bf16(float f) {
  uint32_t u;
  static_assert(sizeof(u) == sizeof(f));
  __builtin_memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu)) return uint16_t((u >> 16) | 0x40);
  u += 0x7fffu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}
inline float bf16_to_f32(uint16_t h) {
  uint32_t u = uint32_t(h) << 16;
  float f;
  __builtin_memcpy(&f, &u, 4);
  return f;
}

}  // namespace atmm

// Opaque handle behind atmm_table* (atmm_b200.h).
struct atmm_table {
  atmm::TilingTable t;
};
