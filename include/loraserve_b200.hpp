// loraserve_b200.hpp -- header-only C++ shim restoring the reference's
// operator interface (namespace loraserve, /root/reference/proj/include/
// loraserve/) on top of the B200 C ABI (atmm_b200.h).
//
// A reference caller switches by including this header instead of
// batch.hpp / tiling.hpp / model.hpp for the ATMM path and linking
// libatmm_b200.so.  Names, argument meaning and exception types follow the
// reference:
//   plan_batch            batch.hpp:28     -> loraserve_b200::plan_batch
//   run_bypass            batch.hpp:48     -> loraserve_b200::run_bypass
//   TilingConfig/ShapeKey tiling.hpp:22-83 -> same names
//   TilingTable           tiling.hpp:153   -> loraserve_b200::TilingTable
//   delta_w / merge       model.hpp:120-188-> delta_w / merge_into / unmerge_into
//   atmm_multiply         atmm.hpp:144     -> loraserve_b200::atmm_multiply
//   errors.hpp classes    -> same class names, rethrown from ATMM status codes
// The adapter set lives on the device (AdapterRegistry, adapter.hpp:18-110).
#pragma once

#include <array>
#include <map>
#include <compare>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "atmm_b200.h"

namespace loraserve_b200 {

// ------------------------------------------------------------- errors ----
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ShapeError : public Error { using Error::Error; };
class ConfigError : public Error { using Error::Error; };
class ModeError : public Error { using Error::Error; };
class IoError : public Error { using Error::Error; };
class ParseError : public Error { using Error::Error; };
class UnknownAdapterError : public Error { using Error::Error; };
class DeviceError : public Error { using Error::Error; };

inline void check(int status) {
  if (status == ATMM_OK) return;
  const std::string msg = atmm_last_error();
  switch (status) {
    case ATMM_ERR_SHAPE: throw ShapeError(msg);
    case ATMM_ERR_CONFIG: throw ConfigError(msg);
    case ATMM_ERR_MODE: throw ModeError(msg);
    case ATMM_ERR_IO: throw IoError(msg);
    case ATMM_ERR_PARSE: throw ParseError(msg);
    case ATMM_ERR_UNKNOWN_ADAPTER: throw UnknownAdapterError(msg);
    default: throw DeviceError(msg);
  }
}

// ------------------------------------------------------------- tiling ----
struct TilingConfig {
  int outer_m = 0, outer_n = 0, outer_k = 0;
  int inner_m = 0, inner_n = 0, inner_k = 0;
  auto operator<=>(const TilingConfig&) const = default;
  std::array<int32_t, 6> edges() const { return {outer_m, outer_n, outer_k, inner_m, inner_n, inner_k}; }
  static TilingConfig from(const int32_t* e) { return {e[0], e[1], e[2], e[3], e[4], e[5]}; }
  bool structurally_valid() const { return atmm_config_valid(edges().data()) == 1; }
  void validate() const {
    if (!structurally_valid()) throw ConfigError("invalid tiling config");
  }
};

struct ShapeKey {
  int m_bucket = 32, k = 0, n = 0;
  auto operator<=>(const ShapeKey&) const = default;
};
inline int m_bucket_of(std::size_t m) { return atmm_m_bucket_of(static_cast<int64_t>(m)); }
inline ShapeKey shape_key(std::size_t m, std::size_t k, std::size_t n) {
  return ShapeKey{m_bucket_of(m), static_cast<int>(k), static_cast<int>(n)};
}

class TilingTable {
 public:
  TilingTable() { check(atmm_table_create(nullptr, &h_)); }
  explicit TilingTable(TilingConfig d) {
    auto e = d.edges();
    check(atmm_table_create(e.data(), &h_));
  }
  ~TilingTable() { atmm_table_destroy(h_); }
  TilingTable(const TilingTable&) = delete;
  TilingTable& operator=(const TilingTable&) = delete;
  TilingTable(TilingTable&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}

  void insert(ShapeKey key, TilingConfig config, std::int64_t measured_ns) {
    auto e = config.edges();
    check(atmm_table_insert(h_, key.m_bucket, key.k, key.n, e.data(), measured_ns, nullptr));
  }
  TilingConfig lookup(std::size_t m, std::size_t k, std::size_t n) const {
    int32_t out[6];
    check(atmm_table_lookup(h_, static_cast<int64_t>(m), static_cast<int64_t>(k), static_cast<int64_t>(n), out));
    return TilingConfig::from(out);
  }
  std::size_t size() const {
    int64_t s = 0;
    check(atmm_table_size(h_, &s));
    return static_cast<std::size_t>(s);
  }
  void save(const std::string& path) const { check(atmm_table_save(h_, path.c_str())); }
  static TilingTable load(const std::string& path) {
    TilingTable t(nullptr);
    check(atmm_table_load(path.c_str(), &t.h_));
    return t;
  }
  const atmm_table* handle() const { return h_; }

 private:
  explicit TilingTable(std::nullptr_t) {}
  atmm_table* h_ = nullptr;
};

// ------------------------------------------------------------ planner ----
struct Segment {
  int adapter_id = 0;
  std::vector<std::size_t> rows;
};
struct BatchPlan {
  std::vector<Segment> segments;
  std::size_t total_rows = 0;
};

inline BatchPlan plan_batch(const std::vector<int>& assignment) {
  const int64_t n = static_cast<int64_t>(assignment.size());
  std::vector<int32_t> a(assignment.begin(), assignment.end());
  std::vector<int32_t> seg(std::max<int64_t>(n, 1));
  std::vector<int64_t> off(std::max<int64_t>(n, 1) + 1), rows(std::max<int64_t>(n, 1));
  int64_t S = 0;
  check(atmm_plan_batch(a.data(), n, seg.data(), off.data(), rows.data(), &S));
  BatchPlan p;
  p.total_rows = static_cast<std::size_t>(n);
  for (int64_t s = 0; s < S; ++s) {
    Segment g;
    g.adapter_id = seg[s];
    for (int64_t i = off[s]; i < off[s + 1]; ++i) g.rows.push_back(static_cast<std::size_t>(rows[i]));
    p.segments.push_back(std::move(g));
  }
  return p;
}

// ----------------------------------------------------- adapter registry --
class AdapterRegistry {
 public:
  AdapterRegistry(int device, std::size_t num_layers, std::size_t d_in, std::size_t d_out)
      : d_in_(d_in), d_out_(d_out) {
    check(atmm_registry_create(device, static_cast<int64_t>(num_layers), static_cast<int64_t>(d_in),
                               static_cast<int64_t>(d_out), &h_));
  }
  ~AdapterRegistry() { atmm_registry_destroy(h_); }
  AdapterRegistry(const AdapterRegistry&) = delete;
  AdapterRegistry& operator=(const AdapterRegistry&) = delete;

  // down: [L][d_in x r], up: [L][r x d_out], host fp32 (LoraAdapter layout).
  void put(int adapter_id, std::size_t rank, const float* down, const float* up, float scale = 1.0f) {
    check(atmm_registry_put(h_, adapter_id, static_cast<int64_t>(rank), down, up, scale));
  }
  // mode_switch's adapter swap, ordered on `stream` (pinned host memory for
  // an asynchronous copy); same result as put().
  void put_async(int adapter_id, std::size_t rank, const float* down, const float* up, float scale = 1.0f,
                 void* stream = nullptr) {
    check(atmm_registry_put_async(h_, adapter_id, static_cast<int64_t>(rank), down, up, scale, stream));
  }
  // A slot = rank-concatenation of existing adapters with signs folded into
  // up: one bypass then adds sum_i sign_i s_i (x.down_i).up_i.
  void put_combined(int new_id, const std::vector<std::pair<int, float>>& parts) {
    std::vector<int32_t> ids;
    std::vector<float> signs;
    for (const auto& [id, sign] : parts) {
      ids.push_back(id);
      signs.push_back(sign);
    }
    check(atmm_registry_put_combined(h_, new_id, static_cast<int64_t>(ids.size()), ids.data(), signs.data()));
  }
  // load_model_fixture's adapters (model_io.hpp:71-114); returns the count.
  std::size_t load_fixture(const std::string& dir) {
    int64_t n = 0;
    check(atmm_registry_load_fixture(h_, dir.c_str(), &n));
    return static_cast<std::size_t>(n);
  }
  bool contains(int adapter_id) const { return atmm_registry_contains(h_, adapter_id) == 1; }
  atmm_registry* handle() const { return h_; }
  std::size_t d_in() const { return d_in_; }
  std::size_t d_out() const { return d_out_; }

 private:
  atmm_registry* h_ = nullptr;
  std::size_t d_in_, d_out_;
};

// run_bypass (batch.hpp:48): fresh n x d_out bypass from host fp32 x.
inline std::vector<float> run_bypass(const AdapterRegistry& reg, const std::vector<float>& x,
                                     const std::vector<int>& assignment, std::size_t layer,
                                     const TilingTable* table = nullptr) {
  const std::size_t n = assignment.size();
  if (x.size() != n * reg.d_in()) throw ShapeError("run_bypass: x must be n x d_in");
  std::vector<int32_t> a(assignment.begin(), assignment.end());
  std::vector<float> out(n * reg.d_out());
  check(atmm_run_bypass_host(reg.handle(), x.data(), static_cast<int64_t>(n), a.data(),
                             static_cast<int64_t>(layer), table ? table->handle() : nullptr, out.data()));
  return out;
}

// delta_w (model.hpp:130-140) for one layer, host fp32 d_in x d_out.
inline std::vector<float> delta_w(const AdapterRegistry& reg, int adapter_id, std::size_t layer) {
  std::vector<float> out(reg.d_in() * reg.d_out());
  check(atmm_delta_w_host(reg.handle(), adapter_id, static_cast<int64_t>(layer), out.data()));
  return out;
}

// merge / unmerge one layer in place on a device weight (W +-= s.down.up).
inline void merge_into(const AdapterRegistry& reg, int adapter_id, std::size_t layer, void* w_device,
                       std::size_t ldw, int w_dtype, void* stream = nullptr) {
  check(atmm_merge_apply(reg.handle(), adapter_id, static_cast<int64_t>(layer), w_device,
                         static_cast<int64_t>(ldw), w_dtype, +1.0f, stream));
}
inline void unmerge_into(const AdapterRegistry& reg, int adapter_id, std::size_t layer, void* w_device,
                         std::size_t ldw, int w_dtype, void* stream = nullptr) {
  check(atmm_merge_apply(reg.handle(), adapter_id, static_cast<int64_t>(layer), w_device,
                         static_cast<int64_t>(ldw), w_dtype, -1.0f, stream));
}

// merge / unmerge every layer [layer0, layer0 + num_layers) in ONE launch;
// layer l's W at w_device + (l - layer0) * w_layer_stride elements.
inline void merge_layers_into(const AdapterRegistry& reg, int adapter_id, std::size_t layer0, std::size_t num_layers,
                              void* w_device, std::size_t ldw, std::size_t w_layer_stride, int w_dtype, float sign,
                              void* stream = nullptr) {
  check(atmm_merge_apply_layers(reg.handle(), adapter_id, static_cast<int64_t>(layer0),
                                static_cast<int64_t>(num_layers), w_device, static_cast<int64_t>(ldw),
                                static_cast<int64_t>(w_layer_stride), w_dtype, sign, stream));
}

// atmm_multiply_into (atmm.hpp:111-142) on device buffers with a dense right
// operand, the base GEMM of every layer (model.hpp:238): C = A . B, bf16 A/B
// row-major, C bf16 or fp32 (c_dtype ATMM_BF16 / ATMM_F32), overwritten.
inline void gemm(const void* a, std::size_t lda, const void* b, std::size_t ldb, void* c, std::size_t ldc, int c_dtype,
                 std::size_t m, std::size_t k, std::size_t n, void* stream = nullptr) {
  check(atmm_gemm(a, static_cast<int64_t>(lda), b, static_cast<int64_t>(ldb), c, static_cast<int64_t>(ldc), c_dtype,
                  static_cast<int64_t>(m), static_cast<int64_t>(k), static_cast<int64_t>(n), stream));
}

// forward_mixture's per-layer bypass (model.hpp:252-328) on device buffers:
// guest rows (adapter != merged_id) get (x.down_a).up_a - (x.down_m).up_m in
// ONE launch through combined slots (ids combined_base - k); merged rows are
// untouched.  X: n x d_in bf16, Y: n x d_out (y_dtype).
class MixturePlan {
 public:
  MixturePlan(AdapterRegistry& reg, const std::vector<int>& assignment, int merged_id, int combined_base = -(1 << 20)) {
    if (!reg.contains(merged_id)) throw ModeError("mixture integrity: subtraction branch missing");
    std::vector<int32_t> guest_rows, virt;
    std::map<int, int> combo;
    for (std::size_t row = 0; row < assignment.size(); ++row) {
      const int a = assignment[row];
      if (a == merged_id) continue;
      auto it = combo.find(a);
      if (it == combo.end()) {
        const int vid = combined_base - static_cast<int>(combo.size());
        reg.put_combined(vid, {{a, 1.0f}, {merged_id, -1.0f}});
        it = combo.emplace(a, vid).first;
      }
      guest_rows.push_back(static_cast<int32_t>(row));
      virt.push_back(it->second);
    }
    if (!guest_rows.empty()) {
      check(atmm_plan_create_mapped(reg.handle(), virt.data(), guest_rows.data(), static_cast<int64_t>(virt.size()),
                                    static_cast<int64_t>(assignment.size()), nullptr, &plan_));
    }
  }
  ~MixturePlan() { atmm_plan_destroy(plan_); }
  MixturePlan(const MixturePlan&) = delete;
  MixturePlan& operator=(const MixturePlan&) = delete;
  void apply(std::size_t layer, const void* x, std::size_t ldx, void* y, std::size_t ldy, int y_dtype,
             float scale = 1.0f, void* stream = nullptr) const {
    if (!plan_) return;
    check(atmm_bypass_apply(plan_, static_cast<int64_t>(layer), x, static_cast<int64_t>(ldx), y,
                            static_cast<int64_t>(ldy), y_dtype, scale, stream));
  }

  const atmm_plan* handle() const { return plan_; }  // null: every row is the merged adapter's

 private:
  atmm_plan* plan_ = nullptr;
};

// --------------------------------------------------------- layer forward --
// forward_unmerged / forward_mixture / forward_merged (model.hpp:192-328) on
// device buffers: cur <- tanh(cur . W_l + bypass_l(cur)) over num_layers.
// W: num_layers x [d][d] bf16 (row stride ldw, layer stride w_layer_stride);
// x / out: n x d bf16.  The bypass runs as extra K blocks of the base GEMM.
class LayerForward {
 public:
  // forward_unmerged: every row's own adapter.
  LayerForward(AdapterRegistry& reg, const std::vector<int>& assignment) {
    std::vector<int32_t> a(assignment.begin(), assignment.end());
    check(atmm_plan_create(reg.handle(), a.data(), static_cast<int64_t>(a.size()), nullptr, &plan_));
    check(atmm_forward_create(plan_, 0, 0, 0, &f_));
  }
  // forward_mixture over merged weights (the plan's registry must outlive this).
  LayerForward(const MixturePlan& mp, int device, std::size_t n, std::size_t hidden_dim) {
    check(atmm_forward_create(mp.handle(), device, static_cast<int64_t>(n), static_cast<int64_t>(hidden_dim), &f_));
  }
  // forward_merged: no bypass.
  LayerForward(int device, std::size_t n, std::size_t hidden_dim) {
    check(atmm_forward_create(nullptr, device, static_cast<int64_t>(n), static_cast<int64_t>(hidden_dim), &f_));
  }
  ~LayerForward() {
    atmm_forward_destroy(f_);
    atmm_plan_destroy(plan_);
  }
  LayerForward(const LayerForward&) = delete;
  LayerForward& operator=(const LayerForward&) = delete;
  void run(const void* w, std::size_t ldw, std::size_t w_layer_stride, std::size_t num_layers, const void* x,
           std::size_t ldx, void* out, std::size_t ldo, void* stream = nullptr) {
    check(atmm_forward_run(f_, w, static_cast<int64_t>(ldw), static_cast<int64_t>(w_layer_stride),
                           static_cast<int64_t>(num_layers), x, static_cast<int64_t>(ldx), out,
                           static_cast<int64_t>(ldo), stream));
  }

 private:
  atmm_plan* plan_ = nullptr;
  atmm_forward* f_ = nullptr;
};

// ------------------------------------------------------------- fixtures --
// save_matrix / load_matrix<float> (matrix.hpp:183-218), the reference's format.
inline void save_matrix(const std::string& path, std::size_t rows, std::size_t cols, const std::vector<float>& m) {
  if (m.size() != rows * cols) throw ShapeError("save_matrix: data must be rows x cols");
  check(atmm_matrix_save(path.c_str(), static_cast<int64_t>(rows), static_cast<int64_t>(cols), m.data()));
}
inline std::vector<float> load_matrix(const std::string& path, std::size_t* rows, std::size_t* cols) {
  int64_t r = 0, c = 0;
  check(atmm_matrix_load(path.c_str(), &r, &c, nullptr, 0));
  std::vector<float> out(static_cast<std::size_t>(r * c));
  check(atmm_matrix_load(path.c_str(), &r, &c, out.data(), r * c));
  if (rows) *rows = static_cast<std::size_t>(r);
  if (cols) *cols = static_cast<std::size_t>(c);
  return out;
}

// atmm_multiply (atmm.hpp:144-154): host fp32 a (m x k) . b (k x n).
inline std::vector<float> atmm_multiply(const std::vector<float>& a, std::size_t m, std::size_t k,
                                        const std::vector<float>& b, std::size_t n, const TilingConfig& cfg) {
  if (a.size() != m * k || b.size() != k * n) throw ShapeError("atmm_multiply: shape mismatch");
  std::vector<float> c(m * n);
  auto e = cfg.edges();
  check(atmm_multiply_host(a.data(), static_cast<int64_t>(m), static_cast<int64_t>(k), b.data(),
                           static_cast<int64_t>(n), c.data(), e.data()));
  return c;
}

}  // namespace loraserve_b200
