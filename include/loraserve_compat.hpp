// loraserve_compat.hpp -- drop-in for the reference's ATMM operator interface.
//
// A caller of the reference (namespace loraserve, /root/reference/proj/
// include/loraserve/{matrix,adapter,tiling,atmm,batch,model}.hpp) switches to
// the B200 operator by replacing those includes with this header and linking
// libatmm_b200.so: the types, function names, signatures, return values and
// exception classes below are the reference's.  Every product runs on the
// B200 through the C ABI (include/atmm_b200.h), fp32-faithfully: each fp32
// operand is split into three bf16 parts and multiplied on tcgen05 tensor
// cores with fp32 accumulation (atmm_*_f32), so results meet the reference's
// own 1e-4 * max(1, max|ref|) gates.  There is no CPU fallback: without a B200
// every operator throws DeviceError.
//
//   reference                                  here (device path)
//   atmm_multiply_into / atmm_multiply          atmm_multiply_host
//     (atmm.hpp:111-154)
//   plan_batch (batch.hpp:28-42)                atmm_plan_batch
//   run_bypass (batch.hpp:48-81)                atmm_run_bypass_host (precise registry)
//   delta_w (model.hpp:130-140)                 atmm_delta_w_host (precise registry)
//   merge / unmerge (model.hpp:144-188)         atmm_merge_f32_host (+ the ModeError contract)
//   forward_merged / _unmerged / _mixture       atmm_forward_f32_host
//     (model.hpp:192-328)
//   init_delora / mode_switch (serving.hpp:24-74)
//   TilingTable / tiling_search / benchmark_config (tiling.hpp, atmm.hpp:188-355)
//   flops::read / reset / Scope (flops.hpp)     atmm_flops_read / reset
//
// Adapters reach the device through a per-thread cache of precise registries
// (one per (num_layers, hidden_dim)), keyed by adapter id and re-uploaded
// only when the LoraAdapter object changes: serving loops pay the factor
// upload once.  Out of scope (not the ATMM path): task heads / decode,
// scheduler, serving loop, workload generator, fusion planner.
#pragma once

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <compare>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "atmm_b200.h"

namespace loraserve {

// ------------------------------------------------------------- errors ----
// errors.hpp:10-61: the same classes and constructors.
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ShapeError : public Error {
 public:
  explicit ShapeError(const std::string& msg) : Error(msg) {}
  ShapeError(std::size_t ar, std::size_t ac, std::size_t br, std::size_t bc, const std::string& op)
      : Error(op + ": shape mismatch " + std::to_string(ar) + "x" + std::to_string(ac) + " vs " +
              std::to_string(br) + "x" + std::to_string(bc)) {}
};
class ConfigError : public Error {
 public:
  using Error::Error;
};
class ModeError : public Error {
 public:
  using Error::Error;
};
class IoError : public Error {
 public:
  using Error::Error;
};
class ParseError : public Error {
 public:
  ParseError(const std::string& msg, std::size_t line) : Error(msg + " (line " + std::to_string(line) + ")"), line_(line) {}
  std::size_t line() const { return line_; }

 private:
  std::size_t line_;
};
class UnknownAdapterError : public Error {
 public:
  explicit UnknownAdapterError(int id) : Error("unknown adapter id " + std::to_string(id)), id_(id) {}
  int id() const { return id_; }

 private:
  int id_;
};
// No reference counterpart: the device is missing or a CUDA call failed.
class DeviceError : public Error {
 public:
  using Error::Error;
};

namespace detail {
// Rethrows an ATMM status as the reference's exception class.
inline void check(int status, int unknown_id = 0) {
  if (status == ATMM_OK) return;
  const std::string msg = atmm_last_error();
  switch (status) {
    case ATMM_ERR_SHAPE: throw ShapeError(msg);
    case ATMM_ERR_CONFIG: throw ConfigError(msg);
    case ATMM_ERR_MODE: throw ModeError(msg);
    case ATMM_ERR_IO: throw IoError(msg);
    case ATMM_ERR_PARSE: throw ParseError(msg, 0);
    case ATMM_ERR_UNKNOWN_ADAPTER: throw UnknownAdapterError(unknown_id);
    default: throw DeviceError(msg);
  }
}
}  // namespace detail

// ---------------------------------------------------------------- flops --
// flops.hpp: the library's thread-local algorithmic FLOP counter.
namespace flops {
inline std::uint64_t read() { return atmm_flops_read(); }
inline void reset() { atmm_flops_reset(); }
class Scope {
 public:
  Scope() : start_(read()) {}
  std::uint64_t elapsed() const { return read() - start_; }

 private:
  std::uint64_t start_;
};
}  // namespace flops

// ------------------------------------------------------------- matrices --
// matrix.hpp:23-94: row-major carriers (host memory, the reference's ABI).
template <typename T>
class Matrix {
  static_assert(std::is_floating_point_v<T>);

 public:
  Matrix() = default;
  Matrix(std::size_t rows, std::size_t cols) : rows_(rows), cols_(cols), data_(rows * cols, T(0)) {
    if (rows == 0 || cols == 0) {
      throw ShapeError("matrix dimensions must be >= 1, got " + std::to_string(rows) + "x" + std::to_string(cols));
    }
  }
  std::size_t rows() const { return rows_; }
  std::size_t cols() const { return cols_; }
  std::size_t size() const { return data_.size(); }
  T* data() { return data_.data(); }
  const T* data() const { return data_.data(); }
  T& operator()(std::size_t i, std::size_t j) { return data_[i * cols_ + j]; }
  const T& operator()(std::size_t i, std::size_t j) const { return data_[i * cols_ + j]; }
  void fill(T v) { std::fill(data_.begin(), data_.end(), v); }

 private:
  std::size_t rows_ = 0, cols_ = 0;
  std::vector<T> data_;
};

template <typename T>
struct MatSpan {
  T* data = nullptr;
  std::size_t rows = 0, cols = 0;
  MatSpan() = default;
  MatSpan(T* d, std::size_t r, std::size_t c) : data(d), rows(r), cols(c) {}
  MatSpan(Matrix<T>& m) : data(m.data()), rows(m.rows()), cols(m.cols()) {}
  T& operator()(std::size_t i, std::size_t j) const { return data[i * cols + j]; }
};

template <typename T>
struct ConstMatSpan {
  const T* data = nullptr;
  std::size_t rows = 0, cols = 0;
  ConstMatSpan() = default;
  ConstMatSpan(const T* d, std::size_t r, std::size_t c) : data(d), rows(r), cols(c) {}
  ConstMatSpan(const Matrix<T>& m) : data(m.data()), rows(m.rows()), cols(m.cols()) {}
  ConstMatSpan(MatSpan<T> m) : data(m.data), rows(m.rows), cols(m.cols) {}
  const T& operator()(std::size_t i, std::size_t j) const { return data[i * cols + j]; }
};

// random.hpp:12-27: the synthetic inputs (std::mt19937_64 + the standard
// uniform distribution, so a caller's seeded data is bit-identical).
using Rng = std::mt19937_64;
template <typename T>
void fill_uniform(MatSpan<T> m, Rng& rng, T lo = T(-1), T hi = T(1)) {
  std::uniform_real_distribution<T> dist(lo, hi);
  for (std::size_t i = 0, e = m.rows * m.cols; i < e; ++i) m.data[i] = dist(rng);
}
template <typename T>
Matrix<T> random_matrix(std::size_t rows, std::size_t cols, Rng& rng, T lo = T(-1), T hi = T(1)) {
  Matrix<T> m(rows, cols);
  fill_uniform<T>(m, rng, lo, hi);
  return m;
}

// --------------------------------------------------------------- tiling --
// tiling.hpp:22-254 through the C ABI (the same validity, bucketing, lookup
// and JSON; entries may carry the B200 launch, ignored by the reference).
struct TilingConfig {
  int outer_m = 0, outer_n = 0, outer_k = 0;
  int inner_m = 0, inner_n = 0, inner_k = 0;
  auto operator<=>(const TilingConfig&) const = default;
  std::array<int, 6> edges() const { return {outer_m, outer_n, outer_k, inner_m, inner_n, inner_k}; }
  std::size_t footprint_elems() const {
    return std::size_t(outer_m) * outer_k + std::size_t(outer_k) * outer_n + std::size_t(outer_m) * outer_n;
  }
  bool structurally_valid() const {
    const auto e = edges();
    const int32_t v[6] = {e[0], e[1], e[2], e[3], e[4], e[5]};
    return atmm_config_valid(v) == 1;
  }
  void validate() const {
    if (!structurally_valid()) throw ConfigError("invalid tiling config " + to_string());
  }
  std::string to_string() const {
    std::string s = "(";
    const auto e = edges();
    for (std::size_t i = 0; i < 6; ++i) s += std::to_string(e[i]) + (i < 5 ? "," : ")");
    return s;
  }
  static TilingConfig from(const int32_t* v) { return {v[0], v[1], v[2], v[3], v[4], v[5]}; }
};

struct ShapeKey {
  int m_bucket = 32;
  int k = 0;
  int n = 0;
  auto operator<=>(const ShapeKey&) const = default;
};
inline int m_bucket_of(std::size_t m) { return atmm_m_bucket_of(static_cast<int64_t>(m)); }
inline ShapeKey shape_key(std::size_t m, std::size_t k, std::size_t n) {
  return ShapeKey{m_bucket_of(m), static_cast<int>(k), static_cast<int>(n)};
}

class TilingTable {
 public:
  TilingTable() : h_(make(nullptr)) {}
  explicit TilingTable(TilingConfig default_config) : h_(make(&default_config)) {}
  void insert(ShapeKey key, TilingConfig config, std::int64_t measured_ns) {
    const auto e = edges(config);
    detail::check(atmm_table_insert(h_.get(), key.m_bucket, key.k, key.n, e.data(), measured_ns, nullptr));
  }
  void set_default(TilingConfig config) {
    const auto e = edges(config);
    detail::check(atmm_table_set_default(h_.get(), e.data(), nullptr));
  }
  TilingConfig lookup(std::size_t m, std::size_t k, std::size_t n) const {
    int32_t out[6];
    detail::check(atmm_table_lookup(h_.get(), int64_t(m), int64_t(k), int64_t(n), out));
    return TilingConfig::from(out);
  }
  std::size_t size() const {
    int64_t s = 0;
    detail::check(atmm_table_size(h_.get(), &s));
    return static_cast<std::size_t>(s);
  }
  bool empty() const { return size() == 0; }
  void save(const std::string& path) const { detail::check(atmm_table_save(h_.get(), path.c_str())); }
  static TilingTable load(const std::string& path) {
    atmm_table* t = nullptr;
    detail::check(atmm_table_load(path.c_str(), &t));
    return TilingTable(t);
  }
  const atmm_table* handle() const { return h_.get(); }
  explicit TilingTable(atmm_table* adopt) : h_(adopt, &atmm_table_destroy) {}

 private:
  static std::array<int32_t, 6> edges(const TilingConfig& c) {
    const auto e = c.edges();
    return {e[0], e[1], e[2], e[3], e[4], e[5]};
  }
  static std::shared_ptr<atmm_table> make(const TilingConfig* d) {
    atmm_table* t = nullptr;
    if (d) {
      const auto e = edges(*d);
      detail::check(atmm_table_create(e.data(), &t));
    } else {
      detail::check(atmm_table_create(nullptr, &t));
    }
    return std::shared_ptr<atmm_table>(t, &atmm_table_destroy);
  }
  std::shared_ptr<atmm_table> h_;
};

inline TilingConfig lookup_config(const TilingTable& table, std::size_t m, std::size_t k, std::size_t n) {
  return table.lookup(m, k, n);
}

// ----------------------------------------------------------------- ATMM --
// atmm.hpp:111-154: C = A . B, fp32-faithful on the tensor cores; the config
// is validated like the reference's (the B200 tiles are the GEMM's own).
template <typename T>
void atmm_multiply_into(ConstMatSpan<T> a, ConstMatSpan<T> b, MatSpan<T> c, const TilingConfig& cfg) {
  static_assert(std::is_same_v<T, float>, "the B200 operator computes the reference's fp32 path");
  if (a.cols != b.rows) throw ShapeError(a.rows, a.cols, b.rows, b.cols, "atmm_multiply");
  if (c.rows != a.rows || c.cols != b.cols) throw ShapeError(c.rows, c.cols, a.rows, b.cols, "atmm_multiply output");
  cfg.validate();
  const auto e = cfg.edges();
  const int32_t v[6] = {e[0], e[1], e[2], e[3], e[4], e[5]};
  detail::check(atmm_multiply_host(a.data, int64_t(a.rows), int64_t(a.cols), b.data, int64_t(b.cols), c.data, v));
}
template <typename T>
Matrix<T> atmm_multiply(ConstMatSpan<T> a, ConstMatSpan<T> b, const TilingConfig& cfg) {
  Matrix<T> c(a.rows, b.cols);
  atmm_multiply_into<T>(a, b, c, cfg);
  return c;
}

// ------------------------------------------------------------- adapters --
// adapter.hpp:18-110: per-layer factor pairs, immutable after construction.
class LoraAdapter {
 public:
  LoraAdapter(int id, std::size_t num_layers, std::size_t hidden_dim, std::size_t rank, std::vector<Matrix<float>> down,
              std::vector<Matrix<float>> up)
      : id_(id), rank_(rank), hidden_dim_(hidden_dim), down_(std::move(down)), up_(std::move(up)) {
    if (rank_ >= hidden_dim_) throw ConfigError("adapter rank must be < hidden dim");
    if (down_.size() != num_layers || up_.size() != num_layers) {
      throw ConfigError("adapter needs a down/up pair for every layer");
    }
    for (std::size_t l = 0; l < num_layers; ++l) {
      if (down_[l].rows() != hidden_dim_ || down_[l].cols() != rank_ || up_[l].rows() != rank_ ||
          up_[l].cols() != hidden_dim_) {
        throw ShapeError("adapter layer " + std::to_string(l) + " factor shapes do not match (d=" +
                         std::to_string(hidden_dim_) + ", r=" + std::to_string(rank_) + ")");
      }
    }
  }
  // adapter.hpp:53-73: down, up ~ U(+-1/sqrt(r)), layer by layer.
  static LoraAdapter random(int id, std::size_t num_layers, std::size_t hidden_dim, std::size_t rank,
                            std::uint64_t seed) {
    Rng rng(seed);
    const float s = 1.0f / std::sqrt(static_cast<float>(rank));
    std::vector<Matrix<float>> down, up;
    for (std::size_t l = 0; l < num_layers; ++l) {
      down.push_back(random_matrix<float>(hidden_dim, rank, rng, -s, s));
      up.push_back(random_matrix<float>(rank, hidden_dim, rng, -s, s));
    }
    return LoraAdapter(id, num_layers, hidden_dim, rank, std::move(down), std::move(up));
  }
  int id() const { return id_; }
  std::size_t rank() const { return rank_; }
  std::size_t hidden_dim() const { return hidden_dim_; }
  std::size_t num_layers() const { return down_.size(); }
  ConstMatSpan<float> down(std::size_t layer) const { return down_.at(layer); }
  ConstMatSpan<float> up(std::size_t layer) const { return up_.at(layer); }
  std::size_t bytes() const { return num_layers() * 2 * hidden_dim_ * rank_ * sizeof(float); }

 private:
  int id_;
  std::size_t rank_, hidden_dim_;
  std::vector<Matrix<float>> down_, up_;
};

using AdapterSet = std::map<int, LoraAdapter>;

inline const LoraAdapter& adapter_at(const AdapterSet& set, int id) {
  auto it = set.find(id);
  if (it == set.end()) throw UnknownAdapterError(id);
  return it->second;
}

// ----------------------------------------------------------- the device --
namespace detail {
// Per-thread device registries (one per (layers, hidden)), fp32-faithful,
// holding the adapters callers pass by reference.  An adapter is uploaded
// once and re-uploaded only when a different LoraAdapter object (or one with
// different factors at the sampled positions) appears under its id.
class DeviceCtx {
 public:
  ~DeviceCtx() {
    for (auto& [key, r] : regs_) atmm_registry_destroy(r.h);
  }
  atmm_registry* registry(std::size_t layers, std::size_t d) {
    auto it = regs_.find({layers, d});
    if (it != regs_.end()) return it->second.h;
    Reg r;
    check(atmm_registry_create(0, int64_t(layers), int64_t(d), int64_t(d), &r.h));
    const int st = atmm_registry_set_precise(r.h, 1);
    if (st != ATMM_OK) {
      atmm_registry_destroy(r.h);
      check(st);
    }
    return regs_.emplace(std::make_pair(layers, d), r).first->second.h;
  }
  atmm_registry* holding(const LoraAdapter& a) {
    atmm_registry* h = registry(a.num_layers(), a.hidden_dim());
    Reg& r = regs_.at({a.num_layers(), a.hidden_dim()});
    const Held want{&a, fingerprint(a)};
    auto it = r.held.find(a.id());
    if (it != r.held.end() && it->second.obj == want.obj && it->second.print == want.print) return h;
    const std::size_t d = a.hidden_dim(), rk = a.rank(), L = a.num_layers();
    std::vector<float> down(L * d * rk), up(L * rk * d);
    for (std::size_t l = 0; l < L; ++l) {
      std::copy(a.down(l).data, a.down(l).data + d * rk, down.begin() + l * d * rk);
      std::copy(a.up(l).data, a.up(l).data + rk * d, up.begin() + l * rk * d);
    }
    check(atmm_registry_put(h, a.id(), int64_t(rk), down.data(), up.data(), 1.0f));
    r.held[a.id()] = want;
    return h;
  }

 private:
  struct Held {
    const LoraAdapter* obj = nullptr;
    std::uint64_t print = 0;
  };
  struct Reg {
    atmm_registry* h = nullptr;
    std::map<int, Held> held;
  };
  static std::uint64_t fingerprint(const LoraAdapter& a) {
    std::uint64_t h = 1469598103934665603ull ^ a.rank() ^ (std::uint64_t(a.num_layers()) << 32);
    auto mix = [&h](float v) {
      std::uint32_t u;
      std::memcpy(&u, &v, 4);
      h = (h ^ u) * 1099511628211ull;
    };
    for (std::size_t l = 0; l < a.num_layers(); ++l) {
      const std::size_t nd = a.down(l).rows * a.down(l).cols, nu = a.up(l).rows * a.up(l).cols;
      for (std::size_t i = 0; i < nd; i += 1 + nd / 64) mix(a.down(l).data[i]);
      for (std::size_t i = 0; i < nu; i += 1 + nu / 64) mix(a.up(l).data[i]);
    }
    return h;
  }
  std::map<std::pair<std::size_t, std::size_t>, Reg> regs_;
};
inline DeviceCtx& device() {
  thread_local DeviceCtx ctx;
  return ctx;
}

// An atmm plan (routing tables + launches) owned for one call.
struct Plan {
  atmm_plan* h = nullptr;
  Plan() = default;
  Plan(atmm_registry* r, const std::vector<int32_t>& assignment) {
    check(atmm_plan_create(r, assignment.data(), int64_t(assignment.size()), nullptr, &h));
  }
  Plan(atmm_registry* r, const std::vector<int32_t>& assignment, const std::vector<int32_t>& rows, std::size_t n_rows) {
    check(atmm_plan_create_mapped(r, assignment.data(), rows.data(), int64_t(assignment.size()), int64_t(n_rows),
                                  nullptr, &h));
  }
  ~Plan() { atmm_plan_destroy(h); }
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;
};
}  // namespace detail

// ---------------------------------------------------------------- batch --
// batch.hpp:17-81.
struct Segment {
  int adapter_id = 0;
  std::vector<std::size_t> rows;
};
struct BatchPlan {
  std::vector<Segment> segments;
  std::size_t total_rows = 0;
};

inline BatchPlan plan_batch(std::span<const int> assignment) {
  const int64_t n = static_cast<int64_t>(assignment.size());
  std::vector<int32_t> a(assignment.begin(), assignment.end());
  std::vector<int32_t> seg(std::max<int64_t>(n, 1));
  std::vector<int64_t> off(std::max<int64_t>(n, 1) + 1), rows(std::max<int64_t>(n, 1));
  int64_t S = 0;
  detail::check(atmm_plan_batch(a.data(), n, seg.data(), off.data(), rows.data(), &S));
  BatchPlan p;
  p.total_rows = static_cast<std::size_t>(n);
  for (int64_t s = 0; s < S; ++s) {
    Segment g{seg[s], {}};
    for (int64_t i = off[s]; i < off[s + 1]; ++i) g.rows.push_back(static_cast<std::size_t>(rows[i]));
    p.segments.push_back(std::move(g));
  }
  return p;
}

// run_bypass (batch.hpp:48-81): a fresh n x d bypass, every segment at its
// own rank, fp32-faithful on the device.
inline Matrix<float> run_bypass(ConstMatSpan<float> x, const BatchPlan& plan, const AdapterSet& adapters,
                                std::size_t layer, const TilingTable& table) {
  if (x.rows != plan.total_rows) {
    throw ShapeError("run_bypass: batch has " + std::to_string(x.rows) + " rows but plan covers " +
                     std::to_string(plan.total_rows));
  }
  Matrix<float> out(x.rows, x.cols);
  std::vector<int32_t> assignment(x.rows, 0);
  atmm_registry* reg = nullptr;
  for (const Segment& seg : plan.segments) {
    const LoraAdapter& a = adapter_at(adapters, seg.adapter_id);
    if (a.hidden_dim() != x.cols) throw ShapeError(x.rows, x.cols, a.hidden_dim(), a.rank(), "run_bypass");
    reg = detail::device().holding(a);
    for (std::size_t r : seg.rows) assignment[r] = seg.adapter_id;
  }
  if (!reg) return out;
  detail::check(atmm_run_bypass_host(reg, x.data, int64_t(x.rows), assignment.data(), int64_t(layer), table.handle(),
                                     out.data()));
  return out;
}

// --------------------------------------------------------------- model ---
// model.hpp:25-112: the base model (host weights, address-stable) and state.
class BaseModel {
 public:
  BaseModel(std::size_t num_layers, std::size_t hidden_dim, std::size_t vocab_size)
      : num_layers_(num_layers), hidden_dim_(hidden_dim), vocab_size_(vocab_size),
        weights_(num_layers * hidden_dim * hidden_dim, 0.0f) {
    if (num_layers < 1 || hidden_dim < 16 || vocab_size < 2) throw ConfigError("model needs L >= 1, d >= 16, V >= 2");
  }
  // model.hpp:44-56: layer weights ~ U(+-1/sqrt(d)) drawn layer by layer
  // (the vocabulary head the reference draws next is not modelled here).
  static BaseModel random(std::size_t num_layers, std::size_t hidden_dim, std::size_t vocab_size, std::uint64_t seed) {
    BaseModel m(num_layers, hidden_dim, vocab_size);
    Rng rng(seed);
    const float s = 1.0f / std::sqrt(static_cast<float>(hidden_dim));
    for (std::size_t l = 0; l < num_layers; ++l) fill_uniform<float>(m.layer(l), rng, -s, s);
    return m;
  }
  std::size_t num_layers() const { return num_layers_; }
  std::size_t hidden_dim() const { return hidden_dim_; }
  std::size_t vocab_size() const { return vocab_size_; }
  MatSpan<float> layer(std::size_t i) { return {weights_.data() + i * hidden_dim_ * hidden_dim_, hidden_dim_, hidden_dim_}; }
  ConstMatSpan<float> layer(std::size_t i) const {
    return {weights_.data() + i * hidden_dim_ * hidden_dim_, hidden_dim_, hidden_dim_};
  }
  float* weights() { return weights_.data(); }
  const float* weights() const { return weights_.data(); }

 private:
  std::size_t num_layers_, hidden_dim_, vocab_size_;
  std::vector<float> weights_;
};

enum class InferMode { Unmerged, Merged, Mixture };
inline const char* mode_name(InferMode m) {
  return m == InferMode::Unmerged ? "unmerged" : (m == InferMode::Merged ? "merged" : "mixture");
}
struct ModelState {
  InferMode mode = InferMode::Unmerged;
  int merged_adapter = -1;
  const LoraAdapter* delora_branch = nullptr;
};
using DurationNs = std::chrono::nanoseconds;

namespace detail {
inline void require_match(const BaseModel& model, const LoraAdapter& a) {
  if (a.num_layers() != model.num_layers() || a.hidden_dim() != model.hidden_dim()) {
    throw ShapeError("adapter does not match model dimensions");
  }
}
inline DurationNs since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration_cast<DurationNs>(std::chrono::steady_clock::now() - t0);
}
}  // namespace detail

inline Matrix<float> delta_w(const LoraAdapter& adapter, std::size_t layer, const TilingTable& /*table*/) {
  if (layer >= adapter.num_layers()) {
    throw ConfigError("layer index " + std::to_string(layer) + " out of range (L=" +
                      std::to_string(adapter.num_layers()) + ")");
  }
  Matrix<float> out(adapter.hidden_dim(), adapter.hidden_dim());
  detail::check(atmm_delta_w_host(detail::device().holding(adapter), adapter.id(), int64_t(layer), out.data()));
  return out;
}

// merge / unmerge (model.hpp:144-188): all layers in place, one device pass
// each; the mode contract is the reference's.
inline DurationNs merge(BaseModel& model, ModelState& state, const LoraAdapter& adapter, const TilingTable&) {
  if (state.mode != InferMode::Unmerged) {
    throw ModeError(std::string("merge requires unmerged state (currently ") + mode_name(state.mode) + ")");
  }
  detail::require_match(model, adapter);
  const auto t0 = std::chrono::steady_clock::now();
  detail::check(atmm_merge_f32_host(detail::device().holding(adapter), adapter.id(), model.weights(), +1.0f));
  state.mode = InferMode::Merged;
  state.merged_adapter = adapter.id();
  state.delora_branch = nullptr;
  return detail::since(t0);
}

inline DurationNs unmerge(BaseModel& model, ModelState& state, const LoraAdapter& adapter, const TilingTable&) {
  if (state.mode == InferMode::Unmerged) throw ModeError("unmerge requires merged or mixture state");
  if (state.merged_adapter != adapter.id()) {
    throw ModeError("unmerge of adapter " + std::to_string(adapter.id()) + " but adapter " +
                    std::to_string(state.merged_adapter) + " is merged");
  }
  const auto t0 = std::chrono::steady_clock::now();
  detail::check(atmm_merge_f32_host(detail::device().holding(adapter), adapter.id(), model.weights(), -1.0f));
  state.mode = InferMode::Unmerged;
  state.merged_adapter = -1;
  state.delora_branch = nullptr;
  return detail::since(t0);
}

namespace detail {
inline Matrix<float> forward(const BaseModel& model, ConstMatSpan<float> x, const std::vector<const Plan*>& plans,
                             const std::vector<float>& scales) {
  const std::size_t d = model.hidden_dim();
  if (x.cols != d) throw ShapeError("input cols must equal hidden_dim");
  Matrix<float> out(x.rows, d);
  std::vector<const atmm_plan*> hs;
  for (const Plan* p : plans) hs.push_back(p->h);
  check(atmm_forward_f32_host(model.weights(), int64_t(model.num_layers()), int64_t(x.rows), int64_t(d), x.data,
                              out.data(), hs.data(), scales.data(), int64_t(hs.size())));
  return out;
}
}  // namespace detail

// forward_merged (model.hpp:192-211): tanh(x W) through every layer.
inline Matrix<float> forward_merged(const BaseModel& model, const ModelState& state, ConstMatSpan<float> x,
                                    const TilingTable&) {
  if (state.mode != InferMode::Merged) throw ModeError("forward_merged requires merged state");
  return detail::forward(model, x, {}, {});
}

// forward_unmerged (model.hpp:216-246): tanh(x W + bypass(x)) per layer.
inline Matrix<float> forward_unmerged(const BaseModel& model, const ModelState& state, ConstMatSpan<float> x,
                                      std::span<const int> assignment, const AdapterSet& adapters,
                                      const TilingTable&) {
  if (state.mode != InferMode::Unmerged) throw ModeError("forward_unmerged requires unmerged state");
  if (x.cols != model.hidden_dim()) throw ShapeError("input cols must equal hidden_dim");
  if (assignment.size() != x.rows) throw ShapeError("assignment size must equal row count");
  atmm_registry* reg = nullptr;
  for (int id : assignment) {
    const LoraAdapter& a = adapter_at(adapters, id);  // fail fast on unknown ids (model.hpp:226-228)
    detail::require_match(model, a);
    reg = detail::device().holding(a);
  }
  const detail::Plan plan(reg, std::vector<int32_t>(assignment.begin(), assignment.end()));
  return detail::forward(model, x, {&plan}, {1.0f});
}

// forward_mixture (model.hpp:251-328): the merged adapter's rows ride the
// merged weights; every guest row adds its own bypass and cancels the
// merged adapter's (x W_merged - (x down_m) up_m + (x down_a) up_a).
inline Matrix<float> forward_mixture(const BaseModel& model, const ModelState& state, ConstMatSpan<float> x,
                                     std::span<const int> assignment, const AdapterSet& adapters,
                                     const TilingTable&) {
  if (state.mode != InferMode::Mixture) throw ModeError("forward_mixture requires mixture state");
  if (state.delora_branch == nullptr || state.delora_branch->id() != state.merged_adapter) {
    throw ModeError("mixture integrity: subtraction branch missing or not weight-identical to the merged adapter");
  }
  if (x.cols != model.hidden_dim()) throw ShapeError("input cols must equal hidden_dim");
  if (assignment.size() != x.rows) throw ShapeError("assignment size must equal row count");
  std::vector<int32_t> guest_rows, guest_ids;
  for (std::size_t row = 0; row < x.rows; ++row) {
    if (assignment[row] == state.merged_adapter) continue;
    guest_rows.push_back(static_cast<int32_t>(row));
    guest_ids.push_back(assignment[row]);
  }
  if (guest_rows.empty()) return detail::forward(model, x, {}, {});
  atmm_registry* reg = nullptr;
  for (int id : guest_ids) {
    const LoraAdapter& a = adapter_at(adapters, id);
    detail::require_match(model, a);
    reg = detail::device().holding(a);
  }
  const LoraAdapter& merged = adapter_at(adapters, state.merged_adapter);
  reg = detail::device().holding(merged);
  const detail::Plan own(reg, guest_ids, guest_rows, x.rows);
  const detail::Plan cancel(reg, std::vector<int32_t>(guest_rows.size(), merged.id()), guest_rows, x.rows);
  return detail::forward(model, x, {&own, &cancel}, {1.0f, -1.0f});
}

// serving.hpp:24-33: the subtraction branch is the merged adapter itself.
inline void init_delora(ModelState& state, const LoraAdapter& merged_adapter) {
  if (state.merged_adapter != merged_adapter.id()) throw ModeError("deLoRA branch must reference the merged adapter");
  state.delora_branch = &merged_adapter;
}

// serving.hpp:38-74: the minimal sequence of one-shot un/merges for a mode
// transition; merged -> mixture of the same adapter touches no weights.
inline DurationNs mode_switch(BaseModel& model, ModelState& state, InferMode to_mode, int target_adapter,
                              const AdapterSet& adapters, const TilingTable& table) {
  const auto t0 = std::chrono::steady_clock::now();
  if (to_mode == InferMode::Unmerged) {
    if (state.mode != InferMode::Unmerged) unmerge(model, state, adapter_at(adapters, state.merged_adapter), table);
    return detail::since(t0);
  }
  if (target_adapter < 0) throw ModeError("merged/mixture transition needs a target adapter");
  const LoraAdapter& target = adapter_at(adapters, target_adapter);
  if (state.mode != InferMode::Unmerged && state.merged_adapter != target_adapter) {
    unmerge(model, state, adapter_at(adapters, state.merged_adapter), table);
  }
  if (state.mode == InferMode::Unmerged) merge(model, state, target, table);
  if (to_mode == InferMode::Mixture) {
    init_delora(state, target);
    state.mode = InferMode::Mixture;
  } else {
    state.delora_branch = nullptr;
    state.mode = InferMode::Merged;
  }
  return detail::since(t0);
}

// ------------------------------------------------- offline tiling search --
// atmm.hpp:188-355 on the B200.  A GemmShape (m, k, n) with n < k is read as
// the bypass of segments of m rows at hidden k and rank n (the reference's
// rank-shaped grid entries, atmm.hpp:350-353); other shapes have no B200
// bypass kernel and are reported as failures.  Candidates are reference
// TilingConfigs, read as B200 launches (atmm_b200.h: tile rows, K slice per
// CTA -> cluster, expand chunk).
struct GemmShape {
  std::size_t m = 0, k = 0, n = 0;
};
struct BenchResult {
  std::int64_t median_ns = 0;
  bool timer_warning = false;
};

namespace detail {
inline std::array<int32_t, 5> launch_of(const TilingConfig& c, std::size_t d) {
  const auto e = c.edges();
  const int32_t v[6] = {e[0], e[1], e[2], e[3], e[4], e[5]};
  atmm_table* t = nullptr;
  check(atmm_table_create(v, &t));
  std::array<int32_t, 5> l{};
  const int st = atmm_table_resolve_launch(t, 32, int64_t(d), 16, int64_t(d), l.data());
  atmm_table_destroy(t);
  check(st);
  return l;
}
inline atmm_tune_shape tune_shape(const GemmShape& s) {
  const int64_t segs = std::clamp<int64_t>(1024 / std::max<int64_t>(int64_t(s.m), 1), 4, 64);
  return atmm_tune_shape{int64_t(s.m), int64_t(s.k), int64_t(s.n), int64_t(s.k), segs};
}
}  // namespace detail

inline BenchResult benchmark_config(std::size_t m, std::size_t k, std::size_t n, const TilingConfig& cfg, int trials,
                                    std::uint64_t seed = 0x5eedbeef) {
  if (trials < 3) throw ConfigError("benchmark_config needs trials >= 3");
  cfg.validate();
  if (n >= k) throw ConfigError("benchmark_config: B200 shapes are bypass shapes (m rows, hidden k, rank n < k)");
  const atmm_tune_shape sh = detail::tune_shape({m, k, n});
  const auto l = detail::launch_of(cfg, k);
  BenchResult r;
  detail::check(atmm_benchmark_launch(0, &sh, l.data(), trials, seed, &r.median_ns));
  return r;
}

inline TilingTable tiling_search(const std::vector<GemmShape>& shape_grid, const std::vector<TilingConfig>& candidates,
                                 int trials, std::vector<std::string>* failures = nullptr) {
  if (shape_grid.empty() || candidates.empty()) throw ConfigError("tiling_search needs a nonempty grid and candidates");
  std::vector<atmm_tune_shape> shapes;
  for (const GemmShape& s : shape_grid) {
    if (s.n < s.k) {
      shapes.push_back(detail::tune_shape(s));
    } else if (failures) {
      failures->push_back("shape " + std::to_string(s.m) + "x" + std::to_string(s.k) + "x" + std::to_string(s.n) +
                          ": no B200 bypass kernel for this shape, omitted");
    }
  }
  if (shapes.empty()) throw ConfigError("tiling_search: no bypass-shaped grid entries");
  std::vector<int32_t> launches;
  for (const TilingConfig& c : candidates) {
    c.validate();
    const auto l = detail::launch_of(c, shapes.front().d_in);
    launches.insert(launches.end(), l.begin(), l.end());
  }
  std::string buf(1 << 16, '\0');
  atmm_table* t = nullptr;
  detail::check(atmm_tiling_search(0, shapes.data(), int64_t(shapes.size()), launches.data(),
                                   int64_t(candidates.size()), trials, &t, buf.data(), buf.size()));
  if (failures) {
    std::size_t p = 0;
    const std::string all(buf.c_str());
    while (p < all.size()) {
      const std::size_t q = all.find('\n', p);
      failures->push_back(all.substr(p, q == std::string::npos ? std::string::npos : q - p));
      if (q == std::string::npos) break;
      p = q + 1;
    }
  }
  return TilingTable(t);
}

// atmm.hpp:341-355: the hidden-d shape grid, bypass entries (m x d x r).
inline std::vector<GemmShape> default_shape_grid(std::size_t d, const std::vector<std::size_t>& ranks = {16, 32, 64, 128}) {
  std::vector<GemmShape> grid;
  for (std::size_t r : ranks) {
    for (std::size_t m : {32, 64, 128, 256, 512}) grid.push_back({m, d, r});
  }
  return grid;
}

}  // namespace loraserve
