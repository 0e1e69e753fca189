// host.cpp -- host-side logic of the ATMM operator that needs no GPU:
// tiling configs and the shape-keyed table (+ JSON persistence), the batch
// planner, request sharding, and their C-ABI entry points.
//
// Reference (paths under /root/reference/proj/include/loraserve/):
//   tiling.hpp:22-65   TilingConfig            tiling.hpp:68-83  ShapeKey / m_bucket_of
//   tiling.hpp:88-149  candidate enumeration   tiling.hpp:153-254 TilingTable (+JSON)
//   batch.hpp:28-42    plan_batch
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <memory>
#include <numeric>
#include <sstream>
#include <variant>

#include "common.hpp"

namespace atmm {

namespace {
thread_local std::string g_last_error;
thread_local uint64_t g_flops = 0;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
void flops_add(uint64_t n) { g_flops += n; }

// ------------------------------------------------------------- tiling ---

bool TilingConfig::structurally_valid() const {
  for (int32_t v : e) {
    if (v < 16 || (v & (v - 1)) != 0) return false;
  }
  return e[3] <= e[0] && e[4] <= e[1] && e[5] <= e[2] && e[0] % e[3] == 0 &&
         e[1] % e[4] == 0 && e[2] % e[5] == 0;
}

std::string TilingConfig::str() const {
  std::string s = "(";
  for (size_t i = 0; i < 6; ++i) {
    s += std::to_string(e[i]);
    s += i + 1 < 6 ? "," : ")";
  }
  return s;
}

TilingConfig reference_default_config() { return TilingConfig{{64, 32, 32, 32, 32, 32}}; }

static void validate_config(const TilingConfig& c) {
  if (!c.structurally_valid()) fail(ATMM_ERR_CONFIG, "invalid tiling config " + c.str());
}

int32_t m_bucket_of(int64_t m) {
  if (m <= 32) return 32;
  return static_cast<int32_t>((m + 31) / 32 * 32);
}

TilingTable::TilingTable() : default_(reference_default_config()), heuristic_default_(true) {}
TilingTable::TilingTable(const TilingConfig& dflt) : default_(dflt), heuristic_default_(false) {
  validate_config(dflt);
}

void TilingTable::insert(ShapeKey key, const TilingConfig& cfg, int64_t ns,
                         const LaunchCfg* sm100) {
  validate_config(cfg);
  TableEntry e;
  e.config = cfg;
  e.measured_ns = ns;
  if (sm100) {
    validate_launch(*sm100);
    e.has_sm100 = true;
    e.sm100 = *sm100;
  }
  entries_[key] = e;
}

void validate_launch(const LaunchCfg& l) {
  if (l.tile_m < 1 || l.tile_m > 128 || l.cluster < 1 || l.cluster > 16 || l.bn < 64 || l.bn > 256 ||
      l.bn % 64 != 0 || l.stages < 0 || l.stages > 8 || l.path < 0 || l.path > 4) {
    fail(ATMM_ERR_CONFIG, "invalid sm100 launch parameters");
  }
}

void TilingTable::set_default(const TilingConfig& cfg, const LaunchCfg* sm100) {
  validate_config(cfg);
  if (sm100 && sm100->tile_m == 0) {  // {0, ...}: shapes the table misses resolve through the B200 heuristic
    default_ = cfg;
    heuristic_default_ = true;
    has_default_sm100_ = false;
    return;
  }
  if (sm100) validate_launch(*sm100);
  default_ = cfg;
  heuristic_default_ = false;
  has_default_sm100_ = sm100 != nullptr;
  if (sm100) default_sm100_ = *sm100;
}

const TableEntry* TilingTable::find(int64_t m, int64_t k, int64_t n) const {
  const ShapeKey key{m_bucket_of(m), static_cast<int32_t>(k), static_cast<int32_t>(n)};
  if (auto it = entries_.find(key); it != entries_.end()) return &it->second;
  const TableEntry* best = nullptr;
  int32_t best_dist = 0;
  for (const auto& [ek, entry] : entries_) {  // ascending m_bucket: ties keep the smaller
    if (ek.k != key.k || ek.n != key.n) continue;
    const int32_t dist = std::abs(ek.m_bucket - key.m_bucket);
    if (best == nullptr || dist < best_dist) {
      best = &entry;
      best_dist = dist;
    }
  }
  if (best != nullptr && best_dist <= 32) return best;
  return nullptr;
}

TilingConfig TilingTable::lookup(int64_t m, int64_t k, int64_t n) const {
  const TableEntry* e = find(m, k, n);
  return e ? e->config : default_;
}

static int32_t clamp_pow2_rows(int32_t v) {
  int32_t t = 16;
  while (t < v && t < 128) t <<= 1;
  return std::min(t, 128);
}

// The six reference edges read as B200 launch parameters (atmm_b200.h).
LaunchCfg launch_from_config(const TilingConfig& cfg, int64_t d_in) {
  LaunchCfg l;
  l.tile_m = clamp_pow2_rows(cfg.e[0]);
  const int64_t ks = std::max<int64_t>(cfg.e[2], 64);
  l.cluster = static_cast<int32_t>(std::clamp<int64_t>((d_in + ks - 1) / ks, 1, 16));
  l.bn = std::clamp(cfg.e[1] / 64 * 64, 64, 256);
  l.stages = 0;
  return l;
}

// Heuristic B200 launch when the table has no profile for the shape:
// ~512-wide K slices per CTA (cluster of 8 at d = 4096), whole 128-row tiles,
// expand chunks of 128 (small segments, rank > 32) or 256 columns.
LaunchCfg heuristic_launch(int64_t m, int64_t d_in, int64_t rank, int64_t d_out) {
  (void)d_out;
  LaunchCfg l;
  l.tile_m = 128;
  l.cluster = static_cast<int32_t>(std::clamp<int64_t>((d_in + 511) / 512, 1, 16));
  // Small segments are latency bound: 128-column chunks keep TMEM at 256
  // columns so two CTAs fit per SM (see resolve_group).
  l.bn = (m <= 64 || rank > 32) ? 128 : 256;
  l.stages = 0;
  return l;
}

LaunchCfg TilingTable::resolve_launch(int64_t m, int64_t d_in, int64_t rank, int64_t d_out) const {
  // The fused launch is keyed like the reference's shrink lookup
  // table.lookup(ns, d, r) (batch.hpp:70).
  if (const TableEntry* e = find(m, d_in, rank)) {
    return e->has_sm100 ? e->sm100 : launch_from_config(e->config, d_in);
  }
  if (heuristic_default_) return heuristic_launch(m, d_in, rank, d_out);
  if (has_default_sm100_) return default_sm100_;
  return launch_from_config(default_, d_in);
}

// ---- candidates (tiling.hpp:88-149) ----
std::vector<TilingConfig> candidate_configs(size_t budget, size_t width) {
  if (budget == 0 || width == 0) fail(ATMM_ERR_CONFIG, "cache budget and scalar width must be positive");
  static constexpr int32_t kEdges[5] = {16, 32, 64, 128, 256};
  std::vector<TilingConfig> out;
  for (int32_t om : kEdges)
    for (int32_t on : kEdges)
      for (int32_t ok : kEdges) {
        const size_t fp = (size_t(om) * ok + size_t(ok) * on + size_t(om) * on) * width;
        if (fp > budget) continue;
        for (int32_t im : kEdges) {
          if (im > om) break;
          for (int32_t in : kEdges) {
            if (in > on) break;
            for (int32_t ik : kEdges) {
              if (ik > ok) break;
              out.push_back(TilingConfig{{om, on, ok, im, in, ik}});
            }
          }
        }
      }
  if (out.empty()) {
    fail(ATMM_ERR_CONFIG, "no feasible tiling config for cache budget " + std::to_string(budget) + " bytes");
  }
  return out;
}

std::vector<TilingConfig> default_candidates(size_t budget, size_t width) {
  // B200 curated list read as (tile rows, expand chunk, K slice per CTA,
  // UMMA_M, N granule, K stage): K slices 256 / 512 / 1024 give clusters of
  // 16 / 8 / 4 CTAs at d = 4096.  Filtered by the reference's footprint rule
  // (tiling.hpp:137-143) so the list honours the same budget contract.
  static const TilingConfig curated[] = {
      {{128, 128, 256, 128, 16, 64}}, {{128, 256, 256, 128, 16, 64}},
      {{128, 128, 512, 128, 16, 64}}, {{128, 256, 512, 128, 16, 64}},
      {{128, 64, 512, 128, 16, 64}},  {{128, 64, 1024, 128, 16, 64}},
      {{64, 128, 256, 64, 16, 64}},   {{64, 128, 512, 64, 16, 64}},
      {{64, 256, 512, 64, 16, 64}},   {{64, 128, 1024, 64, 16, 64}},
      {{32, 256, 512, 32, 16, 64}},   {{32, 128, 1024, 32, 16, 64}},
  };
  std::vector<TilingConfig> out;
  for (const auto& c : curated) {
    if (static_cast<size_t>(c.footprint_elems()) * width <= budget) out.push_back(c);
  }
  if (out.empty()) {
    fail(ATMM_ERR_CONFIG, "no feasible default candidate for cache budget " + std::to_string(budget) + " bytes");
  }
  return out;
}

// ---- minimal JSON (enough for the TilingTable schema) ----
namespace json {

struct Value;
using Object = std::map<std::string, Value>;
using Array = std::vector<Value>;
struct Value {
  std::variant<std::nullptr_t, bool, double, std::string, Array, Object> v;
  bool is_num() const { return std::holds_alternative<double>(v); }
  bool is_arr() const { return std::holds_alternative<Array>(v); }
  bool is_obj() const { return std::holds_alternative<Object>(v); }
  const Array& arr() const { return std::get<Array>(v); }
  const Object& obj() const { return std::get<Object>(v); }
  double num() const { return std::get<double>(v); }
};

class Parser {
 public:
  explicit Parser(const std::string& s) : s_(s) {}
  Value parse() {
    Value v = value();
    ws();
    if (i_ != s_.size()) bad("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void bad(const char* what) {
    fail(ATMM_ERR_IO, std::string("bad tiling table json: ") + what + " at offset " + std::to_string(i_));
  }
  void ws() {
    while (i_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[i_]))) ++i_;
  }
  bool lit(const char* t) {
    const size_t n = std::strlen(t);
    if (s_.compare(i_, n, t) == 0) {
      i_ += n;
      return true;
    }
    return false;
  }
  Value value() {
    ws();
    if (i_ >= s_.size()) bad("unexpected end");
    const char c = s_[i_];
    if (c == '{') return object();
    if (c == '[') return array();
    if (c == '"') return Value{string()};
    if (lit("true")) return Value{true};
    if (lit("false")) return Value{false};
    if (lit("null")) return Value{nullptr};
    return number();
  }
  std::string string() {
    ++i_;
    std::string out;
    while (i_ < s_.size() && s_[i_] != '"') {
      if (s_[i_] == '\\') {
        ++i_;
        if (i_ >= s_.size()) bad("bad escape");
        const char e = s_[i_];
        if (e == 'n') out += '\n';
        else if (e == 't') out += '\t';
        else if (e == 'u') { out += '?'; i_ += 4; }
        else out += e;
        ++i_;
      } else {
        out += s_[i_++];
      }
    }
    if (i_ >= s_.size()) bad("unterminated string");
    ++i_;
    return out;
  }
  Value number() {
    const char* b = s_.c_str() + i_;
    char* e = nullptr;
    const double d = std::strtod(b, &e);
    if (e == b) bad("unexpected character");
    i_ += static_cast<size_t>(e - b);
    return Value{d};
  }
  Value array() {
    ++i_;
    Array a;
    ws();
    if (i_ < s_.size() && s_[i_] == ']') {
      ++i_;
      return Value{a};
    }
    for (;;) {
      a.push_back(value());
      ws();
      if (i_ < s_.size() && s_[i_] == ',') { ++i_; continue; }
      if (i_ < s_.size() && s_[i_] == ']') { ++i_; break; }
      bad("expected , or ]");
    }
    return Value{a};
  }
  Value object() {
    ++i_;
    Object o;
    ws();
    if (i_ < s_.size() && s_[i_] == '}') {
      ++i_;
      return Value{o};
    }
    for (;;) {
      ws();
      if (i_ >= s_.size() || s_[i_] != '"') bad("expected key");
      std::string k = string();
      ws();
      if (i_ >= s_.size() || s_[i_] != ':') bad("expected :");
      ++i_;
      o[k] = value();
      ws();
      if (i_ < s_.size() && s_[i_] == ',') { ++i_; continue; }
      if (i_ < s_.size() && s_[i_] == '}') { ++i_; break; }
      bad("expected , or }");
    }
    return Value{o};
  }
  const std::string& s_;
  size_t i_ = 0;
};

const Value& at(const Object& o, const char* key) {
  auto it = o.find(key);
  if (it == o.end()) fail(ATMM_ERR_IO, std::string("tiling table json: missing key '") + key + "'");
  return it->second;
}
int64_t as_int(const Value& v, const char* what) {
  if (!v.is_num()) fail(ATMM_ERR_IO, std::string("tiling table json: ") + what + " must be a number");
  return static_cast<int64_t>(std::llround(v.num()));
}

}  // namespace json

static TilingConfig cfg_from_json(const json::Value& v) {
  if (!v.is_arr() || v.arr().size() != 6) fail(ATMM_ERR_IO, "tiling config must be an array of 6 ints");
  TilingConfig c;
  for (int i = 0; i < 6; ++i) c.e[i] = static_cast<int32_t>(json::as_int(v.arr()[i], "config edge"));
  return c;
}

static std::string cfg_json(const TilingConfig& c) {
  std::string s = "[";
  for (int i = 0; i < 6; ++i) s += std::to_string(c.e[i]) + (i < 5 ? ", " : "]");
  return s;
}

static std::string launch_json(const LaunchCfg& l) {
  std::ostringstream o;
  o << "{\"bn\": " << l.bn << ", \"cluster\": " << l.cluster;
  if (l.path != 0) o << ", \"path\": " << l.path;
  o << ", \"stages\": " << l.stages << ", \"tile_m\": " << l.tile_m << "}";
  return o.str();
}

static LaunchCfg launch_from_json(const json::Object& so) {
  LaunchCfg l;
  l.tile_m = static_cast<int32_t>(json::as_int(json::at(so, "tile_m"), "tile_m"));
  l.cluster = static_cast<int32_t>(json::as_int(json::at(so, "cluster"), "cluster"));
  l.bn = static_cast<int32_t>(json::as_int(json::at(so, "bn"), "bn"));
  l.stages = static_cast<int32_t>(json::as_int(json::at(so, "stages"), "stages"));
  if (auto it = so.find("path"); it != so.end()) l.path = static_cast<int32_t>(json::as_int(it->second, "path"));
  return l;
}

std::string TilingTable::to_json() const {
  std::ostringstream o;
  o << "{\n  \"default\": " << cfg_json(default_) << ",\n";
  if (has_default_sm100_) o << "  \"default_sm100\": " << launch_json(default_sm100_) << ",\n";
  else if (heuristic_default_) o << "  \"default_sm100\": \"heuristic\",\n";
  o << "  \"entries\": [";
  bool first = true;
  for (const auto& [k, e] : entries_) {
    o << (first ? "\n" : ",\n");
    first = false;
    o << "    {\"config\": " << cfg_json(e.config) << ", \"k\": " << k.k << ", \"m_bucket\": "
      << k.m_bucket << ", \"n\": " << k.n << ", \"ns\": " << e.measured_ns;
    if (e.has_sm100) o << ", \"sm100\": " << launch_json(e.sm100);
    o << "}";
  }
  o << (first ? "]\n}\n" : "\n  ]\n}\n");
  return o.str();
}

TilingTable TilingTable::from_json(const std::string& text) {
  const json::Value root = json::Parser(text).parse();
  if (!root.is_obj()) fail(ATMM_ERR_IO, "tiling table json: root must be an object");
  TilingTable t(cfg_from_json(json::at(root.obj(), "default")));
  if (auto it = root.obj().find("default_sm100"); it != root.obj().end() && it->second.is_obj()) {
    const LaunchCfg dl = launch_from_json(it->second.obj());
    t.set_default(t.default_config(), &dl);
  } else if (it != root.obj().end() && std::holds_alternative<std::string>(it->second.v) &&
             std::get<std::string>(it->second.v) == "heuristic") {
    const LaunchCfg heur{0, 0, 0, 0, 0};
    t.set_default(t.default_config(), &heur);
  }
  const json::Value& ents = json::at(root.obj(), "entries");
  if (!ents.is_arr()) fail(ATMM_ERR_IO, "tiling table json: entries must be an array");
  for (const json::Value& ev : ents.arr()) {
    if (!ev.is_obj()) fail(ATMM_ERR_IO, "tiling table json: entry must be an object");
    const json::Object& e = ev.obj();
    ShapeKey key{static_cast<int32_t>(json::as_int(json::at(e, "m_bucket"), "m_bucket")),
                 static_cast<int32_t>(json::as_int(json::at(e, "k"), "k")),
                 static_cast<int32_t>(json::as_int(json::at(e, "n"), "n"))};
    const TilingConfig cfg = cfg_from_json(json::at(e, "config"));
    const int64_t ns = json::as_int(json::at(e, "ns"), "ns");
    LaunchCfg l;
    const LaunchCfg* lp = nullptr;
    if (auto it = e.find("sm100"); it != e.end() && it->second.is_obj()) {
      l = launch_from_json(it->second.obj());
      lp = &l;
    }
    t.insert(key, cfg, ns, lp);
  }
  return t;
}

// ------------------------------------------------------------ planner ---

// plan_batch (batch.hpp:28-42): groups rows by adapter id in a std::map
// (ascending id), each group keeping batch order.  Counting pass over the
// sorted distinct ids; O(n log S).
BatchPlan plan_batch(const int32_t* assignment, int64_t n) {
  if (n <= 0 || assignment == nullptr) fail(ATMM_ERR_CONFIG, "plan_batch needs a nonempty assignment");
  std::map<int32_t, int64_t> counts;
  for (int64_t i = 0; i < n; ++i) counts[assignment[i]] += 1;
  BatchPlan p;
  p.seg_adapter.reserve(counts.size());
  p.seg_offsets.reserve(counts.size() + 1);
  std::map<int32_t, int64_t> cursor;
  int64_t pos = 0;
  for (const auto& [id, c] : counts) {
    p.seg_adapter.push_back(id);
    p.seg_offsets.push_back(pos);
    cursor[id] = pos;
    pos += c;
  }
  p.seg_offsets.push_back(pos);
  p.row_index.assign(static_cast<size_t>(n), 0);
  for (int64_t i = 0; i < n; ++i) p.row_index[static_cast<size_t>(cursor[assignment[i]]++)] = i;
  return p;
}

// ---- reference fixture I/O ----
std::vector<float> load_matrix_f32(const std::string& path, int64_t& rows, int64_t& cols) {
  std::ifstream in(path, std::ios::binary);
  if (!in) fail(ATMM_ERR_IO, "cannot open for read: " + path);
  uint32_t r = 0, c = 0;
  uint8_t width = 0;
  in.read(reinterpret_cast<char*>(&r), 4);
  in.read(reinterpret_cast<char*>(&c), 4);
  in.read(reinterpret_cast<char*>(&width), 1);
  if (!in) fail(ATMM_ERR_IO, "truncated header: " + path);
  if (width != sizeof(float)) {
    fail(ATMM_ERR_IO, "scalar width mismatch in " + path + ": file has " + std::to_string(width) + ", expected 4");
  }
  rows = r;
  cols = c;
  std::vector<float> out(static_cast<size_t>(r) * c);
  in.read(reinterpret_cast<char*>(out.data()), static_cast<std::streamsize>(out.size() * sizeof(float)));
  if (!in) fail(ATMM_ERR_IO, "truncated payload: " + path);
  return out;
}

void save_matrix_f32(const std::string& path, int64_t rows, int64_t cols, const float* data) {
  if (rows < 0 || cols < 0 || rows > 0xffffffffLL || cols > 0xffffffffLL) fail(ATMM_ERR_SHAPE, "matrix too large for the u32 header");
  std::ofstream out(path, std::ios::binary);
  if (!out) fail(ATMM_ERR_IO, "cannot open for write: " + path);
  const uint32_t r = static_cast<uint32_t>(rows), c = static_cast<uint32_t>(cols);
  const uint8_t width = sizeof(float);
  out.write(reinterpret_cast<const char*>(&r), 4);
  out.write(reinterpret_cast<const char*>(&c), 4);
  out.write(reinterpret_cast<const char*>(&width), 1);
  out.write(reinterpret_cast<const char*>(data), static_cast<std::streamsize>(sizeof(float) * rows * cols));
  if (!out) fail(ATMM_ERR_IO, "short write: " + path);
}

FixtureManifest read_fixture_manifest(const std::string& dir) {
  std::ifstream in(dir + "/manifest.json");
  if (!in) fail(ATMM_ERR_IO, "cannot read manifest in " + dir);
  std::stringstream ss;
  ss << in.rdbuf();
  const std::string text = ss.str();
  json::Value root;
  try {
    root = json::Parser(text).parse();
  } catch (const Failure& e) {
    fail(ATMM_ERR_IO, std::string("bad manifest: ") + e.what());
  }
  if (!root.is_obj()) fail(ATMM_ERR_IO, "bad manifest: root must be an object");
  auto need = [&](const json::Object& o, const char* key) -> const json::Value& {
    auto it = o.find(key);
    if (it == o.end()) fail(ATMM_ERR_IO, std::string("bad manifest: missing key '") + key + "'");
    return it->second;
  };
  auto as_str = [](const json::Value& v) -> std::string {
    if (!std::holds_alternative<std::string>(v.v)) fail(ATMM_ERR_IO, "bad manifest: file names must be strings");
    return std::get<std::string>(v.v);
  };
  FixtureManifest m;
  m.num_layers = json::as_int(need(root.obj(), "num_layers"), "num_layers");
  m.hidden_dim = json::as_int(need(root.obj(), "hidden_dim"), "hidden_dim");
  const json::Value& ads = need(root.obj(), "adapters");
  if (!ads.is_arr()) fail(ATMM_ERR_IO, "bad manifest: adapters must be an array");
  for (const json::Value& av : ads.arr()) {
    if (!av.is_obj()) fail(ATMM_ERR_IO, "bad manifest: adapter entries must be objects");
    FixtureAdapter a;
    a.id = static_cast<int32_t>(json::as_int(need(av.obj(), "id"), "adapter id"));
    a.rank = json::as_int(need(av.obj(), "rank"), "adapter rank");
    for (const char* key : {"down", "up"}) {
      const json::Value& files = need(av.obj(), key);
      if (!files.is_arr()) fail(ATMM_ERR_IO, std::string("bad manifest: adapter ") + key + " must be an array");
      for (const json::Value& f : files.arr()) (key[0] == 'd' ? a.down : a.up).push_back(as_str(f));
    }
    if (static_cast<int64_t>(a.down.size()) != m.num_layers || static_cast<int64_t>(a.up.size()) != m.num_layers) {
      fail(ATMM_ERR_IO, "manifest lists wrong layer count for adapter " + std::to_string(a.id));
    }
    m.adapters.push_back(std::move(a));
  }
  return m;
}

}  // namespace atmm

// =========================================================================
// C ABI (host-only part)
// =========================================================================
using namespace atmm;

extern "C" {

int atmm_matrix_save(const char* path, int64_t rows, int64_t cols, const float* data) {
  return guarded([&] {
    if (!path || (!data && rows * cols > 0)) fail(ATMM_ERR_CONFIG, "null path or data");
    save_matrix_f32(path, rows, cols, data);
  });
}

int atmm_fixture_info(const char* dir, int64_t* num_layers, int64_t* hidden_dim, int64_t* num_adapters,
                      int32_t* ids, int64_t* ranks, int64_t capacity) {
  return guarded([&] {
    if (!dir) fail(ATMM_ERR_CONFIG, "null directory");
    const FixtureManifest m = read_fixture_manifest(dir);
    if (num_layers) *num_layers = m.num_layers;
    if (hidden_dim) *hidden_dim = m.hidden_dim;
    if (num_adapters) *num_adapters = static_cast<int64_t>(m.adapters.size());
    for (size_t i = 0; i < m.adapters.size() && static_cast<int64_t>(i) < capacity; ++i) {
      if (ids) ids[i] = m.adapters[i].id;
      if (ranks) ranks[i] = m.adapters[i].rank;
    }
  });
}

int atmm_matrix_load(const char* path, int64_t* rows, int64_t* cols, float* out, int64_t capacity) {
  return guarded([&] {
    if (!path || !rows || !cols) fail(ATMM_ERR_CONFIG, "null path or dims");
    int64_t r = 0, c = 0;
    std::vector<float> m = load_matrix_f32(path, r, c);
    *rows = r;
    *cols = c;
    if (out) {
      if (capacity < r * c) fail(ATMM_ERR_SHAPE, "output buffer too small");
      std::copy(m.begin(), m.end(), out);
    }
  });
}

const char* atmm_last_error(void) { return g_last_error.c_str(); }
uint64_t atmm_flops_read(void) { return g_flops; }
void atmm_flops_reset(void) { g_flops = 0; }

int atmm_bypass_flops(const int32_t* assignment, int64_t n, const int32_t* adapter_ids, const int64_t* adapter_ranks,
                      int64_t num_adapters, int64_t d_in, int64_t d_out, uint64_t* flops) {
  return guarded([&] {
    if (!flops || (num_adapters > 0 && (!adapter_ids || !adapter_ranks))) fail(ATMM_ERR_CONFIG, "null argument");
    if (d_in < 1 || d_out < 1) fail(ATMM_ERR_SHAPE, "dimensions must be >= 1");
    std::map<int32_t, int64_t> rank_of;
    for (int64_t i = 0; i < num_adapters; ++i) rank_of[adapter_ids[i]] = adapter_ranks[i];
    const BatchPlan bp = plan_batch(assignment, n);
    uint64_t f = 0;
    for (size_t s = 0; s < bp.seg_adapter.size(); ++s) {
      auto it = rank_of.find(bp.seg_adapter[s]);
      if (it == rank_of.end()) fail(ATMM_ERR_UNKNOWN_ADAPTER, "unknown adapter id " + std::to_string(bp.seg_adapter[s]));
      const uint64_t ns = static_cast<uint64_t>(bp.seg_offsets[s + 1] - bp.seg_offsets[s]);
      // shrink 2*ns*d_in*r + expand 2*ns*r*d_out (batch.hpp:70-73 via atmm.hpp:123)
      f += 2ull * ns * static_cast<uint64_t>(it->second) * static_cast<uint64_t>(d_in + d_out);
    }
    *flops = f;
  });
}
int atmm_abi_version(void) { return ATMM_ABI_VERSION; }

int atmm_plan_batch(const int32_t* assignment, int64_t n, int32_t* seg_adapter,
                    int64_t* seg_offsets, int64_t* row_index, int64_t* num_segments) {
  return guarded([&] {
    const BatchPlan p = plan_batch(assignment, n);
    const size_t S = p.seg_adapter.size();
    if (seg_adapter) std::copy(p.seg_adapter.begin(), p.seg_adapter.end(), seg_adapter);
    if (seg_offsets) std::copy(p.seg_offsets.begin(), p.seg_offsets.end(), seg_offsets);
    if (row_index) std::copy(p.row_index.begin(), p.row_index.end(), row_index);
    if (num_segments) *num_segments = static_cast<int64_t>(S);
  });
}

int atmm_config_valid(const int32_t cfg[6]) {
  if (!cfg) return 0;
  TilingConfig c;
  std::copy(cfg, cfg + 6, c.e.begin());
  return c.structurally_valid() ? 1 : 0;
}

int atmm_m_bucket_of(int64_t m) { return m_bucket_of(m); }

int atmm_table_create(const int32_t* default_cfg, atmm_table** out) {
  return guarded([&] {
    if (!out) fail(ATMM_ERR_CONFIG, "null output");
    auto t = std::make_unique<atmm_table>();
    if (default_cfg) {
      TilingConfig c;
      std::copy(default_cfg, default_cfg + 6, c.e.begin());
      t->t = TilingTable(c);
    }
    *out = t.release();
  });
}

void atmm_table_destroy(atmm_table* t) { delete t; }

int atmm_table_insert(atmm_table* t, int32_t m_bucket, int32_t k, int32_t n, const int32_t cfg[6],
                      int64_t measured_ns, const int32_t* sm100) {
  return guarded([&] {
    if (!t || !cfg) fail(ATMM_ERR_CONFIG, "null table or config");
    TilingConfig c;
    std::copy(cfg, cfg + 6, c.e.begin());
    LaunchCfg l;
    if (sm100) l = launch_from_ints(sm100);
    t->t.insert(ShapeKey{m_bucket, k, n}, c, measured_ns, sm100 ? &l : nullptr);
  });
}

int atmm_table_set_default(atmm_table* t, const int32_t cfg[6], const int32_t* sm100) {
  return guarded([&] {
    if (!t || !cfg) fail(ATMM_ERR_CONFIG, "null table or config");
    TilingConfig c;
    std::copy(cfg, cfg + 6, c.e.begin());
    LaunchCfg l;
    if (sm100) l = launch_from_ints(sm100);
    t->t.set_default(c, sm100 ? &l : nullptr);
  });
}

int atmm_table_lookup(const atmm_table* t, int64_t m, int64_t k, int64_t n, int32_t cfg_out[6]) {
  return guarded([&] {
    if (!t || !cfg_out) fail(ATMM_ERR_CONFIG, "null table or output");
    const TilingConfig c = t->t.lookup(m, k, n);
    std::copy(c.e.begin(), c.e.end(), cfg_out);
  });
}

int atmm_table_size(const atmm_table* t, int64_t* size) {
  return guarded([&] {
    if (!t || !size) fail(ATMM_ERR_CONFIG, "null table or output");
    *size = static_cast<int64_t>(t->t.entries().size());
  });
}

int atmm_table_find(const atmm_table* t, int64_t m, int64_t k, int64_t n, int32_t launch_out[5], int* found) {
  return guarded([&] {
    if (!t || !launch_out || !found) fail(ATMM_ERR_CONFIG, "null table or output");
    const TableEntry* e = t->t.find(m, k, n);
    *found = e ? 1 : 0;
    if (e) launch_to_ints(e->has_sm100 ? e->sm100 : launch_from_config(e->config, k), launch_out);
  });
}

int atmm_table_resolve_launch(const atmm_table* t, int64_t m, int64_t d_in, int64_t rank,
                              int64_t d_out, int32_t launch_out[4]) {
  return guarded([&] {
    if (!launch_out) fail(ATMM_ERR_CONFIG, "null output");
    const LaunchCfg l = t ? t->t.resolve_launch(m, d_in, rank, d_out) : heuristic_launch(m, d_in, rank, d_out);
    launch_to_ints(l, launch_out);
  });
}

int atmm_table_save(const atmm_table* t, const char* path) {
  return guarded([&] {
    if (!t || !path) fail(ATMM_ERR_CONFIG, "null table or path");
    std::ofstream out(path);
    if (!out) fail(ATMM_ERR_IO, std::string("cannot open for write: ") + path);
    out << t->t.to_json();
    if (!out) fail(ATMM_ERR_IO, std::string("short write: ") + path);
  });
}

int atmm_table_load(const char* path, atmm_table** out) {
  return guarded([&] {
    if (!path || !out) fail(ATMM_ERR_CONFIG, "null path or output");
    std::ifstream in(path);
    if (!in) fail(ATMM_ERR_IO, std::string("cannot open for read: ") + path);
    std::stringstream ss;
    ss << in.rdbuf();
    auto t = std::make_unique<atmm_table>();
    t->t = TilingTable::from_json(ss.str());
    *out = t.release();
  });
}

static int copy_configs(const std::vector<TilingConfig>& v, int32_t* out, size_t cap, size_t* count) {
  if (count) *count = v.size();
  for (size_t i = 0; i < v.size() && i < cap && out; ++i) std::copy(v[i].e.begin(), v[i].e.end(), out + 6 * i);
  return ATMM_OK;
}

int atmm_candidate_configs(size_t budget, size_t width, int32_t* out, size_t cap, size_t* count) {
  return guarded([&] { copy_configs(candidate_configs(budget, width), out, cap, count); });
}

int atmm_default_candidates(size_t budget, size_t width, int32_t* out, size_t cap, size_t* count) {
  return guarded([&] { copy_configs(default_candidates(budget, width), out, cap, count); });
}

// LPT over whole segments: segments sorted by cost
// descending (ties: ascending adapter id), each placed on the currently
// least-loaded shard (ties: lowest shard index).
// The reference TilingConfig recorded beside a B200 launch (the JSON
// "config" field, read by the reference's TilingTable::load): outer_m = tile
// rows, outer_n = expand chunk, outer_k = K slice per CTA (powers of two).
static TilingConfig config_of_launch(const LaunchCfg& l, int64_t d_in) {
  auto pow2_ceil = [](int64_t v) {
    int64_t p = 16;
    while (p < v) p <<= 1;
    return p;
  };
  const int64_t om = pow2_ceil(l.tile_m), on = pow2_ceil(l.bn);
  int64_t ok = 64;
  while (ok * 2 * l.cluster <= d_in) ok <<= 1;
  return TilingConfig{{static_cast<int32_t>(om), static_cast<int32_t>(on), static_cast<int32_t>(ok),
                       static_cast<int32_t>(std::min<int64_t>(om, 128)), 16, 64}};
}

// The selection half of tiling_search (atmm.hpp:293-329) over a score grid:
// per-shape argmin (ties to the lexicographically smallest launch; shapes
// whose candidates all failed -- INT64_MAX -- are omitted and reported), the
// most frequent winner as the default.  Two grid shapes can share a table key
// (m_bucket, d_in, rank) while differing in batch size (segments): the
// reference keeps the faster measurement of one GEMM shape; here the entry
// measured on the larger batch (segments x m rows) is kept -- a bigger batch
// is not comparable by time, and it is the loaded serving case -- with the
// faster one winning between equal batches.
int atmm_table_from_scores(const atmm_tune_shape* shapes, int64_t num_shapes, const int32_t* launches,
                           int64_t num_launches, const int64_t* scores, atmm_table** out, char* failures,
                           size_t failures_cap) {
  return guarded([&] {
    if (!shapes || !launches || !scores || !out || num_shapes < 1 || num_launches < 1) {
      fail(ATMM_ERR_CONFIG, "table_from_scores needs a nonempty grid, candidates and scores");
    }
    std::vector<LaunchCfg> cands;
    for (int64_t i = 0; i < num_launches; ++i) {
      cands.push_back(launch_from_ints(launches + 5 * i));
      validate_launch(cands.back());
    }
    auto table = std::make_unique<atmm_table>();
    std::map<LaunchCfg, int> wins;
    std::map<LaunchCfg, TilingConfig> cfg_of;
    std::map<ShapeKey, int64_t> batch_of;  // rows of the batch each entry was measured on
    std::string fails;
    constexpr int64_t kFailed = std::numeric_limits<int64_t>::max();
    for (int64_t si = 0; si < num_shapes; ++si) {
      const int64_t* sc = scores + si * num_launches;
      int64_t best = -1;
      for (int64_t ci = 0; ci < num_launches; ++ci) {
        if (sc[ci] == kFailed) continue;
        if (best < 0 || sc[ci] < sc[best] || (sc[ci] == sc[best] && cands[ci] < cands[best])) best = ci;
      }
      const atmm_tune_shape& sh = shapes[si];
      if (best < 0) {
        fails += "shape " + std::to_string(sh.segments) + "x" + std::to_string(sh.m) + " rows, d " +
                 std::to_string(sh.d_in) + ", r " + std::to_string(sh.rank) + ": all candidates failed, omitted\n";
        continue;
      }
      const LaunchCfg& lc = cands[static_cast<size_t>(best)];
      const ShapeKey key{m_bucket_of(sh.m), static_cast<int32_t>(sh.d_in), static_cast<int32_t>(sh.rank)};
      const TilingConfig tc = config_of_launch(lc, sh.d_in);
      auto it = table->t.entries().find(key);
      const int64_t rows = sh.m * sh.segments;
      auto bt = batch_of.find(key);
      if (it == table->t.entries().end() || rows > bt->second ||
          (rows == bt->second && sc[best] < it->second.measured_ns)) {
        table->t.insert(key, tc, sc[best], &lc);
        batch_of[key] = rows;
      }
      wins[lc] += 1;
      cfg_of[lc] = tc;
    }
    if (!wins.empty()) {
      const LaunchCfg* top = nullptr;
      int top_count = -1;
      for (const auto& [lc, count] : wins) {  // map order: ties go to the lexicographically smallest
        if (count > top_count) {
          top = &lc;
          top_count = count;
        }
      }
      table->t.set_default(cfg_of[*top], top);
    }
    if (failures && failures_cap > 0) {
      std::strncpy(failures, fails.c_str(), failures_cap - 1);
      failures[failures_cap - 1] = 0;
    }
    *out = table.release();
  });
}

int atmm_shard_rows(const int32_t* assignment, int64_t n, const int32_t* adapter_ids,
                    const int64_t* adapter_ranks, int64_t num_adapters, int64_t d_in, int64_t d_out,
                    int32_t num_shards, int32_t* shard_of_row) {
  return guarded([&] {
    if (num_shards < 1) fail(ATMM_ERR_CONFIG, "num_shards must be >= 1");
    if (!shard_of_row) fail(ATMM_ERR_CONFIG, "null output");
    const BatchPlan p = plan_batch(assignment, n);
    const size_t S = p.seg_adapter.size();
    std::vector<double> cost(S);
    for (size_t s = 0; s < S; ++s) {
      int64_t r = -1;
      for (int64_t a = 0; a < num_adapters; ++a) {
        if (adapter_ids[a] == p.seg_adapter[s]) {
          r = adapter_ranks[a];
          break;
        }
      }
      if (r < 0) fail(ATMM_ERR_UNKNOWN_ADAPTER, "unknown adapter id " + std::to_string(p.seg_adapter[s]));
      const double rows = static_cast<double>(p.seg_offsets[s + 1] - p.seg_offsets[s]);
      // bytes: X rows read, Y rows read+write (bf16), factors once.
      cost[s] = rows * (2.0 * d_in + 4.0 * d_out) + 2.0 * r * (d_in + d_out);
    }
    std::vector<size_t> order(S);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return cost[a] > cost[b]; });
    std::vector<double> load(static_cast<size_t>(num_shards), 0.0);
    for (size_t s : order) {
      size_t best = 0;
      for (size_t g = 1; g < load.size(); ++g) {
        if (load[g] < load[best]) best = g;
      }
      load[best] += cost[s];
      for (int64_t i = p.seg_offsets[s]; i < p.seg_offsets[s + 1]; ++i) {
        shard_of_row[p.row_index[static_cast<size_t>(i)]] = static_cast<int32_t>(best);
      }
    }
  });
}

}  // extern "C"
