// ref_driver.cpp -- C-ABI shim over the UNMODIFIED reference headers.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file
// against /root/reference/proj/include (read in place, never copied) into
// oracle/_ref/libloraserve_ref.so.  It serves two purposes:
//   1. pin the C restatement (oracle/atmm_oracle.c) against the reference's
//      own arithmetic on identical inputs (tests/test_oracle.py, and the
//      fixture generator tests/golden/make_golden.py);
//   2. the CPU baseline arm of bench.py (`--impl reference`), which times the
//      reference's run_bypass + add_inplace / delta_w + add_inplace.
// No reference source is reproduced here; every entry point just forwards to
// the loraserve:: function named in its comment.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <span>
#include <vector>

#include "loraserve/atmm.hpp"
#include "loraserve/batch.hpp"
#include "loraserve/matrix.hpp"
#include "loraserve/model.hpp"
#include "loraserve/model_io.hpp"
#include "loraserve/random.hpp"
#include "loraserve/serving.hpp"
#include "loraserve/tiling.hpp"

using namespace loraserve;

namespace {

// Exception class -> status code (the mapping the product's C ABI uses too).
int status_of(const std::exception& e) {
  if (dynamic_cast<const ShapeError*>(&e)) return 1;
  if (dynamic_cast<const ConfigError*>(&e)) return 2;
  if (dynamic_cast<const ModeError*>(&e)) return 3;
  if (dynamic_cast<const ParseError*>(&e)) return 5;
  if (dynamic_cast<const IoError*>(&e)) return 4;
  if (dynamic_cast<const UnknownAdapterError*>(&e)) return 6;
  return 9;
}

TilingConfig cfg_of(const int32_t* c) { return TilingConfig{c[0], c[1], c[2], c[3], c[4], c[5]}; }

}  // namespace

extern "C" {

// ---- RNG (random.hpp) ----------------------------------------------------
void* ref_rng_new(uint64_t seed) { return new Rng(seed); }
void ref_rng_free(void* r) { delete static_cast<Rng*>(r); }
uint64_t ref_rng_next(void* r) { return (*static_cast<Rng*>(r))(); }
void ref_fill_uniform(void* r, float* out, size_t count, float lo, float hi) {
  MatSpan<float> m(out, 1, count);
  fill_uniform<float>(m, *static_cast<Rng*>(r), lo, hi);
}
void ref_seeded_shuffle_u64(void* r, uint64_t* v, size_t n) {
  std::vector<uint64_t> vec(v, v + n);
  seeded_shuffle(vec, *static_cast<Rng*>(r));
  std::memcpy(v, vec.data(), n * sizeof(uint64_t));
}
// LoraAdapter::random -> factors copied out ([L][d*r], [L][r*d]).
int ref_adapter_random(int id, size_t L, size_t d, size_t r, uint64_t seed, float* down,
                       float* up) {
  try {
    LoraAdapter a = LoraAdapter::random(id, L, d, r, seed);
    for (size_t l = 0; l < L; ++l) {
      std::memcpy(down + l * d * r, a.down(l).data, d * r * sizeof(float));
      std::memcpy(up + l * r * d, a.up(l).data, r * d * sizeof(float));
    }
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}
// BaseModel::random -> layer weights copied out ([L][d*d]).
int ref_model_random(size_t L, size_t d, size_t V, uint64_t seed, float* w) {
  try {
    BaseModel m = BaseModel::random(L, d, V, seed);
    for (size_t l = 0; l < L; ++l) std::memcpy(w + l * d * d, m.layer(l).data, d * d * 4);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// ---- matrix core ---------------------------------------------------------
int ref_gemm_reference(const float* a, const float* b, float* c, size_t m, size_t k, size_t n) {
  try {
    Matrix<float> out = gemm_reference<float>(ConstMatSpan<float>(a, m, k),
                                              ConstMatSpan<float>(b, k, n));
    std::memcpy(c, out.data(), m * n * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}
// atmm_multiply_into with an explicit config (atmm.hpp:112).
int ref_atmm_multiply(const float* a, size_t a_rows, size_t a_cols, const float* b,
                      size_t b_rows, size_t b_cols, float* c, const int32_t* cfg) {
  try {
    atmm_multiply_into<float>(ConstMatSpan<float>(a, a_rows, a_cols),
                              ConstMatSpan<float>(b, b_rows, b_cols),
                              MatSpan<float>(c, a_rows, b_cols), cfg_of(cfg));
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}
void ref_add_inplace(float* t, const float* d, size_t count) {
  add_inplace<float>(MatSpan<float>(t, 1, count), ConstMatSpan<float>(d, 1, count));
}
void ref_sub_inplace(float* t, const float* d, size_t count) {
  sub_inplace<float>(MatSpan<float>(t, 1, count), ConstMatSpan<float>(d, 1, count));
}

// ---- tiling (tiling.hpp) -------------------------------------------------
int ref_m_bucket_of(uint64_t m) { return m_bucket_of(m); }
int ref_config_valid(const int32_t* cfg) { return cfg_of(cfg).structurally_valid() ? 1 : 0; }
int ref_candidate_count(size_t budget, size_t width) {
  try {
    return static_cast<int>(candidate_configs(budget, width).size());
  } catch (const std::exception& e) {
    return -status_of(e);
  }
}
// Fills out[count*6]; returns number written.
int ref_candidate_configs(size_t budget, size_t width, int32_t* out, size_t cap) {
  try {
    auto v = candidate_configs(budget, width);
    size_t i = 0;
    for (; i < v.size() && i < cap; ++i) {
      auto e = v[i].edges();
      for (int j = 0; j < 6; ++j) out[i * 6 + j] = e[j];
    }
    return static_cast<int>(i);
  } catch (const std::exception& e) {
    return -status_of(e);
  }
}
int ref_default_candidates(size_t budget, size_t width, int32_t* out, size_t cap) {
  try {
    auto v = default_candidates(budget, width);
    size_t i = 0;
    for (; i < v.size() && i < cap; ++i) {
      auto e = v[i].edges();
      for (int j = 0; j < 6; ++j) out[i * 6 + j] = e[j];
    }
    return static_cast<int>(i);
  } catch (const std::exception& e) {
    return -status_of(e);
  }
}
// TilingTable built from (keys, configs, ns) + default, then lookup(m,k,n).
int ref_table_lookup(const int32_t* keys, const int32_t* configs, size_t num, const int32_t* dflt,
                     uint64_t m, uint64_t k, uint64_t n, int32_t* out) {
  try {
    TilingTable t(cfg_of(dflt));
    for (size_t i = 0; i < num; ++i) {
      t.insert(ShapeKey{keys[3 * i], keys[3 * i + 1], keys[3 * i + 2]}, cfg_of(configs + 6 * i),
               1000);
    }
    auto e = t.lookup(m, k, n).edges();
    for (int j = 0; j < 6; ++j) out[j] = e[j];
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}
// TilingTable::load(path) -> lookup (used to check the product's JSON output
// is loadable by the reference and resolves identically).
int ref_table_load_lookup(const char* path, uint64_t m, uint64_t k, uint64_t n, int32_t* out) {
  try {
    TilingTable t = TilingTable::load(path);
    auto e = t.lookup(m, k, n).edges();
    for (int j = 0; j < 6; ++j) out[j] = e[j];
    return static_cast<int>(t.size()) >= 0 ? 0 : 9;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}
int ref_table_save(const int32_t* keys, const int32_t* configs, const int64_t* ns, size_t num,
                   const int32_t* dflt, const char* path) {
  try {
    TilingTable t(cfg_of(dflt));
    for (size_t i = 0; i < num; ++i) {
      t.insert(ShapeKey{keys[3 * i], keys[3 * i + 1], keys[3 * i + 2]}, cfg_of(configs + 6 * i),
               ns[i]);
    }
    t.save(path);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// ---- batch engine (batch.hpp) --------------------------------------------
// plan_batch -> CSR (seg_adapter[S], seg_offsets[S+1], row_index[n]); returns
// S, or -status on exception.
long ref_plan_batch(const int32_t* assignment, size_t n, int32_t* seg_adapter,
                    int64_t* seg_offsets, int64_t* row_index) {
  try {
    std::vector<int> a(assignment, assignment + n);
    BatchPlan p = plan_batch(std::span<const int>(a.data(), a.size()));
    int64_t pos = 0;
    for (size_t s = 0; s < p.segments.size(); ++s) {
      seg_adapter[s] = p.segments[s].adapter_id;
      seg_offsets[s] = pos;
      for (size_t r : p.segments[s].rows) row_index[pos++] = static_cast<int64_t>(r);
    }
    seg_offsets[p.segments.size()] = pos;
    return static_cast<long>(p.segments.size());
  } catch (const std::exception& e) {
    return -status_of(e);
  }
}

// A reference-side serving context: the AdapterSet is built once (outside
// any timed region) from caller factors; layer count 1.
struct RefCtx {
  AdapterSet adapters;
  TilingTable table;
  size_t d = 0;
};

void* ref_ctx_new(size_t d, size_t num_adapters, const int32_t* ids, const int64_t* ranks,
                  const float* const* downs, const float* const* ups) {
  try {
    auto ctx = std::make_unique<RefCtx>();
    ctx->d = d;
    for (size_t i = 0; i < num_adapters; ++i) {
      const size_t r = static_cast<size_t>(ranks[i]);
      std::vector<Matrix<float>> dn, u;
      Matrix<float> dm(d, r), um(r, d);
      std::memcpy(dm.data(), downs[i], d * r * sizeof(float));
      std::memcpy(um.data(), ups[i], r * d * sizeof(float));
      dn.push_back(std::move(dm));
      u.push_back(std::move(um));
      ctx->adapters.emplace(ids[i], LoraAdapter(ids[i], 1, d, r, std::move(dn), std::move(u)));
    }
    return ctx.release();
  } catch (const std::exception&) {
    return nullptr;
  }
}
void ref_ctx_free(void* c) { delete static_cast<RefCtx*>(c); }

// run_bypass (batch.hpp:48) -> out (n x d, fresh bypass).
int ref_ctx_run_bypass(void* c, const float* x, size_t n, const int32_t* assignment, float* out) {
  auto* ctx = static_cast<RefCtx*>(c);
  try {
    std::vector<int> a(assignment, assignment + n);
    BatchPlan plan = plan_batch(std::span<const int>(a.data(), a.size()));
    Matrix<float> bypass =
        run_bypass(ConstMatSpan<float>(x, n, ctx->d), plan, ctx->adapters, 0, ctx->table);
    std::memcpy(out, bypass.data(), n * ctx->d * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// The unmerged-forward residual site (model.hpp:239-241): y += run_bypass(x).
// Times plan_batch + run_bypass + add_inplace; returns ns via *elapsed_ns.
int ref_ctx_bypass_residual(void* c, const float* x, size_t n, const int32_t* assignment,
                            float* y, int64_t* elapsed_ns) {
  auto* ctx = static_cast<RefCtx*>(c);
  try {
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<int> a(assignment, assignment + n);
    BatchPlan plan = plan_batch(std::span<const int>(a.data(), a.size()));
    Matrix<float> bypass =
        run_bypass(ConstMatSpan<float>(x, n, ctx->d), plan, ctx->adapters, 0, ctx->table);
    add_inplace<float>(MatSpan<float>(y, n, ctx->d), bypass);
    const auto t1 = std::chrono::steady_clock::now();
    if (elapsed_ns) *elapsed_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// delta_w for rectangular factors through atmm_multiply_into at the lookup
// the reference uses (model.hpp:120-125), then add_inplace / sub_inplace
// (model.hpp:157-158,180-181).  sign >= 0 merges, < 0 unmerges.
int ref_merge_rect(float* w, size_t d_in, size_t r, size_t d_out, const float* down,
                   const float* up, int sign, float* scratch, int64_t* elapsed_ns) {
  try {
    TilingTable table;
    const auto t0 = std::chrono::steady_clock::now();
    atmm_multiply_into<float>(ConstMatSpan<float>(down, d_in, r), ConstMatSpan<float>(up, r, d_out),
                              MatSpan<float>(scratch, d_in, d_out), table.lookup(d_in, r, d_out));
    if (sign >= 0) {
      add_inplace<float>(MatSpan<float>(w, d_in, d_out), ConstMatSpan<float>(scratch, d_in, d_out));
    } else {
      sub_inplace<float>(MatSpan<float>(w, d_in, d_out), ConstMatSpan<float>(scratch, d_in, d_out));
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (elapsed_ns) *elapsed_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// Square merge/unmerge through BaseModel + ModelState (model.hpp:144-188),
// including the ModeError contract.  w is [L][d*d] in/out.
int ref_model_merge_cycle(float* w, size_t L, size_t d, size_t r, const float* down,
                          const float* up, int cycles) {
  try {
    BaseModel model(L, d, 2);
    for (size_t l = 0; l < L; ++l) std::memcpy(model.layer(l).data, w + l * d * d, d * d * 4);
    std::vector<Matrix<float>> dn, u;
    for (size_t l = 0; l < L; ++l) {
      Matrix<float> dm(d, r), um(r, d);
      std::memcpy(dm.data(), down + l * d * r, d * r * 4);
      std::memcpy(um.data(), up + l * r * d, r * d * 4);
      dn.push_back(std::move(dm));
      u.push_back(std::move(um));
    }
    LoraAdapter a(1, L, d, r, std::move(dn), std::move(u));
    TilingTable table;
    ModelState state;
    for (int c = 0; c < cycles; ++c) {
      merge(model, state, a, table);
      unmerge(model, state, a, table);
    }
    if (cycles == 0) merge(model, state, a, table);  // merged state out
    for (size_t l = 0; l < L; ++l) std::memcpy(w + l * d * d, model.layer(l).data, d * d * 4);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

// ---- fixture I/O (matrix.hpp:183-218, model_io.hpp:25-114) ----
// save_matrix<float> of a rows x cols matrix; 0 = ok, 1 = IoError.
int ref_save_matrix(const char* path, size_t rows, size_t cols, const float* data) {
  try {
    save_matrix<float>(ConstMatSpan<float>{data, rows, cols}, path);
    return 0;
  } catch (const Error&) {
    return 1;
  }
}
// save_model_fixture of a random model (seed) with the given adapters
// (ids, ranks, factors [L][d x r] / [L][r x d] concatenated per adapter).
int ref_save_fixture(const char* dir, size_t L, size_t d, size_t V, uint64_t seed, size_t num_adapters,
                     const int32_t* ids, const int64_t* ranks, const float* factors) {
  try {
    BaseModel model = BaseModel::random(L, d, V, seed);
    AdapterSet set;
    const float* f = factors;
    for (size_t a = 0; a < num_adapters; ++a) {
      const size_t r = static_cast<size_t>(ranks[a]);
      std::vector<Matrix<float>> down, up;
      for (size_t l = 0; l < L; ++l) {
        Matrix<float> m(d, r);
        std::copy(f, f + d * r, m.data());
        f += d * r;
        down.push_back(std::move(m));
      }
      for (size_t l = 0; l < L; ++l) {
        Matrix<float> m(r, d);
        std::copy(f, f + r * d, m.data());
        f += r * d;
        up.push_back(std::move(m));
      }
      set.emplace(ids[a], LoraAdapter(ids[a], L, d, r, std::move(down), std::move(up), std::nullopt));
    }
    save_model_fixture(model, set, dir);
    return 0;
  } catch (const Error&) {
    return 1;
  }
}


// The stack forward through BaseModel + ModelState (model.hpp:192-328):
// mode 0 forward_unmerged, 1 forward_merged (W used as given), 2
// forward_mixture: the reference merges adapter merged_id into W (merge,
// model.hpp:144), attaches the subtraction branch (init_delora) and runs
// forward_mixture; w then holds the merged weights on return.
// w is [L][d*d]; downs[a] / ups[a] are [L][d*r] / [L][r*d].
int ref_forward(int mode, size_t L, size_t d, float* w, size_t num_adapters, const int32_t* ids,
                const int64_t* ranks, const float* const* downs, const float* const* ups, const float* x,
                size_t n, const int32_t* assignment, int32_t merged_id, float* out) {
  try {
    BaseModel model(L, d, 2);
    for (size_t l = 0; l < L; ++l) std::memcpy(model.layer(l).data, w + l * d * d, d * d * 4);
    AdapterSet adapters;
    for (size_t i = 0; i < num_adapters; ++i) {
      const size_t r = static_cast<size_t>(ranks[i]);
      std::vector<Matrix<float>> dn, u;
      for (size_t l = 0; l < L; ++l) {
        Matrix<float> dm(d, r), um(r, d);
        std::memcpy(dm.data(), downs[i] + l * d * r, d * r * 4);
        std::memcpy(um.data(), ups[i] + l * r * d, r * d * 4);
        dn.push_back(std::move(dm));
        u.push_back(std::move(um));
      }
      adapters.emplace(ids[i], LoraAdapter(ids[i], L, d, r, std::move(dn), std::move(u)));
    }
    TilingTable table;
    ModelState state;
    ConstMatSpan<float> xs(x, n, d);
    std::vector<int> a(assignment ? assignment : nullptr, assignment ? assignment + n : nullptr);
    Matrix<float> res(1, 1);
    if (mode == 0) {
      res = forward_unmerged(model, state, xs, std::span<const int>(a.data(), a.size()), adapters, table);
    } else if (mode == 1) {
      state.mode = InferMode::Merged;
      res = forward_merged(model, state, xs, table);
    } else {
      merge(model, state, adapter_at(adapters, merged_id), table);
      init_delora(state, adapter_at(adapters, merged_id));
      state.mode = InferMode::Mixture;
      res = forward_mixture(model, state, xs, std::span<const int>(a.data(), a.size()), adapters, table);
      for (size_t l = 0; l < L; ++l) std::memcpy(w + l * d * d, model.layer(l).data, d * d * 4);
    }
    std::memcpy(out, res.data(), n * d * 4);
    return 0;
  } catch (const std::exception& e) {
    return status_of(e);
  }
}

}  // extern "C"
