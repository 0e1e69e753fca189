// acceptance_shim.cpp -- the reference's acceptance criteria 1-4
// (proj/tests/acceptance.cpp:59-211) and its merge / mode-contract unit cases
// (proj/tests/test_model.cpp:62-100, serving.hpp:38-74) restated against the
// drop-in header include/loraserve_compat.hpp: the calls are the reference's
// signatures (namespace loraserve), only the includes differ.  Every operator
// runs on the B200 (fp32-faithful split-bf16 tensor-core products); the
// tolerances are the reference's own 1e-4 * max(1, max|ref|).
//
//   ./acceptance_shim          -> exit code = number of failed checks
#include <chrono>
#include <cstdio>
#include <string>
#include <vector>

#include "loraserve_compat.hpp"
#include "loraserve_compat_testing.hpp"

using namespace loraserve;

namespace {

int failures = 0;

void report(const char* what, bool ok, const std::string& detail) {
  std::printf("%s  %-34s %s\n", ok ? "PASS" : "FAIL", what, detail.c_str());
  std::fflush(stdout);
  failures += ok ? 0 : 1;
}

double secs(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

double tol_of(ConstMatSpan<float> ref) { return 1e-4 * std::max(1.0, max_abs<float>(ref)); }

// acceptance.cpp:59-101 -- ATMM vs the fp64 oracle, 50 random shapes x 5 configs.
void atmm_oracle_equivalence() {
  const auto t0 = std::chrono::steady_clock::now();
  Rng rng(0xa1);
  std::uniform_int_distribution<std::size_t> dim(1, 512);
  const TilingConfig configs[] = {{16, 64, 64, 16, 16, 64}, {64, 32, 32, 32, 32, 32}, {64, 64, 64, 32, 64, 64},
                                  {128, 128, 64, 64, 32, 32}, {256, 128, 128, 64, 64, 32}};
  double worst = 0.0;
  std::string bad;
  for (int i = 0; i < 50 && bad.empty(); ++i) {
    const std::size_t m = dim(rng), k = dim(rng), n = dim(rng);
    const Matrix<float> a = random_matrix<float>(m, k, rng);
    const Matrix<float> b = random_matrix<float>(k, n, rng);
    const Matrix<float> ref = gemm_reference<float>(a, b);
    const double tol = tol_of(ref);
    for (const TilingConfig& cfg : configs) {
      const double d = max_abs_diff<float>(atmm_multiply<float>(a, b, cfg), ref);
      worst = std::max(worst, d / tol);
      if (d > tol) {
        bad = std::to_string(m) + "x" + std::to_string(k) + "x" + std::to_string(n) + " " + cfg.to_string();
        break;
      }
    }
  }
  const double s = secs(t0);
  report("1 atmm-oracle-equivalence", bad.empty() && s < 120.0,
         bad.empty() ? "50 shapes x 5 configs, worst diff/tol " + std::to_string(worst) + ", " + std::to_string(s) + " s"
                     : "mismatch at " + bad);
}

// acceptance.cpp:107-172 -- mixture == unmerged on guest rows; merged ==
// unmerged when every row is the merged adapter's.
void mixture_and_merge_equivalence() {
  const auto t0 = std::chrono::steady_clock::now();
  const std::size_t L = 4, d = 256, V = 64;
  const std::size_t ranks[] = {8, 16, 32, 64};
  TilingTable table;
  double worst_mix = 0.0, worst_merge = 0.0;
  bool ok_mix = true, ok_merge = true;
  for (int inst = 0; inst < 100; ++inst) {
    const std::uint64_t seed = 9000 + inst;
    BaseModel model = BaseModel::random(L, d, V, seed);
    AdapterSet adapters;
    adapters.emplace(1, LoraAdapter::random(1, L, d, ranks[inst % 4], seed * 3 + 1));
    adapters.emplace(2, LoraAdapter::random(2, L, d, ranks[(inst + 1) % 4], seed * 3 + 2));
    Rng rng(seed ^ 0x55);
    const Matrix<float> x = random_matrix<float>(4, d, rng);
    const std::vector<int> mixed = {1, 2, 2, 1}, all_one(4, 1);
    ModelState state;
    const Matrix<float> unmerged = forward_unmerged(model, state, x, mixed, adapters, table);
    const Matrix<float> unmerged_one = forward_unmerged(model, state, x, all_one, adapters, table);
    merge(model, state, adapter_at(adapters, 1), table);
    const Matrix<float> merged = forward_merged(model, state, x, table);
    init_delora(state, adapter_at(adapters, 1));
    state.mode = InferMode::Mixture;
    const Matrix<float> mixture = forward_mixture(model, state, x, mixed, adapters, table);
    const double tol = tol_of(unmerged);
    for (std::size_t row = 0; row < 4; ++row) {
      if (mixed[row] == 1) continue;
      const double dd = max_abs_diff<float>(ConstMatSpan<float>(mixture.data() + row * d, 1, d),
                                            ConstMatSpan<float>(unmerged.data() + row * d, 1, d));
      worst_mix = std::max(worst_mix, dd / tol);
      ok_mix = ok_mix && dd <= tol;
    }
    const double d3 = max_abs_diff<float>(merged, unmerged_one);
    worst_merge = std::max(worst_merge, d3 / tol);
    ok_merge = ok_merge && d3 <= tol;
  }
  const double s = secs(t0);
  report("2 delora-mixture-identity", ok_mix && s < 60.0,
         "100 instances, worst diff/tol " + std::to_string(worst_mix) + ", " + std::to_string(s) + " s");
  report("3 merged-unmerged-equivalence", ok_merge, "100 instances, worst diff/tol " + std::to_string(worst_merge));
}

// acceptance.cpp:177-211 -- 100 merge/unmerge cycles: bounded drift, no reallocation.
void merge_unmerge_round_trip() {
  const std::size_t L = 4, d = 256, V = 64, r = 64;
  TilingTable table;
  BaseModel model = BaseModel::random(L, d, V, 44);
  AdapterSet adapters;
  adapters.emplace(1, LoraAdapter::random(1, L, d, r, 45));
  std::vector<Matrix<float>> before;
  std::vector<const float*> addr;
  double scale = 0.0;
  for (std::size_t l = 0; l < L; ++l) {
    Matrix<float> c(d, d);
    std::copy(model.layer(l).data, model.layer(l).data + d * d, c.data());
    scale = std::max(scale, max_abs<float>(c));
    before.push_back(std::move(c));
    addr.push_back(model.layer(l).data);
  }
  ModelState state;
  const LoraAdapter& a = adapter_at(adapters, 1);
  for (int cycle = 0; cycle < 100; ++cycle) {
    merge(model, state, a, table);
    unmerge(model, state, a, table);
  }
  double drift = 0.0;
  bool stable = true;
  for (std::size_t l = 0; l < L; ++l) {
    drift = std::max(drift, max_abs_diff<float>(model.layer(l), before[l]));
    stable = stable && model.layer(l).data == addr[l];
  }
  const double tol = 1e-4 * std::max(1.0, scale);
  report("4 merge-unmerge-round-trip", drift <= tol && stable,
         "100 cycles, drift " + std::to_string(drift) + " (tol " + std::to_string(tol) + "), " +
             (stable ? "address-stable" : "REALLOCATED"));
}

// test_model.cpp:62-100 + serving.hpp:38-74: merge flips the mode, applies
// delta_w in place; double merge / wrong unmerge are ModeErrors; mode_switch
// takes the minimal path.
void mode_contract() {
  TilingTable table;
  const std::size_t L = 3, d = 64;
  BaseModel model = BaseModel::random(L, d, 8, 1);
  AdapterSet adapters;
  adapters.emplace(1, LoraAdapter::random(1, L, d, 4, 11));
  adapters.emplace(2, LoraAdapter::random(2, L, d, 8, 12));
  ModelState state;
  std::vector<Matrix<float>> before;
  for (std::size_t l = 0; l < L; ++l) {
    Matrix<float> c(d, d);
    std::copy(model.layer(l).data, model.layer(l).data + d * d, c.data());
    before.push_back(std::move(c));
  }
  const LoraAdapter& a1 = adapter_at(adapters, 1);
  merge(model, state, a1, table);
  bool ok = state.mode == InferMode::Merged && state.merged_adapter == 1;
  for (std::size_t l = 0; l < L; ++l) {
    Matrix<float> expect = before[l];
    add_inplace<float>(expect, delta_w(a1, l, table));
    ok = ok && max_abs_diff<float>(model.layer(l), expect) <= 1e-6;
  }
  bool threw = false;
  try {
    merge(model, state, a1, table);
  } catch (const ModeError&) {
    threw = true;
  }
  ok = ok && threw;
  threw = false;
  try {
    unmerge(model, state, adapter_at(adapters, 2), table);
  } catch (const ModeError&) {
    threw = true;
  }
  ok = ok && threw;
  unmerge(model, state, a1, table);
  ok = ok && state.mode == InferMode::Unmerged;
  for (std::size_t l = 0; l < L; ++l) {
    ok = ok && max_abs_diff<float>(model.layer(l), before[l]) <= 4 * 1.2e-7 * max_abs<float>(before[l]) + 1e-6;
  }
  // mode_switch: unmerged -> mixture(2) merges once; -> merged(2) writes nothing
  mode_switch(model, state, InferMode::Mixture, 2, adapters, table);
  ok = ok && state.mode == InferMode::Mixture && state.merged_adapter == 2 && state.delora_branch == &adapter_at(adapters, 2);
  Matrix<float> snap(d, d);
  std::copy(model.layer(0).data, model.layer(0).data + d * d, snap.data());
  mode_switch(model, state, InferMode::Merged, 2, adapters, table);
  ok = ok && state.mode == InferMode::Merged && max_abs_diff<float>(model.layer(0), snap) == 0.0;
  mode_switch(model, state, InferMode::Unmerged, -1, adapters, table);
  ok = ok && state.mode == InferMode::Unmerged;
  threw = false;
  try {
    (void)adapter_at(adapters, 99);
  } catch (const UnknownAdapterError& e) {
    threw = e.id() == 99;
  }
  ok = ok && threw;
  // bypass FLOPs are padding-free (test_batch.cpp:96-128)
  const Matrix<float> x = [] {
    Rng rng(10);
    return random_matrix<float>(6, 64, rng);
  }();
  const std::vector<int> assignment = {1, 2, 1, 2, 1, 2};
  flops::Scope scope;
  (void)run_bypass(x, plan_batch(assignment), adapters, 0, table);
  ok = ok && scope.elapsed() == 3ull * 2 * 64 * 4 * 2 + 3ull * 2 * 64 * 8 * 2;
  report("mode contract / mode_switch / flops", ok, "test_model.cpp:62-100, serving.hpp:38-74");
}

}  // namespace

int main() {
  try {
    atmm_oracle_equivalence();
    mixture_and_merge_equivalence();
    merge_unmerge_round_trip();
    mode_contract();
  } catch (const Error& e) {
    std::printf("FAIL  exception: %s\n", e.what());
    return 100;
  }
  return failures;
}
