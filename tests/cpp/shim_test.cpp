// shim_test.cpp -- plain-main restatement of the reference's Catch2 cases for
// the hot path (test_batch.cpp, test_tiling.cpp, test_atmm.cpp,
// test_model.cpp), written against include/loraserve_b200.hpp.
//   ./shim_test host   -> host-only checks (CPU box)
//   ./shim_test gpu    -> host checks + device parity checks (B200)
// Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "loraserve_b200.hpp"

using namespace loraserve_b200;

static int g_fail = 0;
#define CHECK(cond)                                                       \
  do {                                                                    \
    if (!(cond)) {                                                        \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);         \
      ++g_fail;                                                           \
    }                                                                     \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                       \
  do {                                                                    \
    bool thrown_ = false;                                                 \
    try {                                                                 \
      (void)(expr);                                                       \
    } catch (const type&) {                                               \
      thrown_ = true;                                                     \
    } catch (...) {                                                       \
    }                                                                     \
    if (!thrown_) {                                                       \
      std::printf("FAIL %s:%d  %s did not throw %s\n", __FILE__, __LINE__, #expr, #type); \
      ++g_fail;                                                           \
    }                                                                     \
  } while (0)

static void host_checks() {
  // test_batch.cpp:40-61 -- plan_batch grouping rules
  BatchPlan p1 = plan_batch({3, 3, 3});
  CHECK(p1.segments.size() == 1);
  CHECK(p1.segments[0].adapter_id == 3);
  CHECK((p1.segments[0].rows == std::vector<std::size_t>{0, 1, 2}));
  BatchPlan p2 = plan_batch({7, 2, 7, 2});
  CHECK(p2.segments.size() == 2);
  CHECK(p2.segments[0].adapter_id == 2);
  CHECK((p2.segments[0].rows == std::vector<std::size_t>{1, 3}));
  CHECK(p2.segments[1].adapter_id == 7);
  CHECK((p2.segments[1].rows == std::vector<std::size_t>{0, 2}));
  BatchPlan p3 = plan_batch({5, 1, 9});
  CHECK(p3.segments.size() == 3);
  for (const Segment& s : p3.segments) CHECK(s.rows.size() == 1);
  CHECK_THROWS_AS(plan_batch({}), ConfigError);
  // device GEMM shape checks run before any device access
  CHECK_THROWS_AS(gemm(nullptr, 8, nullptr, 40, nullptr, 40, ATMM_F32, 4, 8, 36), ShapeError);

  // test_tiling.cpp:55-87 -- validity, bucketing, lookup rules
  CHECK((TilingConfig{64, 32, 32, 32, 32, 32}.structurally_valid()));
  CHECK(!(TilingConfig{48, 32, 32, 16, 16, 16}.structurally_valid()));
  CHECK(!(TilingConfig{8, 32, 32, 8, 16, 16}.structurally_valid()));
  CHECK(!(TilingConfig{32, 32, 32, 64, 16, 16}.structurally_valid()));
  CHECK(m_bucket_of(1) == 32);
  CHECK(m_bucket_of(32) == 32);
  CHECK(m_bucket_of(33) == 64);
  CHECK(m_bucket_of(4096) == 4096);
  CHECK((shape_key(33, 256, 16) == ShapeKey{64, 256, 16}));
  TilingTable table(TilingConfig{32, 32, 32, 32, 32, 32});
  const TilingConfig stored{64, 32, 32, 32, 32, 32};
  table.insert(ShapeKey{64, 256, 16}, stored, 1000);
  CHECK(table.lookup(33, 256, 16) == stored);
  CHECK(table.lookup(90, 256, 16) == stored);
  CHECK((table.lookup(200, 256, 16) == TilingConfig{32, 32, 32, 32, 32, 32}));
  CHECK((table.lookup(64, 128, 16) == TilingConfig{32, 32, 32, 32, 32, 32}));
  table.insert(ShapeKey{128, 256, 16}, TilingConfig{128, 64, 64, 32, 32, 32}, 900);
  CHECK(table.lookup(96, 256, 16) == stored);
  CHECK_THROWS_AS(table.insert(ShapeKey{32, 1, 1}, TilingConfig{24, 16, 16, 8, 16, 16}, 1), ConfigError);

  // test_tiling.cpp:89-104 -- JSON round trip
  TilingTable t2(TilingConfig{64, 32, 32, 32, 32, 32});
  t2.insert(ShapeKey{256, 4096, 32}, TilingConfig{64, 32, 32, 32, 32, 32}, 70000);
  t2.insert(ShapeKey{8192, 4096, 128}, TilingConfig{64, 64, 64, 32, 64, 64}, 100000);
  const std::string path = "/tmp/loraserve_b200_shim_table.json";
  t2.save(path);
  TilingTable back = TilingTable::load(path);
  CHECK(back.size() == 2);
  CHECK((back.lookup(256, 4096, 32) == TilingConfig{64, 32, 32, 32, 32, 32}));
  CHECK((back.lookup(8192, 4096, 128) == TilingConfig{64, 64, 64, 32, 64, 64}));
  CHECK_THROWS_AS(TilingTable::load("/nonexistent/table.json"), IoError);

  // matrix.hpp:183-218 -- binary fixture round trip and errors
  const std::vector<float> m = {1.f, -2.5f, 3.25f, 0.f, 7.f, -0.125f};
  save_matrix("/tmp/loraserve_b200_shim_m.bin", 2, 3, m);
  std::size_t mr = 0, mc = 0;
  CHECK(load_matrix("/tmp/loraserve_b200_shim_m.bin", &mr, &mc) == m);
  CHECK(mr == 2 && mc == 3);
  CHECK_THROWS_AS(load_matrix("/nonexistent/m.bin", nullptr, nullptr), IoError);
  CHECK_THROWS_AS(save_matrix("/tmp/loraserve_b200_shim_m.bin", 4, 3, m), ShapeError);
}

static void gpu_checks() {
  // test_batch.cpp:63-80 -- run_bypass vs the per-row double oracle, here
  // with bf16 inputs (exact in both) and the north-star tolerance.
  const std::size_t d = 256, n = 37;
  std::mt19937 g(7);
  std::uniform_real_distribution<float> u(-1.f, 1.f);
  auto bf16 = [](float f) {
    uint32_t x;
    std::memcpy(&x, &f, 4);
    x = (x + 0x7fffu + ((x >> 16) & 1u)) & 0xffff0000u;
    float r;
    std::memcpy(&r, &x, 4);
    return r;
  };
  AdapterRegistry reg(0, 1, d, d);
  std::vector<std::vector<float>> downs, ups;
  const std::size_t ranks[3] = {8, 16, 32};
  for (int a = 0; a < 3; ++a) {
    const std::size_t r = ranks[a];
    std::vector<float> dn(d * r), up(r * d);
    for (auto& v : dn) v = bf16(u(g) * 0.3f);
    for (auto& v : up) v = bf16(u(g) * 0.3f);
    reg.put(a + 1, r, dn.data(), up.data());
    downs.push_back(dn);
    ups.push_back(up);
  }
  std::vector<float> x(n * d);
  for (auto& v : x) v = bf16(u(g));
  std::vector<int> assignment(n);
  for (std::size_t i = 0; i < n; ++i) assignment[i] = 1 + static_cast<int>(i % 3);
  std::vector<float> got = run_bypass(reg, x, assignment, 0);
  double worst = 0, scale = 1;
  for (std::size_t row = 0; row < n; ++row) {
    const int a = assignment[row] - 1;
    const std::size_t r = ranks[a];
    std::vector<double> mid(r, 0.0);
    for (std::size_t j = 0; j < r; ++j)
      for (std::size_t p = 0; p < d; ++p) mid[j] += double(x[row * d + p]) * downs[a][p * r + j];
    for (std::size_t c = 0; c < d; ++c) {
      double acc = 0;
      for (std::size_t j = 0; j < r; ++j) acc += mid[j] * ups[a][j * d + c];
      worst = std::max(worst, std::fabs(acc - got[row * d + c]));
      scale = std::max(scale, std::fabs(acc));
    }
  }
  CHECK(worst <= 1e-2 * scale);
  CHECK_THROWS_AS(run_bypass(reg, x, std::vector<int>(n, 9), 0), UnknownAdapterError);

  // test_atmm.cpp:62-70 -- bad shapes / configs; matrix KAT
  CHECK_THROWS_AS(atmm_multiply(std::vector<float>(20), 4, 5, std::vector<float>(20), 4,
                                TilingConfig{24, 16, 16, 8, 16, 16}),
                  ConfigError);
  std::vector<float> c = atmm_multiply({1, 2, 3, 4}, 2, 2, {5, 6, 7, 8}, 2, TilingConfig{16, 16, 16, 16, 16, 16});
  CHECK(c[0] == 19 && c[1] == 22 && c[2] == 43 && c[3] == 50);

  // test_model.cpp:27-46 -- rank-1 delta_w KAT
  AdapterRegistry r1(0, 1, 64, 64);
  std::vector<float> dn(64, 0.f), up(64, 0.f);
  dn[3] = 1.f;
  up[5] = 1.f;
  r1.put(9, 1, dn.data(), up.data());
  std::vector<float> dw = delta_w(r1, 9, 0);
  double sum = 0;
  for (float v : dw) sum += std::fabs(v);
  CHECK(dw[3 * 64 + 5] == 1.f);
  CHECK(sum == 1.0);

  // put_async == put (device-side packing), then the mixture plan on device
  // buffers: guest rows get own - merged, merged rows stay untouched.
  AdapterRegistry r2(0, 1, d, d);
  r2.put_async(1, ranks[0], downs[0].data(), ups[0].data());
  r2.put(2, ranks[1], downs[1].data(), ups[1].data());
  CHECK(cudaDeviceSynchronize() == cudaSuccess);
  std::vector<float> own = run_bypass(r2, x, std::vector<int>(n, 1), 0);
  std::vector<float> ref1 = run_bypass(reg, x, std::vector<int>(n, 1), 0);
  CHECK(own == ref1);
  std::vector<int> mix(n);
  for (std::size_t i = 0; i < n; ++i) mix[i] = 1 + static_cast<int>(i % 2);
  MixturePlan mp(r2, mix, /*merged*/ 2);
  std::vector<uint16_t> xb(n * d);
  for (std::size_t i = 0; i < n * d; ++i) {
    uint32_t bits;
    std::memcpy(&bits, &x[i], 4);
    xb[i] = static_cast<uint16_t>(bits >> 16);  // x is bf16-exact
  }
  void *xd = nullptr, *yd = nullptr;
  CHECK(cudaMalloc(&xd, n * d * 2) == cudaSuccess);
  CHECK(cudaMalloc(&yd, n * d * 4) == cudaSuccess);
  CHECK(cudaMemcpy(xd, xb.data(), n * d * 2, cudaMemcpyHostToDevice) == cudaSuccess);
  CHECK(cudaMemset(yd, 0, n * d * 4) == cudaSuccess);
  mp.apply(0, xd, d, yd, d, ATMM_F32);
  std::vector<float> y(n * d);
  CHECK(cudaMemcpy(y.data(), yd, n * d * 4, cudaMemcpyDeviceToHost) == cudaSuccess);
  std::vector<float> cancel = run_bypass(r2, x, std::vector<int>(n, 2), 0);
  double mworst = 0, mscale = 1;
  for (std::size_t row = 0; row < n; ++row) {
    for (std::size_t c2 = 0; c2 < d; ++c2) {
      const double want = mix[row] == 2 ? 0.0 : double(own[row * d + c2]) - cancel[row * d + c2];
      mworst = std::max(mworst, std::fabs(want - y[row * d + c2]));
      mscale = std::max(mscale, std::fabs(want));
      if (mix[row] == 2) CHECK(y[row * d + c2] == 0.f);
    }
  }
  CHECK(mworst <= 1e-2 * mscale);
  // LayerForward (model.hpp:216-246) with W = 0: out = tanh(own bypass)
  void *wd = nullptr, *od = nullptr;
  CHECK(cudaMalloc(&wd, d * d * 2) == cudaSuccess);
  CHECK(cudaMalloc(&od, n * d * 2) == cudaSuccess);
  CHECK(cudaMemset(wd, 0, d * d * 2) == cudaSuccess);
  {
    LayerForward fw(r2, std::vector<int>(n, 1));
    fw.run(wd, d, d * d, 1, xd, d, od, d);
    std::vector<uint16_t> ob(n * d);
    CHECK(cudaMemcpy(ob.data(), od, n * d * 2, cudaMemcpyDeviceToHost) == cudaSuccess);
    double fworst = 0;
    for (std::size_t i = 0; i < n * d; ++i) {
      const uint32_t bits = static_cast<uint32_t>(ob[i]) << 16;
      float got;
      std::memcpy(&got, &bits, 4);
      fworst = std::max(fworst, std::fabs(double(got) - std::tanh(double(own[i]))));
    }
    CHECK(fworst <= 2e-2);  // bf16 output + bf16-rounded mid in run_bypass
    CHECK_THROWS_AS(fw.run(wd, d, d * d, 2, xd, d, od, d), ShapeError);  // the adapters carry one layer
  }
  // gemm (atmm.hpp:111-142 with a dense operand): X . I == X exactly, fp32 out
  {
    std::vector<uint16_t> eye(d * d, 0);
    for (std::size_t i = 0; i < d; ++i) eye[i * d + i] = 0x3F80;  // bf16 1.0
    void* cd = nullptr;
    CHECK(cudaMemcpy(wd, eye.data(), d * d * 2, cudaMemcpyHostToDevice) == cudaSuccess);
    CHECK(cudaMalloc(&cd, n * d * 4) == cudaSuccess);
    gemm(xd, d, wd, d, cd, d, ATMM_F32, n, d, d);
    std::vector<float> cg(n * d);
    std::vector<uint16_t> xdev(n * d);
    CHECK(cudaMemcpy(cg.data(), cd, n * d * 4, cudaMemcpyDeviceToHost) == cudaSuccess);
    CHECK(cudaMemcpy(xdev.data(), xd, n * d * 2, cudaMemcpyDeviceToHost) == cudaSuccess);
    bool same = true;
    for (std::size_t i = 0; i < n * d; ++i) {
      const uint32_t bits = static_cast<uint32_t>(xdev[i]) << 16;
      float want;
      std::memcpy(&want, &bits, 4);
      same = same && cg[i] == want;
    }
    CHECK(same);
    cudaFree(cd);
  }
  cudaFree(wd);
  cudaFree(od);
  cudaFree(xd);
  cudaFree(yd);
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::string(argv[1]) == "gpu";
  try {
    host_checks();
    if (gpu) gpu_checks();
  } catch (const std::exception& e) {
    std::printf("FAIL uncaught exception: %s\n", e.what());
    ++g_fail;
  }
  std::printf("%s: %d failure(s)\n", gpu ? "host+gpu" : "host", g_fail);
  return g_fail;
}
