// C++ host-layer tests (include/cstress_b200.hpp) -- ports of
// /root/reference/proj/tests/test_mset.cpp and test_backends.cpp cases onto
// the B200 backend, written against the C++ mirror of the reference API.
// Exit code = number of failed checks.  `--list` prints the cases (no GPU).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "cstress_b200.hpp"

using namespace cstress_b200;

static int g_fail = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    if (!(cond)) {                                                               \
      ++g_fail;                                                                  \
      std::printf("    CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
    }                                                                            \
  } while (0)
#define CHECK_THROWS_AS(expr, Ex)                                                \
  do {                                                                           \
    bool ok = false;                                                             \
    try {                                                                        \
      (void)(expr);                                                              \
    } catch (const Ex&) {                                                        \
      ok = true;                                                                 \
    } catch (...) {                                                              \
    }                                                                            \
    if (!ok) {                                                                   \
      ++g_fail;                                                                  \
      std::printf("    CHECK_THROWS_AS failed %s:%d: %s\n", __FILE__, __LINE__, #expr); \
    }                                                                            \
  } while (0)

static SignalMatrix rows(std::initializer_list<std::initializer_list<double>> r) {
  SignalMatrix s{Matrix(static_cast<Index>(r.size()), static_cast<Index>(r.begin()->size()))};
  Index i = 0;
  for (const auto& row : r) {
    Index j = 0;
    for (double v : row) s.data(i, j++) = v;
    ++i;
  }
  return s;
}

static SignalMatrix random_signals(Index n, Index N, uint64_t seed) {  // test_mset.cpp:70-72
  return synthesize_uniform(n, N, 0.3, 0.2, 1.0, 0.2, 3.5, seed);
}

static const BackendId B64 = BackendId::b200(0, CS_PRECISION_FP64);
static const BackendId B32 = BackendId::b200(0, CS_PRECISION_FP32);

static void kernel_closed_forms() {  // test_mset.cpp:76-94 through sim_matrix
  Matrix x(3, 1), y(3, 1);
  x(0, 0) = 1, x(1, 0) = 2, x(2, 0) = 3;
  y = x;
  CHECK(sim_matrix(x, y, {KernelKind::gaussian, 1.0})(0, 0) == 1.0);
  CHECK(sim_matrix(x, y, {KernelKind::inverse_distance, 2.0})(0, 0) == 1.0);
  y(2, 0) = 4;
  CHECK(std::fabs(sim_matrix(x, y, {KernelKind::gaussian, 1.0})(0, 0) - std::exp(-0.5)) < 1e-12);
  y(2, 0) = 5;
  CHECK(std::fabs(sim_matrix(x, y, {KernelKind::inverse_distance, 2.0})(0, 0) - 0.5) < 1e-12);
  CHECK_THROWS_AS(sim_matrix(x, Matrix(2, 1), {}), ShapeError);
}

static void selection_cases() {  // test_mset.cpp:96-147
  auto mem = select_memory_vectors(rows({{5.0}, {-3.0}, {9.0}, {0.0}}), 2);
  auto idx = mem.source_indices;
  std::sort(idx.begin(), idx.end());
  CHECK((idx == std::vector<Index>{1, 2}));
  mem = select_memory_vectors(rows({{-10, 1}, {10, 2}, {0, -5}, {1, 5}, {0.5, 0.5}, {0.2, 0.1}}), 4);
  idx = mem.source_indices;
  std::sort(idx.begin(), idx.end());
  CHECK((idx == std::vector<Index>{0, 1, 2, 3}));
  const auto five = rows({{1, 0}, {2, 1}, {3, 2}, {4, 3}, {5, 4}});
  CHECK_THROWS_AS(select_memory_vectors(five, 3), ConstraintViolated);
  CHECK_THROWS_AS(select_memory_vectors(five, 6), InsufficientTraining);
  CHECK_THROWS_AS(select_memory_vectors(rows({{1}, {1}, {1}, {1}, {2}, {3}}), 4), InsufficientTraining);
  try {
    select_memory_vectors(five, 3);
  } catch (const ConstraintViolated& e) {
    CHECK(std::string(e.what()) == "select_memory_vectors: m=3 violates m >= 2n with n=2");
  }
}

static void matmul_cases() {  // test_backends.cpp:99-141
  Matrix A(2, 2), B(2, 2);
  A(0, 0) = 1, A(0, 1) = 2, A(1, 0) = 3, A(1, 1) = 4;
  B(0, 0) = 5, B(0, 1) = 6, B(1, 0) = 7, B(1, 1) = 8;
  const Matrix C = matmul(A, B);
  CHECK(C(0, 0) == 19 && C(0, 1) == 22 && C(1, 0) == 43 && C(1, 1) == 50);
  Matrix Z(2, 3);
  CHECK(batched_solve(A, Matrix(2, 7))(1, 6) == 0.0);
  CHECK_THROWS_AS(matmul(A, Matrix(3, 4)), ShapeError);
}

static void eig_cases() {  // test_mset.cpp:163-199
  Matrix d(3, 3);
  d(0, 0) = 3, d(1, 1) = 1, d(2, 2) = 2;
  const auto e = symmetric_eig(d);
  CHECK(std::fabs(e.eigenvalues[0] - 1) < 1e-12 && std::fabs(e.eigenvalues[2] - 3) < 1e-12);
  Matrix asym(2, 2);
  asym(0, 0) = 1, asym(0, 1) = 0.5, asym(1, 1) = 1;
  CHECK_THROWS_AS(symmetric_eig(asym), ShapeError);
}

static void training_cases() {  // test_mset.cpp:201-250
  const auto tr = random_signals(2, 64, 31);
  const auto model = train(tr, 4, {KernelKind::gaussian, {}}, B64);
  const auto host = model.export_host();
  Matrix Dn = host.memory.D;
  for (Index s = 0; s < 2; ++s)
    for (Index c = 0; c < 4; ++c) Dn(s, c) /= host.signal_scale[size_t(s)];
  const Matrix gram = sim_matrix(Dn, Dn, model.kernel());
  for (Index i = 0; i < 4; ++i) CHECK(gram(i, i) == 1.0);
  CHECK(model.rank() == 4);
  const Matrix I = matmul(host.gram_pinv, gram);
  double worst = 0;
  for (Index i = 0; i < 4; ++i)
    for (Index j = 0; j < 4; ++j) worst = std::max(worst, std::fabs(I(i, j) - (i == j ? 1.0 : 0.0)));
  CHECK(worst < 1e-8);

  CHECK(train(rows({{0}, {1}, {2}, {3}, {3}}), 4, {KernelKind::gaussian, 1.0}, B64).rank() < 4);

  for (const auto& b : {B64, B32}) {
    const auto m2 = train(random_signals(2, 128, 17), 4, {}, b);
    const auto h2 = m2.export_host();
    const auto r = estimate(m2, SignalMatrix{h2.memory.D.transpose()});
    const double tol = b.precision == CS_PRECISION_FP64 ? 1e-8 : 1e-3;
    for (Index s = 0; s < 2; ++s)
      for (Index t = 0; t < 4; ++t)
        CHECK(std::fabs(r.residuals(t, s)) <= tol * h2.signal_scale[size_t(s)]);
  }
  const auto m3 = train(random_signals(3, 64, 13), 8, {}, B32);
  const auto r3 = estimate(m3, SignalMatrix{Matrix(10, 3, 4.2)});
  for (double v : r3.estimates.v) CHECK(std::isfinite(v));

  CHECK_THROWS_AS(train(random_signals(2, 32, 5), 3, {}, B64), ConstraintViolated);
  const auto m4 = train(random_signals(2, 32, 5), 4, {}, B64);
  CHECK_THROWS_AS(estimate(m4, SignalMatrix{Matrix(4, 3)}), ShapeError);
}

static void plugin_cases() {  // test_mset.cpp:324-347
  const auto& algo = algorithm_by_name("mset2");
  CHECK(algo.name() == "mset2");
  const auto model = algo.train(random_signals(2, 64, 61), 4, {}, B32);
  const auto r = algo.estimate(*model, random_signals(2, 16, 67), B32);
  CHECK(r.estimates.rows() == 16);
  struct Other final : PrognosticModel {};
  CHECK_THROWS_AS(algo.estimate(Other{}, random_signals(2, 16, 67), B32), ConfigError);
  CHECK_THROWS_AS(algorithm_by_name("svm"), ConfigError);
}

static void mean_predictor_cases() {  // estimator.cpp:42-69 (host baseline predictor)
  const auto& algo = algorithm_by_name("mean");
  CHECK(algo.name() == "mean");
  Matrix X(4, 2);
  const double v[8] = {1, 2, 3, 6, -1, -1, 5, 1};
  for (int i = 0; i < 8; ++i) X.v[size_t(i)] = v[i];
  const auto model = algo.train(SignalMatrix{X}, 2, {}, B64);
  Matrix O(2, 2);
  O(0, 0) = 4.0, O(1, 0) = 2.0, O(0, 1) = 0.0, O(1, 1) = 1.0;
  const auto r = algo.estimate(*model, SignalMatrix{O}, B64);
  CHECK(r.estimates(0, 0) == 3.0 && r.estimates(1, 0) == 3.0);  // mean of 1, 2, 3, 6
  CHECK(r.estimates(0, 1) == 1.0 && r.estimates(1, 1) == 1.0);  // mean of -1, -1, 5, 1
  CHECK(r.residuals(0, 0) == 1.0 && r.residuals(1, 0) == -1.0 && r.residuals(0, 1) == -1.0);
  CHECK_THROWS_AS(algo.estimate(*model, SignalMatrix{Matrix(2, 3)}, B64), ShapeError);
  const auto mset_model = algorithm_by_name("mset2").train(random_signals(2, 64, 61), 4, {}, B64);
  CHECK_THROWS_AS(algo.estimate(*mset_model, SignalMatrix{O}, B64), ConfigError);
}

int main(int argc, char** argv) {
  const std::vector<std::pair<const char*, std::function<void()>>> cases = {
      {"kernel closed forms", kernel_closed_forms}, {"selection", selection_cases},
      {"matmul / batched_solve", matmul_cases},     {"symmetric_eig", eig_cases},
      {"train / estimate", training_cases},         {"plugin contract", plugin_cases},
      {"mean predictor", mean_predictor_cases},
  };
  if (argc > 1 && std::strcmp(argv[1], "--list") == 0) {
    for (const auto& c : cases) std::printf("%s\n", c.first);
    return 0;
  }
  for (const auto& c : cases) {
    const int before = g_fail;
    try {
      c.second();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("    exception: %s\n", e.what());
    }
    std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", c.first);
  }
  std::printf("%d failed check(s)\n", g_fail);
  return g_fail;
}
