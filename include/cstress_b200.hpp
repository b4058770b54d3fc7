// cstress_b200.hpp -- C++ host layer over the C-ABI (cstress_b200.h).
//
// Mirrors the reference's C++ surface for the MSET2 path
// (/root/reference/proj/include/containerstress/{errors,kernels,backends,mset,
// estimator}.hpp): same names, argument meaning and error classes, with a
// minimal column-major FP64 Matrix in place of Eigen (absent here; the
// reference's Eigen buffers map onto it 1:1).  Header-only;
// link libcstress_b200.so.
#pragma once

#include <cmath>
#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "cstress_b200.h"

namespace cstress_b200 {

using Index = int64_t;

// ------------------------------------------------------------- errors.hpp:9-74
struct Error : std::runtime_error {
  explicit Error(const std::string& w) : std::runtime_error(w) {}
};
#define CSB_ERR(name) \
  struct name : Error { using Error::Error; };
CSB_ERR(MomentInfeasible)
CSB_ERR(BadCorrelation)
CSB_ERR(TooFewSamples)
CSB_ERR(ConstraintViolated)
CSB_ERR(InsufficientTraining)
CSB_ERR(DegenerateModel)
CSB_ERR(EigFailure)
CSB_ERR(ShapeError)
CSB_ERR(EmptyGrid)
CSB_ERR(ConfigError)
CSB_ERR(IoError)
#undef CSB_ERR

[[noreturn]] inline void rethrow(cs_status s) {
  const std::string m = cs_last_error();
  switch (s) {
    case CS_CONSTRAINT_VIOLATED: throw ConstraintViolated(m);
    case CS_INSUFFICIENT_TRAINING: throw InsufficientTraining(m);
    case CS_DEGENERATE_MODEL: throw DegenerateModel(m);
    case CS_EIG_FAILURE: throw EigFailure(m);
    case CS_SHAPE_ERROR: throw ShapeError(m);
    case CS_CONFIG_ERROR: throw ConfigError(m);
    case CS_IO_ERROR: throw IoError(m);
    case CS_MOMENT_INFEASIBLE: throw MomentInfeasible(m);
    case CS_BAD_CORRELATION: throw BadCorrelation(m);
    case CS_TOO_FEW_SAMPLES: throw TooFewSamples(m);
    case CS_EMPTY_GRID: throw EmptyGrid(m);
    default: throw Error(m);
  }
}
inline void check(cs_status s) {
  if (s != CS_OK) rethrow(s);
}

// --------------------------------------------------- column-major FP64 matrix
struct Matrix {
  Index r = 0, c = 0;
  std::vector<double> v;
  Matrix() = default;
  Matrix(Index rows, Index cols, double fill = 0.0) : r(rows), c(cols), v(size_t(rows * cols), fill) {}
  Index rows() const { return r; }
  Index cols() const { return c; }
  double* data() { return v.data(); }
  const double* data() const { return v.data(); }
  double& operator()(Index i, Index j) { return v[size_t(i + j * r)]; }
  double operator()(Index i, Index j) const { return v[size_t(i + j * r)]; }
  Matrix transpose() const {
    Matrix t(c, r);
    for (Index j = 0; j < c; ++j)
      for (Index i = 0; i < r; ++i) t(j, i) = (*this)(i, j);
    return t;
  }
};

// ------------------------------------------------------------ kernels.hpp
enum class KernelKind { inverse_distance = CS_KERNEL_INVERSE_DISTANCE, gaussian = CS_KERNEL_GAUSSIAN };

struct KernelConfig {
  KernelKind kind = KernelKind::inverse_distance;
  std::optional<double> bandwidth;
  void validate() const {
    if (bandwidth && !(*bandwidth > 0.0)) throw ConfigError("kernel bandwidth must be > 0");
  }
  KernelConfig resolved(Index n_signals) const {
    KernelConfig o = *this;
    if (!o.bandwidth) o.bandwidth = std::sqrt(static_cast<double>(n_signals));
    return o;
  }
};

// ----------------------------------------------------------- backends.hpp
struct BackendId {
  int device = 0;
  int precision = CS_PRECISION_FP64;  // CS_PRECISION_FP32: tcgen05 3xFP16 surveillance
  static BackendId b200(int device = 0, int precision = CS_PRECISION_FP64) { return {device, precision}; }
  std::string label() const {
    return "b200[device=" + std::to_string(device) + "/precision=" +
           (precision == CS_PRECISION_FP32 ? "fp32" : "fp64") + "]";
  }
  bool operator==(const BackendId&) const = default;
};

// one context per (host thread, device)
inline cs_ctx* context(int device) {
  struct Holder {
    std::map<int, cs_ctx*> m;
    ~Holder() {
      for (auto& kv : m) cs_ctx_destroy(kv.second);
    }
  };
  thread_local Holder h;
  cs_ctx*& c = h.m[device];
  if (!c) check(cs_ctx_create(device, &c));
  return c;
}

inline Matrix sim_matrix(const Matrix& A, const Matrix& B, const KernelConfig& cfg,
                         const BackendId& b = {}) {
  if (A.rows() != B.rows())
    throw ShapeError("sim_matrix: row counts differ (" + std::to_string(A.rows()) + " vs " +
                     std::to_string(B.rows()) + ")");
  cfg.validate();
  Matrix out(A.cols(), B.cols());
  check(cs_sim_matrix(context(b.device), A.data(), B.data(), A.rows(), A.cols(), B.cols(),
                      static_cast<int>(cfg.kind), cfg.bandwidth.value_or(0.0), out.data()));
  return out;
}

inline Matrix matmul(const Matrix& A, const Matrix& B, const BackendId& b = {}) {
  if (A.cols() != B.rows())
    throw ShapeError("matmul: inner dimensions differ (" + std::to_string(A.cols()) + " vs " +
                     std::to_string(B.rows()) + ")");
  Matrix out(A.rows(), B.cols());
  check(cs_matmul(context(b.device), A.data(), B.data(), A.rows(), A.cols(), B.cols(), out.data()));
  return out;
}

inline Matrix batched_solve(const Matrix& G, const Matrix& S, const BackendId& b = {}) {
  if (G.cols() != S.rows()) throw ShapeError("batched_solve: G_pinv columns must match S rows");
  Matrix out(G.rows(), S.cols());
  check(cs_batched_solve(context(b.device), G.data(), S.data(), G.rows(), S.cols(), out.data()));
  return out;
}

// ---------------------------------------------------------------- mset.hpp
struct SymmetricEig {
  std::vector<double> eigenvalues;
  Matrix eigenvectors;
};

inline SymmetricEig symmetric_eig(const Matrix& G, const BackendId& b = {}) {
  if (G.rows() != G.cols()) throw ShapeError("symmetric_eig: matrix is not square");
  SymmetricEig e{std::vector<double>(size_t(G.rows())), Matrix(G.rows(), G.rows())};
  check(cs_symmetric_eig(context(b.device), G.data(), G.rows(), e.eigenvalues.data(),
                         e.eigenvectors.data()));
  return e;
}

struct SignalMatrix {  // signals.hpp:45-51 (observations x signals)
  Matrix data;
  Index n_observations() const { return data.rows(); }
  Index n_signals() const { return data.cols(); }
};

struct MemoryMatrix {
  Matrix D;
  std::vector<Index> source_indices;
};

inline MemoryMatrix select_memory_vectors(const SignalMatrix& training, Index m, const BackendId& b = {}) {
  MemoryMatrix mem{Matrix(training.n_signals(), m), std::vector<Index>(size_t(m))};
  check(cs_select_memory_vectors(context(b.device), training.data.data(), training.n_observations(),
                                 training.n_signals(), m, mem.source_indices.data(), mem.D.data()));
  return mem;
}

// Device-resident TrainedModel (mset.hpp:46-57); immutable after training.
class TrainedModel {
 public:
  TrainedModel(cs_model* h, BackendId b) : h_(h, &cs_model_destroy), backend_(b) {
    int kind = 0, prec = 0;
    double bw = 0;
    check(cs_model_info(h, &n_, &m_, &rank_, &kind, &bw, &prec));
    kernel_.kind = static_cast<KernelKind>(kind);
    kernel_.bandwidth = bw;
  }
  Index n_signals() const { return n_; }
  Index n_memory() const { return m_; }
  Index rank() const { return rank_; }
  const KernelConfig& kernel() const { return kernel_; }
  const BackendId& backend() const { return backend_; }
  cs_model* handle() const { return h_.get(); }
  // TrainedModel fields on the host (CSM1 / diagnostics)
  struct Host {
    MemoryMatrix memory;
    Matrix gram_pinv;
    std::vector<double> eigen_spectrum, signal_scale;
  };
  Host export_host() const {
    Host o{MemoryMatrix{Matrix(n_, m_), std::vector<Index>(size_t(m_))}, Matrix(m_, m_),
           std::vector<double>(size_t(m_)), std::vector<double>(size_t(n_))};
    check(cs_model_export(h_.get(), o.memory.source_indices.data(), o.memory.D.data(), o.gram_pinv.data(),
                          o.eigen_spectrum.data(), o.signal_scale.data()));
    return o;
  }

 private:
  std::unique_ptr<cs_model, cs_status (*)(cs_model*)> h_;
  BackendId backend_;
  Index n_ = 0, m_ = 0, rank_ = 0;
  KernelConfig kernel_;
};

struct EstimationResult {
  Matrix estimates;  // observations x signals
  Matrix residuals;
};

inline TrainedModel train(const SignalMatrix& training, Index m, const KernelConfig& cfg,
                          const BackendId& b = {}) {
  cfg.validate();
  cs_model* h = nullptr;
  check(cs_mset_train(context(b.device), training.data.data(), training.n_observations(),
                      training.n_signals(), m, static_cast<int>(cfg.kind), cfg.bandwidth.value_or(0.0),
                      b.precision, &h));
  return TrainedModel(h, b);
}

inline EstimationResult estimate(const TrainedModel& model, const SignalMatrix& obs) {
  EstimationResult r{Matrix(obs.n_observations(), obs.n_signals()),
                     Matrix(obs.n_observations(), obs.n_signals())};
  check(cs_mset_estimate(context(model.backend().device), model.handle(), obs.data.data(),
                         obs.n_observations(), obs.n_signals(), r.estimates.data(), r.residuals.data()));
  return r;
}

// ----------------------------------------------------------- estimator.hpp
class PrognosticModel {
 public:
  virtual ~PrognosticModel() = default;
};

class PrognosticAlgorithm {
 public:
  virtual ~PrognosticAlgorithm() = default;
  virtual std::string name() const = 0;
  virtual std::unique_ptr<PrognosticModel> train(const SignalMatrix& training, Index n_memory,
                                                 const KernelConfig& kernel,
                                                 const BackendId& backend) const = 0;
  virtual EstimationResult estimate(const PrognosticModel& model, const SignalMatrix& observations,
                                    const BackendId& backend) const = 0;
};

class MsetAlgorithm final : public PrognosticAlgorithm {
 public:
  struct Model final : PrognosticModel {
    explicit Model(TrainedModel m) : model(std::move(m)) {}
    TrainedModel model;
  };
  std::string name() const override { return "mset2"; }
  std::unique_ptr<PrognosticModel> train(const SignalMatrix& training, Index n_memory,
                                         const KernelConfig& kernel,
                                         const BackendId& backend) const override {
    return std::make_unique<Model>(cstress_b200::train(training, n_memory, kernel, backend));
  }
  EstimationResult estimate(const PrognosticModel& model, const SignalMatrix& observations,
                            const BackendId&) const override {
    const auto* m = dynamic_cast<const Model*>(&model);
    if (!m) throw ConfigError("model was not trained by algorithm mset2");
    return cstress_b200::estimate(m->model, observations);
  }
};

// estimator.cpp:42-60 -- the baseline predictor (column means).  Host code,
// as in the reference: a column mean is not worth a device round trip.
class MeanPredictor final : public PrognosticAlgorithm {
 public:
  struct Model final : PrognosticModel {
    std::vector<double> means;
  };
  std::string name() const override { return "mean"; }
  std::unique_ptr<PrognosticModel> train(const SignalMatrix& training, Index, const KernelConfig&,
                                         const BackendId&) const override {
    auto out = std::make_unique<Model>();
    const Index N = training.n_observations(), n = training.n_signals();
    out->means.assign(size_t(n), 0.0);
    for (Index s = 0; s < n; ++s) {
      double acc = 0.0;
      for (Index t = 0; t < N; ++t) acc += training.data(t, s);
      out->means[size_t(s)] = acc / double(N);
    }
    return out;
  }
  EstimationResult estimate(const PrognosticModel& model, const SignalMatrix& observations,
                            const BackendId&) const override {
    const auto* m = dynamic_cast<const Model*>(&model);
    if (!m) throw ConfigError("model was not trained by algorithm mean");
    const Index N = observations.n_observations(), n = observations.n_signals();
    if (n != Index(m->means.size())) throw ShapeError("mean predictor: signal count mismatch");
    EstimationResult r{Matrix(N, n), Matrix(N, n)};
    for (Index s = 0; s < n; ++s)
      for (Index t = 0; t < N; ++t) {
        r.estimates(t, s) = m->means[size_t(s)];
        r.residuals(t, s) = observations.data(t, s) - m->means[size_t(s)];
      }
    return r;
  }
};

inline const PrognosticAlgorithm& algorithm_by_name(const std::string& name) {  // estimator.cpp:63-69
  static const MsetAlgorithm mset;
  static const MeanPredictor mean;
  if (name == "mset2") return mset;
  if (name == "mean") return mean;
  throw ConfigError("unknown estimator: " + name);
}

// ------------------------------------------------------------- signals.hpp
inline SignalMatrix synthesize_uniform(Index n, Index N, double phi, double rho, double variance,
                                       double skewness, double kurtosis, uint64_t seed) {
  SignalMatrix s{Matrix(N, n)};
  check(cs_synthesize_uniform(n, N, phi, rho, variance, skewness, kurtosis, seed, s.data.data()));
  return s;
}

}  // namespace cstress_b200
