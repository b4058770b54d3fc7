// synth.cpp -- data feed for the sweep / bench: deterministic synthetic
// signals (synthesize, signals.cpp:205-254) for SignalSpec::uniform specs
// (signals.cpp:51-65), plus the seed-derivation helpers (rng.hpp:15-83,
// sweep.cpp:119-126).
//
// Untimed in the reference harness (sweep.cpp:207-208).  Channels are
// generated in parallel host threads (each channel's SplitMix64 substream is
// independent, rng.hpp:26-33), the Cholesky mix and the Fleishman cubic run
// over row blocks in parallel; every output element is computed in the same
// sequential order as a single-threaded run, so results do not depend on the
// thread count.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "cstress_b200.h"

// The C-ABI error channel lives in cstress_b200.cu; synthesis reports through
// a setter it exports.
extern "C" cs_status cs__set_error(cs_status code, const char* msg);

namespace {


uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

struct Gauss {  // rng.hpp:135-182: SplitMix64 + Box-Muller, cos first
  uint64_t state;
  bool spare_ok = false;
  double spare = 0.0;
  explicit Gauss(uint64_t seed) : state(seed) {}
  uint64_t next_u64() {
    state += 0x9e3779b97f4a7c15ULL;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double next() {
    if (spare_ok) {
      spare_ok = false;
      return spare;
    }
    const double u1 = (static_cast<double>(next_u64() >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = static_cast<double>(next_u64() >> 11) * 0x1.0p-53;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double th = 2.0 * M_PI * u2;
    spare = r * std::sin(th);
    spare_ok = true;
    return r * std::cos(th);
  }
};

template <typename F>
void parallel_for(int64_t count, F&& f) {
  const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  const int workers = static_cast<int>(std::min<int64_t>(hw, std::max<int64_t>(count, 1)));
  if (workers <= 1) {
    for (int64_t i = 0; i < count; ++i) f(i);
    return;
  }
  std::vector<std::thread> pool;
  for (int w = 0; w < workers; ++w)
    pool.emplace_back([&, w] {
      for (int64_t i = count * w / workers; i < count * (w + 1) / workers; ++i) f(i);
    });
  for (auto& t : pool) t.join();
}

// Fleishman system (signals.cpp:24-47) and damped Newton (signals.cpp:105-164)
void fl_res(double b, double c, double d, double g1, double g2, double f[3], double J[3][3]) {
  f[0] = b * b + 6.0 * b * d + 2.0 * c * c + 15.0 * d * d - 1.0;
  f[1] = 2.0 * c * (b * b + 24.0 * b * d + 105.0 * d * d + 2.0) - g1;
  f[2] = 24.0 * (b * d + c * c * (1.0 + b * b + 28.0 * b * d) +
                 d * d * (12.0 + 48.0 * b * d + 141.0 * c * c + 225.0 * d * d)) - g2;
  J[0][0] = 2.0 * b + 6.0 * d;
  J[0][1] = 4.0 * c;
  J[0][2] = 6.0 * b + 30.0 * d;
  J[1][0] = 2.0 * c * (2.0 * b + 24.0 * d);
  J[1][1] = 2.0 * (b * b + 24.0 * b * d + 105.0 * d * d + 2.0);
  J[1][2] = 2.0 * c * (24.0 * b + 210.0 * d);
  J[2][0] = 24.0 * (d + c * c * (2.0 * b + 28.0 * d) + 48.0 * d * d * d);
  J[2][1] = 24.0 * (2.0 * c * (1.0 + b * b + 28.0 * b * d) + 282.0 * c * d * d);
  J[2][2] = 24.0 * (b + 28.0 * b * c * c + 2.0 * d * (12.0 + 48.0 * b * d + 141.0 * c * c + 225.0 * d * d) +
                    d * d * (48.0 * b + 450.0 * d));
}

void solve3(double A[3][3], const double rhs[3], double x[3]) {  // full pivoting
  double a[3][3], b[3];
  std::memcpy(a, A, sizeof a);
  std::memcpy(b, rhs, sizeof b);
  int rp[3] = {0, 1, 2}, cp[3] = {0, 1, 2}, rank = 3;
  for (int k = 0; k < 3; ++k) {
    int pi = k, pj = k;
    double best = -1.0;
    for (int i = k; i < 3; ++i)
      for (int j = k; j < 3; ++j)
        if (std::fabs(a[rp[i]][cp[j]]) > best) {
          best = std::fabs(a[rp[i]][cp[j]]);
          pi = i;
          pj = j;
        }
    if (best == 0.0) {
      rank = k;
      break;
    }
    std::swap(rp[k], rp[pi]);
    std::swap(cp[k], cp[pj]);
    for (int i = k + 1; i < 3; ++i) {
      const double l = a[rp[i]][cp[k]] / a[rp[k]][cp[k]];
      for (int j = k; j < 3; ++j) a[rp[i]][cp[j]] -= l * a[rp[k]][cp[j]];
      b[rp[i]] -= l * b[rp[k]];
    }
  }
  double y[3] = {0, 0, 0};
  for (int k = rank - 1; k >= 0; --k) {
    double v = b[rp[k]];
    for (int j = k + 1; j < rank; ++j) v -= a[rp[k]][cp[j]] * y[j];
    y[k] = v / a[rp[k]][cp[k]];
  }
  for (int k = 0; k < 3; ++k) x[cp[k]] = y[k];
}

bool fleishman(double skew, double kurt, double out[4]) {
  const double g1 = skew, g2 = kurt - 3.0;
  double x[3] = {1.0, 0.0, 0.0}, f[3], J[3][3];
  fl_res(x[0], x[1], x[2], g1, g2, f, J);
  auto inf = [](const double v[3]) { return std::max({std::fabs(v[0]), std::fabs(v[1]), std::fabs(v[2])}); };
  auto fin = [](const double v[3]) { return std::isfinite(v[0]) && std::isfinite(v[1]) && std::isfinite(v[2]); };
  for (int it = 0; it < 200 && !(inf(f) < 1e-10); ++it) {
    double step[3];
    solve3(J, f, step);
    if (!fin(step)) break;
    const double f0 = f[0] * f[0] + f[1] * f[1] + f[2] * f[2];
    double lambda = 1.0, xn[3], fn[3], Jn[3][3];
    bool ok = false;
    while (lambda >= 1.0 / 1024.0) {
      for (int i = 0; i < 3; ++i) xn[i] = x[i] - lambda * step[i];
      fl_res(xn[0], xn[1], xn[2], g1, g2, fn, Jn);
      if (fin(fn) && fn[0] * fn[0] + fn[1] * fn[1] + fn[2] * fn[2] < f0) {
        ok = true;
        break;
      }
      lambda *= 0.5;
    }
    if (!ok) break;
    std::memcpy(x, xn, sizeof x);
    std::memcpy(f, fn, sizeof f);
    std::memcpy(J, Jn, sizeof J);
  }
  if (!(inf(f) < 1e-10)) return false;
  out[0] = -x[1];
  out[1] = x[0];
  out[2] = x[1];
  out[3] = x[2];
  return true;
}

// Cholesky of the uniform correlation matrix with the jitter ladder
// (nearest_psd_repair, signals.cpp:166-203); L lower, stored ROW-major
// (L[i * n + j] = L(i, j)) so the inner sums over j walk contiguous memory
// -- the same products in the same order as Eigen's LLT (and the oracle).
bool chol_uniform(int64_t n, double rho, std::vector<double>& L) {
  std::vector<double> tried = {0.0};
  double last = 0.0;
  for (double j = 1e-12; j <= 1e-6; j *= 100.0) {
    tried.push_back(j);
    last = j;
  }
  if (1e-6 > last) tried.push_back(1e-6);
  for (double jit : tried) {
    L.assign(static_cast<size_t>(n * n), 0.0);
    auto A = [&](int64_t i, int64_t j) {
      if (i == j) return 1.0;
      return jit > 0.0 ? rho / (1.0 + jit) : rho;
    };
    bool ok = true;
    for (int64_t k = 0; k < n && ok; ++k) {
      double* lk = L.data() + k * n;
      double x = A(k, k);
      for (int64_t j = 0; j < k; ++j) x -= lk[j] * lk[j];
      if (!(x > 0.0)) {
        ok = false;
        break;
      }
      x = std::sqrt(x);
      lk[k] = x;
      for (int64_t i = k + 1; i < n; ++i) {
        double* li = L.data() + i * n;
        double v = A(i, k);
        for (int64_t j = 0; j < k; ++j) v -= li[j] * lk[j];
        li[k] = v / x;
      }
    }
    if (ok) return true;
  }
  return false;
}

double pop_std(const double* x, int64_t N) {
  double s = 0.0;
  for (int64_t t = 0; t < N; ++t) s += x[t];
  const double mean = s / static_cast<double>(N);
  double ss = 0.0;
  for (int64_t t = 0; t < N; ++t) {
    const double d = x[t] - mean;
    ss += d * d;
  }
  return std::sqrt(ss / static_cast<double>(N));
}

}  // namespace

extern "C" {

uint64_t cs_derive_seed(uint64_t parent, const uint64_t* coords, int ncoords) {
  uint64_t h = mix64(parent);
  for (int i = 0; i < ncoords; ++i) h = mix64(h ^ mix64(coords[i]));
  return h;
}

uint64_t cs_cell_data_seed(uint64_t master, int64_t n, int64_t N, int64_t m, int r) {
  const uint64_t c[4] = {static_cast<uint64_t>(n), static_cast<uint64_t>(N), static_cast<uint64_t>(m),
                         static_cast<uint64_t>(r)};
  return cs_derive_seed(master, c, 4);
}

cs_status cs_synthesize_uniform(int64_t n, int64_t N, double phi, double rho, double variance,
                                double skewness, double kurtosis, uint64_t seed, double* out);
}


// SignalSpec::validate (signals.cpp:67-103) for a uniform spec plus the
// Fleishman solve (signals.cpp:105-164); shared by the host and device feeds.
extern "C" cs_status csb_prepare_uniform(int64_t n, int64_t N, double phi, double rho, double variance,
                                         double skewness, double kurtosis, double fc[4]) {
  if (n < 1) return cs__set_error(CS_CONFIG_ERROR, "SignalSpec: n_signals must be >= 1");
  if (N < 1) return cs__set_error(CS_CONFIG_ERROR, "SignalSpec: n_observations must be >= 1");
  if (!(std::fabs(phi) < 1.0))
    return cs__set_error(CS_CONFIG_ERROR, "SignalSpec: ar_coefficient must lie in (-1, 1)");
  if (n > 1) {
    const double mine = std::min(1.0 - rho, 1.0 + static_cast<double>(n - 1) * rho);
    if (mine < -1e-10)
      return cs__set_error(CS_BAD_CORRELATION, "SignalSpec: cross_correlation has eigenvalues below -1e-10");
  }
  if (!(variance > 0.0)) return cs__set_error(CS_CONFIG_ERROR, "SignalSpec: variance_target must be > 0");
  const double bound = skewness * skewness + 1.0;
  if (!(kurtosis > bound)) {
    char buf[256];
    std::snprintf(buf, sizeof buf,
                  "SignalSpec: kurtosis_target %g for signal 0 violates the Pearson bound (must "
                  "exceed skewness^2 + 1 = %g)",
                  kurtosis, bound);
    return cs__set_error(CS_MOMENT_INFEASIBLE, buf);
  }
  if (!fleishman(skewness, kurtosis, fc)) {
    char buf[160];
    std::snprintf(buf, sizeof buf, "no real Fleishman solution for skewness %g, kurtosis %g", skewness,
                  kurtosis);
    return cs__set_error(CS_MOMENT_INFEASIBLE, buf);
  }
  return CS_OK;
}

// Cholesky factor of the compound-symmetric correlation matrix (unit
// diagonal, off-diagonal rho) with the jitter ladder of nearest_psd_repair
// (signals.cpp:166-203), in closed form: eliminating variable k leaves a
// Schur complement that is again compound symmetric (diagonal a, off-diagonal
// b), so L(k,k) = sqrt(a) and L(j,k) = b / sqrt(a) for every j > k.
bool csb_uniform_cholesky(int64_t n, double rho, std::vector<double>& diag, std::vector<double>& below) {
  std::vector<double> tried = {0.0};
  double last = 0.0;
  for (double j = 1e-12; j <= 1e-6; j *= 100.0) {
    tried.push_back(j);
    last = j;
  }
  if (1e-6 > last) tried.push_back(1e-6);
  diag.assign(static_cast<size_t>(n), 0.0);
  below.assign(static_cast<size_t>(n), 0.0);
  for (double jit : tried) {
    double a = 1.0, b = jit > 0.0 ? rho / (1.0 + jit) : rho;
    bool ok = true;
    for (int64_t k = 0; k < n; ++k) {
      if (!(a > 0.0)) {
        ok = false;
        break;
      }
      const double l = std::sqrt(a);
      const double c = b / l;
      diag[k] = l;
      below[k] = c;
      a -= c * c;
      b -= c * c;
    }
    if (ok) return true;
  }
  return false;
}

extern "C" cs_status cs_synthesize_uniform(int64_t n, int64_t N, double phi, double rho,
                                           double variance, double skewness, double kurtosis,
                                           uint64_t seed, double* out) {
  // SignalSpec::validate (signals.cpp:67-103) for the uniform spec
  if (n < 1) return cs__set_error(CS_CONFIG_ERROR, "SignalSpec: n_signals must be >= 1");
  if (N < 1) return cs__set_error(CS_CONFIG_ERROR, "SignalSpec: n_observations must be >= 1");
  if (!(std::fabs(phi) < 1.0))
    return cs__set_error(CS_CONFIG_ERROR, "SignalSpec: ar_coefficient must lie in (-1, 1)");
  if (n > 1) {
    const double mine = std::min(1.0 - rho, 1.0 + static_cast<double>(n - 1) * rho);
    if (mine < -1e-10)
      return cs__set_error(CS_BAD_CORRELATION, "SignalSpec: cross_correlation has eigenvalues below -1e-10");
  }
  if (!(variance > 0.0)) return cs__set_error(CS_CONFIG_ERROR, "SignalSpec: variance_target must be > 0");
  const double bound = skewness * skewness + 1.0;
  if (!(kurtosis > bound)) {
    char buf[256];
    std::snprintf(buf, sizeof buf,
                  "SignalSpec: kurtosis_target %g for signal 0 violates the Pearson bound (must "
                  "exceed skewness^2 + 1 = %g)",
                  kurtosis, bound);
    return cs__set_error(CS_MOMENT_INFEASIBLE, buf);
  }
  double fc[4];
  if (!fleishman(skewness, kurtosis, fc)) {
    char buf[160];
    std::snprintf(buf, sizeof buf, "no real Fleishman solution for skewness %g, kurtosis %g", skewness,
                  kurtosis);
    return cs__set_error(CS_MOMENT_INFEASIBLE, buf);
  }
  std::vector<double> L;
  if (n > 1 && !chol_uniform(n, rho, L)) {
    return cs__set_error(CS_BAD_CORRELATION,
                         "correlation matrix not positive semidefinite within jitter cap 1e-06");
  }
  // (1)-(2) AR(1) streams, standardised (signals.cpp:214-228)
  parallel_for(n, [&](int64_t s) {
    const uint64_t c = static_cast<uint64_t>(s);
    Gauss g(cs_derive_seed(seed, &c, 1));
    double state = g.next();
    for (int64_t t = 0; t < 1000; ++t) state = phi * state + g.next();
    double* col = out + s * N;
    for (int64_t t = 0; t < N; ++t) {
      state = phi * state + g.next();
      col[t] = state;
    }
    double sum = 0.0;
    for (int64_t t = 0; t < N; ++t) sum += col[t];
    const double mean = sum / static_cast<double>(N);
    double sd = pop_std(col, N);
    if (sd <= 0.0) sd = 1.0;
    for (int64_t t = 0; t < N; ++t) col[t] = (col[t] - mean) / sd;
  });
  // (3) z * L^T (signals.cpp:231-236), row blocks in parallel
  if (n > 1) {
    const int64_t block = 4096;
    parallel_for((N + block - 1) / block, [&](int64_t b) {
      std::vector<double> row(static_cast<size_t>(n));
      const int64_t t1 = std::min(N, (b + 1) * block);
      for (int64_t t = b * block; t < t1; ++t) {
        for (int64_t k = 0; k < n; ++k) row[k] = out[t + k * N];
        for (int64_t s = 0; s < n; ++s) {
          double acc = 0.0;
          const double* ls = L.data() + s * n;  // row s of L (row-major)
          for (int64_t k = 0; k <= s; ++k) acc += row[k] * ls[k];
          out[t + s * N] = acc;
        }
      }
    });
  }
  // (4)-(5) Fleishman cubic and variance scaling (signals.cpp:240-251)
  parallel_for(n, [&](int64_t s) {
    double* col = out + s * N;
    for (int64_t t = 0; t < N; ++t) {
      const double v = col[t];
      col[t] = fc[0] + v * (fc[1] + v * (fc[2] + v * fc[3]));
    }
    double sd = pop_std(col, N);
    if (sd <= 0.0) sd = 1.0;
    const double f = std::sqrt(variance) / sd;
    for (int64_t t = 0; t < N; ++t) col[t] *= f;
  });
  return cs__set_error(CS_OK, "");
}
