// synth.cuh -- device-side data feed: synthesize (signals.cpp:205-254) for
// SignalSpec::uniform specs (signals.cpp:51-65) on the GPU.
//
// Same generator as the reference, parallelised:
//  * SplitMix64 is a counter generator: draw k of a channel stream is
//    mix(seed_s + k*gamma), so Box-Muller pair p (draws 2p+1, 2p+2; cos for the
//    even Gaussian, sin for the odd one, rng.hpp:162-176) is random-access.
//  * AR(1) x_t = phi x_{t-1} + g_t is a linear recurrence: chunks of kChunkT
//    samples run from a zero state in parallel, then chunk carries are chained
//    (one thread per channel) and added back as phi^(i+1) * carry.
//  * The mixing z L^T with the Cholesky factor of a compound-symmetric
//    correlation matrix (unit diagonal, uniform rho) needs O(n) work per row:
//    L(j,k) is the same value c_k for every j > k, so
//    (z L^T)(t,s) = L(s,s) z(t,s) + sum_{k<s} c_k z(t,k) is a running sum.
//  * Fleishman cubic and variance scaling are elementwise + per-column
//    population moments.
// FP64 throughout.  Tolerance parity with the host restatement (CUDA libm and
// the scan's association differ in the last bits).
#pragma once

#include "common.cuh"

namespace csb {

constexpr int kChunkT = 1024;
constexpr int kBurnIn = 1000;  // signals.hpp:12

__device__ __forceinline__ unsigned long long sm64_mix(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// Gaussian number i (0-based) of the stream seeded with `seed`.
__device__ __forceinline__ double gauss_at(unsigned long long seed, long long i) {
  const unsigned long long p = static_cast<unsigned long long>(i >> 1);
  const unsigned long long d1 = seed + (2 * p + 1) * 0x9e3779b97f4a7c15ULL;
  const unsigned long long d2 = seed + (2 * p + 2) * 0x9e3779b97f4a7c15ULL;
  // next_u64 increments the state before mixing: draw k uses state seed + k*gamma,
  // and mix() adds gamma once more -> pass state - gamma.
  const unsigned long long z1 = sm64_mix(d1 - 0x9e3779b97f4a7c15ULL);
  const unsigned long long z2 = sm64_mix(d2 - 0x9e3779b97f4a7c15ULL);
  const double u1 = (static_cast<double>(z1 >> 11) + 1.0) * 0x1.0p-53;
  const double u2 = static_cast<double>(z2 >> 11) * 0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1));
  const double th = 2.0 * 3.14159265358979323846 * u2;
  return (i & 1) ? r * sin(th) : r * cos(th);
}

// Both Gaussians of Box-Muller pair p (numbers 2p and 2p + 1): one log, one
// sqrt and one sincos for two samples.
__device__ __forceinline__ void gauss_pair(unsigned long long seed, unsigned long long p, double& g_even,
                                           double& g_odd) {
  const unsigned long long d1 = seed + (2 * p + 1) * 0x9e3779b97f4a7c15ULL;
  const unsigned long long d2 = seed + (2 * p + 2) * 0x9e3779b97f4a7c15ULL;
  const unsigned long long z1 = sm64_mix(d1 - 0x9e3779b97f4a7c15ULL);
  const unsigned long long z2 = sm64_mix(d2 - 0x9e3779b97f4a7c15ULL);
  const double u1 = (static_cast<double>(z1 >> 11) + 1.0) * 0x1.0p-53;
  const double u2 = static_cast<double>(z2 >> 11) * 0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1));
  const double th = 2.0 * 3.14159265358979323846 * u2;
  double sn, cs;
  sincos(th, &sn, &cs);
  g_even = r * cs;
  g_odd = r * sn;
}

// per-channel stream seeds derive_seed(seed, {s}) (rng.hpp:26-33)
__global__ void synth_seeds_kernel(unsigned long long seed, int n, unsigned long long* seeds) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  unsigned long long h = sm64_mix(seed);
  h = sm64_mix(h ^ sm64_mix(static_cast<unsigned long long>(s)));
  seeds[s] = h;
}

// burn-in state after g_0 and 1000 updates (signals.cpp:217-219), one thread
// per channel.
__global__ void synth_burnin_kernel(const unsigned long long* seeds, int n, double phi,
                                    double* state0) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  double st = gauss_at(seeds[s], 0);
  for (int t = 1; t <= kBurnIn; ++t) st = phi * st + gauss_at(seeds[s], t);
  state0[s] = st;
}

// local recurrences from a zero state; thread = (channel, chunk)
__global__ void synth_ar_local_kernel(const unsigned long long* seeds, int n, int64_t N, double phi,
                                      double* out, double* chunk_end) {
  const int64_t chunks = (N + kChunkT - 1) / kChunkT;
  const int64_t id = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (id >= chunks * n) return;
  const int s = static_cast<int>(id / chunks);
  const int64_t c = id % chunks;
  const int64_t t0 = c * kChunkT, t1 = min(N, t0 + kChunkT);
  const unsigned long long seed = seeds[s];
  double st = 0.0;
  double held = 0.0;  // odd member of the current pair
  for (int64_t t = t0; t < t1; ++t) {
    const long long i = kBurnIn + 1 + t;
    double g;
    if (i & 1) {
      if (t == t0) {
        double ge;
        gauss_pair(seed, static_cast<unsigned long long>(i >> 1), ge, g);
      } else {
        g = held;
      }
    } else {
      gauss_pair(seed, static_cast<unsigned long long>(i >> 1), g, held);
    }
    st = phi * st + g;
    out[t + s * N] = st;
  }
  chunk_end[id] = st;
}

// carry into each chunk (sequential over chunks, one thread per channel)
__global__ void synth_ar_carry_kernel(const double* state0, const double* chunk_end, int n, int64_t N,
                                      double phi, double* carry) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int64_t chunks = (N + kChunkT - 1) / kChunkT;
  const double phiC = pow(phi, static_cast<double>(kChunkT));
  double cin = state0[s];  // state before the first chunk
  for (int64_t c = 0; c < chunks; ++c) {
    carry[s * chunks + c] = cin;
    const int64_t len = min(static_cast<int64_t>(kChunkT), N - c * kChunkT);
    const double pl = len == kChunkT ? phiC : pow(phi, static_cast<double>(len));
    cin = pl * cin + chunk_end[s * chunks + c];
  }
}

// phi^(i + 1) for i < kChunkT (the same pow values the apply pass used to
// compute per element: an FP64 pow per sample made that pass compute-bound)
__global__ void synth_phi_pow_kernel(double phi, double* phipow) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < kChunkT) phipow[i] = pow(phi, static_cast<double>(i + 1));
}

__global__ void synth_ar_apply_kernel(const double* carry, const double* __restrict__ phipow, int n, int64_t N,
                                      double* out) {
  const int64_t total = static_cast<int64_t>(n) * N;
  const int64_t chunks = (N + kChunkT - 1) / kChunkT;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = e / N, t = e % N;
    const int64_t c = t / kChunkT, i = t % kChunkT;
    out[e] += phipow[i] * carry[s * chunks + c];
  }
}

// per-column mean and population std (block per column, tree reduction)
__global__ void __launch_bounds__(256) col_moments_kernel(const double* X, int64_t N, double* mean,
                                                          double* sd) {
  __shared__ double red[256];
  const int64_t s = blockIdx.x;
  const double* col = X + s * N;
  double a = 0.0;
  for (int64_t t = threadIdx.x; t < N; t += blockDim.x) a += col[t];
  red[threadIdx.x] = a;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  const double mu = red[0] / static_cast<double>(N);
  __syncthreads();
  double b = 0.0;
  for (int64_t t = threadIdx.x; t < N; t += blockDim.x) {
    const double d = col[t] - mu;
    b += d * d;
  }
  red[threadIdx.x] = b;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    mean[s] = mu;
    sd[s] = sqrt(red[0] / static_cast<double>(N));
  }
}

// standardise (signals.cpp:224-227), mix with the compound-symmetric
// Cholesky factor (diag[s] = L(s,s), below[k] = L(j,k) for j > k) and apply
// the Fleishman cubic (signals.cpp:241-248) in the same pass.
__global__ void synth_std_mix_kernel(double* X, int n, int64_t N, const double* mean, const double* sd,
                                     const double* diag, const double* below, int mix, double fa, double fb,
                                     double fc, double fd) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= N) return;
  double acc = 0.0;
  for (int s = 0; s < n; ++s) {
    double v = X[t + s * N];
    const double d = sd[s] > 0.0 ? sd[s] : 1.0;
    v = (v - mean[s]) / d;
    double o = v;
    if (mix) {
      o = diag[s] * v + acc;
      acc += below[s] * v;
    }
    X[t + s * N] = fa + o * (fb + o * (fc + o * fd));
  }
}

// per-channel variance factor sqrt(variance) / sd (signals.cpp:249-251),
// formed once per channel instead of per element
__global__ void synth_scale_factor_kernel(const double* sd, int n, double variance, double* f) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n) f[s] = sqrt(variance) / (sd[s] > 0.0 ? sd[s] : 1.0);
}

__global__ void synth_scale_kernel(double* X, int n, int64_t N, const double* __restrict__ f) {
  const int64_t total = static_cast<int64_t>(n) * N;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    X[e] *= f[e / N];
}

}  // namespace csb
