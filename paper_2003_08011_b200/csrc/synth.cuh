// synth.cuh -- device-side data feed: synthesize (signals.cpp:205-254) for
// SignalSpec::uniform specs (signals.cpp:51-65) on the GPU.
//
// Same generator as the reference, parallelised:
//  * SplitMix64 is a counter generator: draw k of a channel stream is
//    mix(seed_s + k*gamma), so Box-Muller pair p (draws 2p+1, 2p+2; cos for the
//    even Gaussian, sin for the odd one, rng.hpp:162-176) is random-access.
//  * AR(1) x_t = phi x_{t-1} + g_t is a linear recurrence: chunks of ct
//    samples run from a zero state in parallel, then chunk carries are chained
//    (one thread per channel) and added back as phi^(i+1) * carry inside
//    the standardise/mix pass; the channel moments come from per-chunk sums
//    (no separate pass over the AR streams).
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

constexpr int kChunkT = 1024;  // longest chunk (phi^(i+1) table size); the
                               // runtime chunk length ct is a power of two in
                               // [32, kChunkT], shorter when n x N is small so
                               // the sequential chunk walks stay short
constexpr int kBurnIn = 1000;  // signals.hpp:12

__device__ __forceinline__ unsigned long long sm64_mix(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
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
  // (sin, cos)(2 pi u2) as sincospi(2 u2): no argument reduction (2 u2 is
  // exact); differs from the reference's rounded 2 pi u2 in the last ulp
  double sn, cs;
  sincospi(2.0 * u2, &sn, &cs);
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

// burn-in state after g_0 and 1000 updates (signals.cpp:217-219): state0 =
// sum_t phi^(1000 - t) g_t, one warp per channel; lane L runs the recurrence
// over t in [32 L, 32 L + 32) from zero (16 Box-Muller pairs) and the lanes'
// partial states are combined with weights phi^(1000 - last t of the lane).
__global__ void synth_burnin_kernel(const unsigned long long* seeds, int n, double phi, double* state0) {
  const int lane = threadIdx.x & 31;
  const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= n) return;  // warp-uniform
  const unsigned long long seed = seeds[s];
  const int t0 = 32 * lane, t1 = min(t0 + 31, kBurnIn);  // inclusive range
  double st = 0.0;
  for (int t = t0; t <= t1; t += 2) {
    double ge, go;
    gauss_pair(seed, static_cast<unsigned long long>(t >> 1), ge, go);
    st = phi * st + ge;
    if (t + 1 <= t1) st = phi * st + go;
  }
  double v = t0 <= t1 ? pow(phi, static_cast<double>(kBurnIn - t1)) * st : 0.0;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) state0[s] = v;
}

// local recurrences from a zero state; thread = (channel, chunk).  A lane
// owns one chunk, so its own time steps are 8 KB apart from its neighbours':
// the values go through a per-warp 32 x 32 shared-memory transpose and leave
// as one coalesced 256-byte row per chunk (direct per-lane stores wrote one
// 8-byte word per 32-byte sector, 13 GB of DRAM writes for 8 GB of output).
constexpr int kArThreads = 128;
__global__ void __launch_bounds__(kArThreads) synth_ar_local_kernel(const unsigned long long* seeds, int n,
                                                                    int64_t N, int ct, double phi,
                                                                    const double* __restrict__ phipow, double* out,
                                                                    double* chunk_end, double* chunk_sums) {
  __shared__ double tile[kArThreads / 32][32][33];
  const int64_t chunks = (N + ct - 1) / ct;
  const int64_t total = chunks * n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t warp0 = blockIdx.x * static_cast<int64_t>(kArThreads) + warp * 32;
  if (warp0 >= total) return;  // whole warp idle
  const int64_t id = warp0 + lane;
  const bool active = id < total;
  const int s = active ? static_cast<int>(id / chunks) : 0;
  const int64_t c = active ? id % chunks : 0;
  const int64_t t0 = c * ct;
  const int len = active ? static_cast<int>(min(static_cast<int64_t>(ct), N - t0)) : 0;
  const unsigned long long seed = active ? seeds[s] : 0ULL;
  const long long base = static_cast<long long>(s) * N + t0;  // out offset of this lane's chunk
  double (*sm)[33] = tile[warp];
  double st = 0.0;
  double held = 0.0;  // odd member of the current pair
  double s1 = 0.0, s2 = 0.0, s3 = 0.0;  // sum l, sum l^2, sum l phi^(i+1)
  for (int k = 0; k < ct; k += 32) {
#pragma unroll 1
    for (int j = 0; j < 32; ++j) {
      const int tt = k + j;
      if (tt < len) {
        const long long i = kBurnIn + 1 + t0 + tt;
        double g;
        if (i & 1) {
          if (tt == 0) {
            double ge;
            gauss_pair(seed, static_cast<unsigned long long>(i >> 1), ge, g);
          } else {
            g = held;
          }
        } else {
          gauss_pair(seed, static_cast<unsigned long long>(i >> 1), g, held);
        }
        st = phi * st + g;
        s1 += st;
        s2 += st * st;
        s3 += st * phipow[tt];
      }
      sm[lane][j] = st;
    }
    __syncwarp();
    // row r = chunk of lane r: 32 consecutive time steps, one per lane
    for (int r = 0; r < 32; ++r) {
      const long long br = __shfl_sync(0xffffffffu, base, r);
      const int lr = __shfl_sync(0xffffffffu, len, r);
      if (k + lane < lr) out[br + k + lane] = sm[r][lane];
    }
    __syncwarp();
  }
  if (active) {
    chunk_end[id] = st;
    chunk_sums[id] = s1;
    chunk_sums[total + id] = s2;
    chunk_sums[2 * total + id] = s3;
  }
}

// carry into each chunk and the channel's moments; one warp per channel.
// The carry recurrence c_{k+1} = phi^len_k c_k + end_k is a chain of affine
// maps: 32 chunks at a time go through a shuffle scan of map compositions,
// chained block to block from the burn-in state.  The moments need no pass
// over the data: with x_t = l_t + phi^(i+1) c (l the chunk-local stream, c the
// chunk's carry, i the offset in the chunk), sum x = sum l + c G1 and sum x^2
// = sum l^2 + 2 c sum l phi^(i+1) + c^2 G2, G1 = sum phi^(i+1), G2 = sum
// phi^(2i+2) over the chunk.  Writes the mean and 1 / population std (floor
// rule signals.cpp:226).
constexpr int kCarryThreads = 128;
__global__ void __launch_bounds__(kCarryThreads) synth_ar_carry_kernel(
    const double* __restrict__ state0, const double* __restrict__ chunk_end, const double* __restrict__ chunk_sums,
    const double* __restrict__ phipow, int n, int64_t N, int ct, double phi, double* __restrict__ carry,
    double* __restrict__ mean, double* __restrict__ isd) {
  const int lane = threadIdx.x & 31;
  const int s = blockIdx.x * (kCarryThreads / 32) + (threadIdx.x >> 5);
  if (s >= n) return;  // warp-uniform
  const int64_t chunks = (N + ct - 1) / ct;
  const int64_t total = chunks * n;
  double G1 = 0.0, G2 = 0.0;
  for (int i = lane; i < ct; i += 32) {
    G1 += phipow[i];
    G2 += phipow[i] * phipow[i];
  }
  for (int o = 16; o > 0; o >>= 1) {
    G1 += __shfl_xor_sync(0xffffffffu, G1, o);
    G2 += __shfl_xor_sync(0xffffffffu, G2, o);
  }
  const double phiC = pow(phi, static_cast<double>(ct));
  double x_in = state0[s];  // state before the current 32-chunk block
  double A = 0.0, B = 0.0;
  for (int64_t c0 = 0; c0 < chunks; c0 += 32) {
    const int64_t c = c0 + lane;
    const bool ok = c < chunks;
    const int64_t id = s * chunks + c;
    int64_t len = 0;
    double a = 1.0, b = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0, g1 = G1, g2 = G2;
    if (ok) {
      len = min(static_cast<int64_t>(ct), N - c * ct);
      b = chunk_end[id];
      s1 = chunk_sums[id];
      s2 = chunk_sums[total + id];
      s3 = chunk_sums[2 * total + id];
      if (len == ct) {
        a = phiC;
      } else {
        a = pow(phi, static_cast<double>(len));
        g1 = g2 = 0.0;
        for (int i = 0; i < len; ++i) {
          g1 += phipow[i];
          g2 += phipow[i] * phipow[i];
        }
      }
    }
    // inclusive scan: (a, b) = f_lane o ... o f_0 of this block
    for (int o = 1; o < 32; o <<= 1) {
      const double ap = __shfl_up_sync(0xffffffffu, a, o);
      const double bp = __shfl_up_sync(0xffffffffu, b, o);
      if (lane >= o) {
        b = a * bp + b;
        a = a * ap;
      }
    }
    const double y = a * x_in + b;  // state after chunk `lane`
    double cin = __shfl_up_sync(0xffffffffu, y, 1);
    if (lane == 0) cin = x_in;
    if (ok) {
      carry[id] = cin;
      A += s1 + cin * g1;
      B += s2 + 2.0 * cin * s3 + cin * cin * g2;
    }
    x_in = __shfl_sync(0xffffffffu, y, 31);  // lanes past the end carry the identity map
  }
  for (int o = 16; o > 0; o >>= 1) {
    A += __shfl_xor_sync(0xffffffffu, A, o);
    B += __shfl_xor_sync(0xffffffffu, B, o);
  }
  if (lane == 0) {
    const double Nd = static_cast<double>(N), mu = A / Nd;
    mean[s] = mu;
    const double d = sqrt(fmax(B / Nd - mu * mu, 0.0));
    isd[s] = 1.0 / (d > 0.0 ? d : 1.0);
  }
}

// phi^(i + 1) for i < kChunkT (the same pow values the apply pass used to
// compute per element: an FP64 pow per sample made that pass compute-bound)
__global__ void synth_phi_pow_kernel(double phi, double* phipow) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < kChunkT) phipow[i] = pow(phi, static_cast<double>(i + 1));
}

// per-column mean and population std in one pass (block per column): sums
// of d = x - x_0 and d^2, shifted by the column's first value so the
// E[d^2] - E[d]^2 form does not cancel; exactly 0 for a constant column.
__global__ void __launch_bounds__(256) col_moments_kernel(const double* X, int64_t N, double* mean,
                                                          double* sd) {
  __shared__ double red[2][8];
  const int64_t s = blockIdx.x;
  const double* col = X + s * N;
  const double K = col[0];
  double a = 0.0, b = 0.0;
  int64_t t = threadIdx.x;
  for (; t + 3 * 256 < N; t += 4 * 256) {
    const double d0 = col[t] - K, d1 = col[t + 256] - K, d2 = col[t + 512] - K, d3 = col[t + 768] - K;
    a += (d0 + d1) + (d2 + d3);
    b += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
  }
  for (; t < N; t += 256) {
    const double d = col[t] - K;
    a += d;
    b += d * d;
  }
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = a;
    red[1][threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double A = 0.0, B = 0.0;
    for (int w = 0; w < 8; ++w) {
      A += red[0][w];
      B += red[1][w];
    }
    const double Nd = static_cast<double>(N);
    const double md = A / Nd;
    mean[s] = K + md;
    sd[s] = sqrt(fmax(B / Nd - md * md, 0.0));
  }
}

// AR value = chunk-local value + phi^(i+1) carry, standardise
// (signals.cpp:224-227; multiply by the channel's 1/sd), mix
// with the compound-symmetric Cholesky factor (diag[s] = L(s,s), below[k] =
// L(j,k) for j > k) and apply the Fleishman cubic (signals.cpp:241-248) in the
// same pass.  Thread per time step, channels in groups of four loaded ahead
// of the dependent running sum.
__global__ void synth_std_mix_kernel(double* X, int n, int64_t N, int ct_log2, const double* __restrict__ carry,
                                     const double* __restrict__ phipow, const double* __restrict__ mean,
                                     const double* __restrict__ isd, const double* __restrict__ diag,
                                     const double* __restrict__ below, int mix, double fa, double fb, double fc,
                                     double fd) {
  const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (t >= N) return;
  const int ct = 1 << ct_log2;
  const int64_t chunks = (N + ct - 1) / ct;
  const double pw = phipow[t & (ct - 1)];
  const double* cy = carry + (t >> ct_log2);
  double acc = 0.0;
  double* x = X + t;
  int s = 0;
  auto one = [&](int c, double v) {
    v = v + pw * cy[c * chunks];  // chunk-local stream + phi^(i+1) carry = AR(1) value
    v = (v - mean[c]) * isd[c];
    double o = v;
    if (mix) {
      o = diag[c] * v + acc;
      acc += below[c] * v;
    }
    x[c * N] = fa + o * (fb + o * (fc + o * fd));
  };
  for (; s + 4 <= n; s += 4) {
    const double v0 = x[s * N], v1 = x[(s + 1) * N], v2 = x[(s + 2) * N], v3 = x[(s + 3) * N];
    one(s, v0);
    one(s + 1, v1);
    one(s + 2, v2);
    one(s + 3, v3);
  }
  for (; s < n; ++s) one(s, x[s * N]);
}

// per-channel variance factor sqrt(variance) / sd (signals.cpp:249-251),
// formed once per channel instead of per element
__global__ void synth_scale_factor_kernel(const double* sd, int n, double variance, double* f) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n) f[s] = sqrt(variance) / (sd[s] > 0.0 ? sd[s] : 1.0);
}

// X(:, s) *= f[s]; block (t-range, channel), no per-element index division
constexpr int kApplyT = 2048;
__global__ void synth_scale_kernel(double* X, int64_t N, const double* __restrict__ f) {
  const double g = f[blockIdx.y];
  double* col = X + static_cast<int64_t>(blockIdx.y) * N;
#pragma unroll
  for (int k = 0; k < kApplyT / 256; ++k) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * kApplyT + k * 256 + threadIdx.x;
    if (t < N) col[t] *= g;
  }
}

// FP32 result of the variance scale: out32 = (float)(X * f[s]) (the same
// double product as synth_scale_kernel, then one rounding)
__global__ void synth_scale_f32_kernel(const double* __restrict__ X, int64_t N, const double* __restrict__ f,
                                       float* __restrict__ out32) {
  const double g = f[blockIdx.y];
  const int64_t off = static_cast<int64_t>(blockIdx.y) * N;
#pragma unroll
  for (int k = 0; k < kApplyT / 256; ++k) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * kApplyT + k * 256 + threadIdx.x;
    if (t < N) out32[off + t] = static_cast<float>(X[off + t] * g);
  }
}

}  // namespace csb
