// kernels_f64.cuh -- FP64 kernels of the training path and of the FP64
// (reference-association) surveillance path.
//
// Design: the reference computes everything in FP64 with a fixed left-to-right
// accumulation order and no FMA contraction (backends.cpp:129-152,
// :217-231; x86-64 baseline build).  B200 has no FP64 tensor-core kind in
// tcgen05, so these are SIMT DMUL/DADD kernels.  Every accumulation below is
// written with __dmul_rn / __dadd_rn / __dsub_rn in ascending depth order, so
// each output element is produced by exactly the reference's operation
// sequence:
//   * sim_exact  == sim_matrix_reference  (bitwise for inverse_distance;
//                                          Gaussian differs only by CUDA exp)
//   * gemm_exact == matmul_reference      (bitwise)
// Tiles: 64x64 outputs per 256-thread CTA, 4x4 register block per thread,
// depth staged through shared memory in chunks of 16 with coalesced global
// loads.  FP64 here is issue-bound (2-3 DP ops per MAC), not HBM-bound.
#pragma once

#include "common.cuh"

namespace csb {

constexpr int kTile = 64;
constexpr int kChunk = 16;
constexpr int kThreads = 256;

__device__ __forceinline__ double kernel_from_d2(double d2, int kind, double h) {
  // kernels.hpp:54-57.  IEEE sqrt / div (nvcc default -prec-div/-prec-sqrt).
  if (kind == CS_KERNEL_GAUSSIAN) return exp(-d2 / __dmul_rn(__dmul_rn(2.0, h), h));
  return 1.0 / __dadd_rn(1.0, sqrt(d2) / h);
}

// out(i, j) = k( sum_r (A(r,i) - B(r,j))^2 ),  A: n x p (lda), B: n x q (ldb).
// backends.cpp:129-152: r ascending, d2 += d*d unfused.
__global__ void __launch_bounds__(kThreads)
sim_exact_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ B,
                 int64_t ldb, int64_t n, int64_t p, int64_t q, int kind, double h,
                 double* __restrict__ out, int64_t ldo) {
  __shared__ double As[kChunk][kTile + 1];
  __shared__ double Bs[kChunk][kTile + 1];
  const int t = threadIdx.x;
  const int tx = t % 16, ty = t / 16;
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kTile;
  const int64_t j0 = static_cast<int64_t>(blockIdx.y) * kTile;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;

  for (int64_t r0 = 0; r0 < n; r0 += kChunk) {
    // coalesced: 16 consecutive threads read 16 consecutive depth values
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int rr = t % kChunk;
      const int cc = t / kChunk + 16 * l;
      const int64_t r = r0 + rr;
      const int64_t i = i0 + cc, j = j0 + cc;
      As[rr][cc] = (r < n && i < p) ? A[r + i * lda] : 0.0;
      Bs[rr][cc] = (r < n && j < q) ? B[r + j * ldb] : 0.0;
    }
    __syncthreads();
    const int rmax = static_cast<int>(n - r0 < kChunk ? n - r0 : kChunk);
    for (int rr = 0; rr < rmax; ++rr) {
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[rr][tx + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = Bs[rr][ty + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const double d = __dsub_rn(av[a], bv[b]);
          acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(d, d));
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int64_t j = j0 + ty + 16 * b;
    if (j >= q) continue;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int64_t i = i0 + tx + 16 * a;
      if (i < p) out[i + j * ldo] = kernel_from_d2(acc[a][b], kind, h);
    }
  }
}

// C(p x q) = op(A)(p x k) * op(B)(k x q); ascending k, acc += a*b unfused
// (backends.cpp:217-231; matmul_optimized :233-272 has the same per-element
// order, so both reference backends are matched bitwise).
template <bool TA, bool TB>
__global__ void __launch_bounds__(kThreads)
gemm_exact_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ B,
                  int64_t ldb, int64_t p, int64_t k, int64_t q, double* __restrict__ C,
                  int64_t ldc) {
  __shared__ double As[kChunk][kTile + 1];
  __shared__ double Bs[kChunk][kTile + 1];
  const int t = threadIdx.x;
  const int tx = t % 16, ty = t / 16;
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kTile;
  const int64_t j0 = static_cast<int64_t>(blockIdx.y) * kTile;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;

  for (int64_t k0 = 0; k0 < k; k0 += kChunk) {
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      if (!TA) {  // A(i, kk) at A[i + kk*lda]: coalesce along i
        const int ii = t % kTile, kk = t / kTile + 4 * l;
        const int64_t i = i0 + ii, kg = k0 + kk;
        As[kk][ii] = (i < p && kg < k) ? A[i + kg * lda] : 0.0;
      } else {    // A stored k x p: op(A)(i, kk) = A[kk + i*lda]: coalesce along kk
        const int kk = t % kChunk, ii = t / kChunk + 16 * l;
        const int64_t i = i0 + ii, kg = k0 + kk;
        As[kk][ii] = (i < p && kg < k) ? A[kg + i * lda] : 0.0;
      }
      if (!TB) {  // B(kk, j) at B[kk + j*ldb]: coalesce along kk
        const int kk = t % kChunk, jj = t / kChunk + 16 * l;
        const int64_t j = j0 + jj, kg = k0 + kk;
        Bs[kk][jj] = (j < q && kg < k) ? B[kg + j * ldb] : 0.0;
      } else {    // B stored q x k: op(B)(kk, j) = B[j + kk*ldb]: coalesce along j
        const int jj = t % kTile, kk = t / kTile + 4 * l;
        const int64_t j = j0 + jj, kg = k0 + kk;
        Bs[kk][jj] = (j < q && kg < k) ? B[j + kg * ldb] : 0.0;
      }
    }
    __syncthreads();
    const int kmax = static_cast<int>(k - k0 < kChunk ? k - k0 : kChunk);
    for (int kk = 0; kk < kmax; ++kk) {
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = As[kk][tx + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = Bs[kk][ty + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(av[a], bv[b]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int64_t j = j0 + ty + 16 * b;
    if (j >= q) continue;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int64_t i = i0 + tx + 16 * a;
      if (i < p) C[i + j * ldc] = acc[a][b];
    }
  }
}

// Dn(s, c) = D(s, c) / scale[s]   (mset.cpp:147-149; division, not reciprocal)
__global__ void div_rows_kernel(const double* __restrict__ D, const double* __restrict__ scale,
                                int64_t n, int64_t m, double* __restrict__ Dn) {
  const int64_t total = n * m;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    Dn[e] = D[e] / scale[e % n];
  }
}

// xn(s, t) = obs(t, s) / scale[s]: transpose N x n (ld) -> n x Nc through smem
// (mset.cpp:186-187).
__global__ void transpose_div_kernel(const double* __restrict__ obs, int64_t ld, int64_t t0,
                                     int64_t Nc, int64_t n, const double* __restrict__ scale,
                                     double* __restrict__ xn) {
  __shared__ double tile[32][33];
  const int64_t tb = static_cast<int64_t>(blockIdx.x) * 32;  // time
  const int64_t sb = static_cast<int64_t>(blockIdx.y) * 32;  // signal
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t t = tb + threadIdx.x, s = sb + k;
    if (t < Nc && s < n) tile[k][threadIdx.x] = obs[(t0 + t) + s * ld] / scale[s];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t s = sb + threadIdx.x, t = tb + k;
    if (t < Nc && s < n) xn[s + t * n] = tile[threadIdx.x][k];
  }
}

// est(t, s) = en(s, t) * scale[s];  resid(t, s) = obs(t, s) - est(t, s)
// (mset.cpp:193-197).
__global__ void finish_estimate_kernel(const double* __restrict__ en, int64_t Nc, int64_t n,
                                       const double* __restrict__ scale,
                                       const double* __restrict__ obs, int64_t ld, int64_t t0,
                                       double* __restrict__ est, double* __restrict__ resid) {
  __shared__ double tile[32][33];
  const int64_t tb = static_cast<int64_t>(blockIdx.x) * 32;
  const int64_t sb = static_cast<int64_t>(blockIdx.y) * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t s = sb + threadIdx.x, t = tb + k;
    if (t < Nc && s < n) tile[k][threadIdx.x] = __dmul_rn(en[s + t * n], scale[s]);
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t t = tb + threadIdx.x, s = sb + k;
    if (t < Nc && s < n) {
      const double e = tile[threadIdx.x][k];
      const int64_t g = (t0 + t) + s * ld;
      if (est) est[g] = e;
      if (resid) resid[g] = __dsub_rn(obs[g], e);
    }
  }
}

// Population std per column, sequential sums (mset.cpp:44-53, mean restated
// as a left-to-right sum; identical to the oracle).  One warp per column:
// the lanes load 32 consecutive rows per instruction (coalesced 256 bytes,
// four blocks in flight), and every lane runs the same left-to-right sum
// over the block, values broadcast by shuffle -- the serial DADD chain is
// the only latency left (the previous 32-columns-per-warp layout ran on
// n / 32 SMs behind a CTA barrier per 64 rows).
__global__ void __launch_bounds__(128)
scale_seq_kernel(const double* __restrict__ X, int64_t N, int64_t n, double* __restrict__ scale) {
  const int lane = threadIdx.x & 31;
  const int64_t s = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (s >= n) return;
  const double* col = X + s * N;
  constexpr int kAhead = 8;  // blocks of 32 rows per group (two groups in flight)
  auto block_sum = [&](double acc, double v, int rows, double mean, bool sq) {
    // eight broadcasts in flight ahead of the serial adds: the chain then
    // waits on DADD latency only, not on a shuffle per element
    for (int q0 = 0; q0 < rows; q0 += 8) {
      double xs[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) xs[u] = __shfl_sync(0xffffffffu, v, (q0 + u) & 31);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (q0 + u >= rows) break;
        if (sq) {
          const double d = __dsub_rn(xs[u], mean);
          acc = __dadd_rn(acc, __dmul_rn(d, d));
        } else {
          acc = __dadd_rn(acc, xs[u]);
        }
      }
    }
    return acc;
  };
  double mean = 0.0, acc = 0.0;
  // software pipelined: the next kAhead blocks are in flight while the
  // serial sum runs over the current ones (one memory latency per column,
  // not one per block group)
  auto load = [&](double* v, int64_t t0) {
#pragma unroll
    for (int k = 0; k < kAhead; ++k) {
      const int64_t t = t0 + 32 * k + lane;
      v[k] = t < N ? __ldg(col + t) : 0.0;
    }
  };
  for (int pass = 0; pass < 2; ++pass) {
    acc = 0.0;
    double v[kAhead], vn[kAhead];
    load(v, 0);
    for (int64_t t0 = 0; t0 < N; t0 += 32 * kAhead) {
      if (t0 + 32 * kAhead < N) load(vn, t0 + 32 * kAhead);
#pragma unroll
      for (int k = 0; k < kAhead; ++k) {
        const int64_t b0 = t0 + 32 * k;
        if (b0 >= N) break;
        const int rows = N - b0 < 32 ? static_cast<int>(N - b0) : 32;
        acc = block_sum(acc, v[k], rows, mean, pass == 1);
      }
#pragma unroll
      for (int k = 0; k < kAhead; ++k) v[k] = vn[k];
    }
    if (pass == 0) mean = acc / static_cast<double>(N);
  }
  if (lane == 0) {
    const double sd = sqrt(acc / static_cast<double>(N));
    scale[s] = sd > 1e-12 ? sd : 1e-12;
  }
}

// max|G| and max|G - G^T| for the symmetric_eig precondition (mset.cpp:60-64).
__global__ void symmetry_stats_kernel(const double* __restrict__ G, int64_t m,
                                      unsigned long long* __restrict__ out /* [2] as bits */) {
  double mag = 0.0, asym = 0.0;
  const int64_t total = m * m;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    const double v = G[e];
    mag = fmax(mag, fabs(v));
    asym = fmax(asym, fabs(v - G[j + i * m]));
  }
  // non-negative doubles order like their bit patterns
  for (int o = 16; o > 0; o >>= 1) {
    mag = fmax(mag, __shfl_xor_sync(0xffffffffu, mag, o));
    asym = fmax(asym, __shfl_xor_sync(0xffffffffu, asym, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&out[0], static_cast<unsigned long long>(__double_as_longlong(mag)));
    atomicMax(&out[1], static_cast<unsigned long long>(__double_as_longlong(asym)));
  }
}

// whitened(:, k) = V(:, m - rank + k) / sqrt(lambda)  (mset.cpp:165-169; the
// kept eigenvalues of an ascending spectrum are a contiguous suffix).
__global__ void whiten_kernel(const double* __restrict__ V, const double* __restrict__ w,
                              int64_t m, int64_t rank, double* __restrict__ W) {
  const int64_t total = m * rank;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e % m, k = e / m;
    const int64_t src = m - rank + k;
    W[e] = V[r + src * m] / sqrt(w[src]);
  }
}

// Column-major m x m identity (right-hand side of potrs for the inverse).
__global__ void set_identity_kernel(double* __restrict__ A, int64_t m) {
  const int64_t total = m * m;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    A[e] = (e % m == e / m) ? 1.0 : 0.0;
}

// Inverse of each 128 x 128 diagonal block of a lower-triangular L (column-
// major, ld m) into the same block of X (lower part; X pre-zeroed): one CTA
// per block, thread j forward-substitutes column j of the block's inverse,
// L's block staged in shared memory (pitch 129).  Base case of the blocked
// triangular inversion in cstress_b200.cu (tri_inverse).
constexpr int kTriInvB = 128;
__global__ void __launch_bounds__(kTriInvB) tri_inv_diag_kernel(const double* __restrict__ L, int64_t m,
                                                                double* __restrict__ X) {
  extern __shared__ double Ls[];  // kTriInvB x (kTriInvB + 1)
  constexpr int P = kTriInvB + 1;
  const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kTriInvB;
  const int b = static_cast<int>(min(static_cast<int64_t>(kTriInvB), m - r0));
  for (int e = threadIdx.x; e < b * b; e += blockDim.x) {
    const int i = e % b, k = e / b;
    Ls[i + k * P] = L[(r0 + i) + (r0 + k) * m];
  }
  __syncthreads();
  const int j = threadIdx.x;
  if (j >= b) return;
  double* x = X + r0 + (r0 + j) * m;  // column j of the block
  x[j] = 1.0 / Ls[j + j * P];
  for (int i = j + 1; i < b; ++i) {
    double acc = 0.0;
    for (int k = j; k < i; ++k) acc = fma(Ls[i + k * P], x[k], acc);
    x[i] = -acc / Ls[i + i * P];
  }
}

// ||D(:, i)||^2 for the GEMM-form Gram matrix (FP32-precision models)
__global__ void col_sqnorm_kernel(const double* __restrict__ D, int64_t n, int64_t m, double* __restrict__ dd) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i >= m) return;
  double a = 0.0;
  for (int64_t r = 0; r < n; ++r) a = fma(D[r + i * n], D[r + i * n], a);
  dd[i] = a;
}
// G(i, j) = k(max(dd_i + dd_j - 2 S(i, j), 0)) from S = D^T D (lower triangle
// read, both triangles written: G exactly symmetric), unit diagonal exact
__global__ void gram_from_dot_kernel(double* __restrict__ G, const double* __restrict__ dd, int64_t m, int kind,
                                     double h) {
  const int64_t total = m * m;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    if (i < j) continue;
    const double v = i == j ? kernel_from_d2(0.0, kind, h)
                            : kernel_from_d2(fmax(dd[i] + dd[j] - 2.0 * G[e], 0.0), kind, h);
    G[e] = v;
    G[j + i * m] = v;
  }
}

// Mirror the lower triangle into the upper one (potri writes the lower
// triangle of the inverse only; potrs's full result is made exactly
// symmetric the same way).
__global__ void symmetrize_lower_kernel(double* __restrict__ A, int64_t m) {
  const int64_t total = m * m;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e % m, j = e / m;  // column-major (i, j)
    if (i < j) A[e] = A[j + i * m];
  }
}

// ||A||_1 = max_j sum_i |A_ij| of a column-major m x m matrix; one block per
// column, maximum folded into *out as the bit pattern of a non-negative
// double (ordered like the value).
__global__ void norm1_kernel(const double* __restrict__ A, int64_t m, unsigned long long* out) {
  __shared__ double part[32];
  for (int64_t j = blockIdx.x; j < m; j += gridDim.x) {
    double a = 0.0;
    for (int64_t i = threadIdx.x; i < m; i += blockDim.x) a += fabs(A[i + j * m]);
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x < 32) {
      a = threadIdx.x < blockDim.x / 32 ? part[threadIdx.x] : 0.0;
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (threadIdx.x == 0) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(a)));
    }
    __syncthreads();
  }
}

}  // namespace csb
