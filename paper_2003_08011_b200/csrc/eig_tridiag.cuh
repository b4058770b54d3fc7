// eig_tridiag.cuh -- eigenvalues of a symmetric matrix without cuSOLVER:
// Householder tridiagonalisation by one thread-block cluster, then Sturm-count
// bisection.  An OPT-IN path (CSB_EIG_OWN=1) for the eigenvalues-only calls
// of the train path (the eager eigen_spectrum and the eigen route's rank
// decision, mset.cpp:153-163) up to kTriMaxM: exact to 1e-12 of max|lambda|
// against LAPACK, but measured 3-12x slower than cuSOLVER's syevd (m = 1000:
// 66 vs 12 ms), which therefore stays the default -- a one-stage reduction
// pays four cluster barriers and latency-bound L2 streams per column; the
// fast design is two-stage.
//
// Tridiagonalisation (the classical one-stage algorithm, Golub & Van Loan
// 8.3.1): for k = 0 .. m-3, a Householder reflector H = I - tau v v^T
// (v_0 = 1) maps column k below the diagonal to (beta, 0, ...); the trailing
// matrix becomes H A22 H = A22 - v w^T - w v^T with p = tau A22 v and
// w = p - (tau / 2)(p^T v) v.  cuSOLVER's blocked sytrd spends ~11 ms at
// m = 1000 on this (latency of its per-column kernels); here one cluster of
// 16 CTAs (non-portable size; 8 where 16 cannot be launched) owns the whole
// reduction: CTA c holds rows [c R, c R + R) of the full symmetric working
// matrix in global memory (L2-resident up to ~2k x 2k), every column step is
// three cluster-wide reductions through distributed shared memory (partials
// summed in rank order: deterministic) and the vectors v, w go through L2.
// Both triangles are updated with the same rounded terms, so the working
// matrix stays exactly symmetric.
//
// Bisection (LAPACK dstebz's method): count(x) = number of negative
// pivots of T - x I = number of eigenvalues < x; eigenvalue k is the point
// where the count passes k, found by bisection of the Gershgorin interval to
// the last bit.  Each thread finds four eigenvalues with interleaved
// (independent) Sturm recurrences to hide the division latency.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace csb {
namespace cg = cooperative_groups;

constexpr int kTriThreads = 512;
constexpr int kTriMaxM = 2048;

struct TriArgs {
  double* A;   // m x m full symmetric working copy, column-major (destroyed)
  int m;
  double* d;   // [m] diagonal of T
  double* e;   // [m - 1] off-diagonal of T
  double* gv;  // [m] Householder vector (global exchange)
  double* gw;  // [m] w vector
};

// block sum of one double per thread (deterministic tree); result on all threads
__device__ __forceinline__ double tri_block_sum(double x, double* scratch) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();  // scratch free
  if (lane == 0) scratch[warp] = x;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < kTriThreads / 32; ++w) s += scratch[w];
  return s;
}

__global__ void __launch_bounds__(kTriThreads, 1) tridiag_cluster_kernel(TriArgs a) {
  cg::cluster_group cluster = cg::this_cluster();
  const int CS = static_cast<int>(cluster.num_blocks());
  const int c = static_cast<int>(cluster.block_rank());
  const int m = a.m;
  double* A = a.A;
  const int R = (m + CS - 1) / CS;
  const int r0 = c * R, r1 = min(m, r0 + R);
  const int RP = R <= 32 ? 32 : (R <= 64 ? 64 : 128);  // rows per phase group (R <= 128)
  const int nph = kTriThreads / RP;                    // column phases
  const int tid = threadIdx.x, rr = tid % RP, ph = tid / RP;
  const int i = r0 + rr;
  const bool own = i < r1;
  __shared__ double scratch[kTriThreads / 32];
  __shared__ double red[2][4];  // this CTA's partials, by step parity (read remotely)
  __shared__ double bc[4];      // broadcast: tau, scal, K
  __shared__ double prow[kTriThreads];
  auto col = [&](int j) { return A + static_cast<size_t>(j) * m; };
  for (int k = 0; k + 2 < m; ++k) {
    const int par = k & 1;
    // (a) column k below the diagonal: alpha = A(k+1, k), sigma = sum of squares below
    double sig = 0.0, alp = 0.0;
    if (ph == 0 && own && i >= k + 1) {
      const double x = col(k)[i];
      if (i == k + 1) alp = x;
      else sig = x * x;
    }
    sig = tri_block_sum(sig, scratch);
    alp = tri_block_sum(alp, scratch);
    if (tid == 0) {
      red[par][0] = sig;
      red[par][1] = alp;
    }
    cluster.sync();
    if (tid == 0) {
      double S = 0.0, Al = 0.0;
      for (int q = 0; q < CS; ++q) {
        const double* rq = cluster.map_shared_rank(&red[par][0], q);
        S += rq[0];
        Al += rq[1];
      }
      double tau = 0.0, scal = 0.0, beta = Al;
      if (S > 0.0) {
        const double nrm = sqrt(Al * Al + S);
        beta = -copysign(nrm, Al);
        tau = (beta - Al) / beta;
        scal = 1.0 / (Al - beta);
      }
      bc[0] = tau;
      bc[1] = scal;
      if (c == 0) {
        a.d[k] = A[static_cast<size_t>(k) * m + k];
        a.e[k] = beta;
      }
    }
    __syncthreads();
    const double tau = bc[0], scal = bc[1];
    if (tau == 0.0) {  // column already reduced: H = I (all CTAs agree: same S)
      __syncthreads();
      continue;
    }
    double vi = 0.0;
    if (own && i >= k + 1) vi = i == k + 1 ? 1.0 : col(k)[i] * scal;
    if (ph == 0 && own && i >= k + 1) a.gv[i] = vi;
    __threadfence();
    cluster.sync();
    // (b) p_i = tau sum_{j > k} A(i, j) v_j over this CTA's rows
    double acc = 0.0;
    if (own && i >= k + 1)
      for (int j = k + 1 + ph; j < m; j += nph) acc = fma(col(j)[i], a.gv[j], acc);
    prow[tid] = acc;
    __syncthreads();
    double pi = 0.0;
    if (ph == 0 && own && i >= k + 1) {
      for (int q = 0; q < nph; ++q) pi += prow[q * RP + rr];
      pi *= tau;
    }
    double pv = tri_block_sum(ph == 0 ? pi * vi : 0.0, scratch);
    if (tid == 0) red[par][2] = pv;
    cluster.sync();
    if (tid == 0) {
      double K = 0.0;
      for (int q = 0; q < CS; ++q) K += cluster.map_shared_rank(&red[par][0], q)[2];
      bc[2] = K;
    }
    __syncthreads();
    const double K = bc[2];
    if (ph == 0 && own && i >= k + 1) a.gw[i] = pi - 0.5 * tau * K * vi;
    __threadfence();
    cluster.sync();
    // (d) A22 -= v w^T + w v^T on this CTA's rows (all trailing columns)
    if (own && i >= k + 1) {
      const double wi = a.gw[i];
      for (int j = k + 1 + ph; j < m; j += nph) {
        const double u = __dadd_rn(__dmul_rn(vi, a.gw[j]), __dmul_rn(wi, a.gv[j]));
        col(j)[i] -= u;
      }
    }
    __threadfence();  // (CTA 0 reads the next diagonal entry, which another CTA may own)
    __syncthreads();  // the next column's entries of this CTA's rows are final
  }
  // the last 2 x 2 block
  __threadfence();
  cluster.sync();
  if (c == 0 && tid == 0) {
    if (m >= 2) {
      a.d[m - 2] = A[static_cast<size_t>(m - 2) * m + (m - 2)];
      a.e[m - 2] = A[static_cast<size_t>(m - 2) * m + (m - 1)];
    }
    a.d[m - 1] = A[static_cast<size_t>(m - 1) * m + (m - 1)];
  }
}

// eigenvalues of the symmetric tridiagonal (d, e) in ascending order
constexpr int kBisectPer = 4;  // eigenvalues per thread (independent recurrences)
__global__ void __launch_bounds__(128) tridiag_bisect_kernel(const double* __restrict__ d,
                                                             const double* __restrict__ e, int m,
                                                             double lo0, double hi0, double pivmin,
                                                             double* __restrict__ w) {
  extern __shared__ double sh[];  // d [m], e^2 [m]
  double* sd = sh;
  double* se2 = sh + m;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    sd[i] = d[i];
    se2[i] = i + 1 < m ? e[i] * e[i] : 0.0;
  }
  __syncthreads();
  const int per_block = blockDim.x * kBisectPer;
  double lo[kBisectPer], hi[kBisectPer];
  int kk[kBisectPer];
  bool act[kBisectPer];
#pragma unroll
  for (int u = 0; u < kBisectPer; ++u) {
    kk[u] = blockIdx.x * per_block + u * blockDim.x + threadIdx.x;
    act[u] = kk[u] < m;
    lo[u] = lo0;
    hi[u] = hi0;
  }
  for (int it = 0; it < 200; ++it) {
    double x[kBisectPer], q[kBisectPer];
    int cnt[kBisectPer];
    bool any = false;
#pragma unroll
    for (int u = 0; u < kBisectPer; ++u) {
      x[u] = 0.5 * (lo[u] + hi[u]);
      if (act[u] && (x[u] <= lo[u] || x[u] >= hi[u])) act[u] = false;  // interval at the last bit
      any |= act[u];
      q[u] = sd[0] - x[u];
      cnt[u] = q[u] < 0.0;
    }
    if (!any) break;
    for (int i = 1; i < m; ++i) {
      const double di = sd[i], e2 = se2[i - 1];
#pragma unroll
      for (int u = 0; u < kBisectPer; ++u) {
        const double qq = fabs(q[u]) < pivmin ? -pivmin : q[u];
        q[u] = (di - x[u]) - e2 / qq;
        cnt[u] += q[u] < 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < kBisectPer; ++u) {
      if (!act[u]) continue;
      if (cnt[u] > kk[u]) hi[u] = x[u];
      else lo[u] = x[u];
    }
  }
#pragma unroll
  for (int u = 0; u < kBisectPer; ++u)
    if (kk[u] < m) w[kk[u]] = 0.5 * (lo[u] + hi[u]);
}

}  // namespace csb
