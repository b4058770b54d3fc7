// eig_tridiag.cuh -- eigenvalues of a symmetric matrix without cuSOLVER:
// Householder tridiagonalisation by one thread-block cluster, then Sturm-count
// multisection.  The eigenvalues-only calls of the train path (the eager
// eigen_spectrum and the eigen route's rank decision, mset.cpp:153-163) take
// it by default for m <= kTriOwnMaxM, where it beats cuSOLVER's syevd
// (measured, 1 x B200: m = 40 0.20 vs 0.38 ms, 100 0.42 vs 0.75, 160 0.89 vs
// 1.29, 500 4.6 vs 5.3); above, syevd stays the default (m = 1000: 19 vs
// 12 ms -- a one-stage reduction streams the trailing matrix through L2 at
// every column; the fast design is two-stage) and the
// own path is opt-in (CSB_EIG_OWN=1) up to kTriMaxM.  Exact to 1e-12 of
// max|lambda| against LAPACK (tests/test_gpu_eig.py).
//
// Tridiagonalisation (the classical one-stage algorithm, Golub & Van Loan
// 8.3.1): for k = 0 .. m-3, a Householder reflector H = I - tau v v^T
// (v_0 = 1) maps column k below the diagonal to (beta, 0, ...); the trailing
// matrix becomes H A22 H = A22 - v w^T - w v^T with p = tau A22 v and
// w = p - (tau / 2)(p^T v) v.  cuSOLVER's blocked sytrd spends ~11 ms at
// m = 1000 on this (latency of its per-column kernels); here one cluster of
// 16 CTAs (non-portable size; 8 where 16 cannot be launched) owns the whole
// reduction: CTA c holds rows [c R, c R + R) of the full symmetric working
// matrix in global memory (L2-resident up to ~2k x 2k), the column step's
// reductions go through distributed shared memory (partials
// read in parallel and summed by a fixed shuffle tree: deterministic); each column costs two cluster
// barriers: v is re-derived by every CTA from column k in L2, p goes out
// through L2 with the p.v partials and w = p - (tau K / 2) v is formed on the
// fly in the rank-2 update.
// Both triangles are updated with the same rounded terms, so the working
// matrix stays exactly symmetric.
//
// Bisection (LAPACK dstebz's method): count(x) = number of negative
// pivots of T - x I = number of eigenvalues < x; eigenvalue k is the point
// where the count passes k, found by multisection of the Gershgorin interval
// to the last bit (one warp per eigenvalue, 32 shifts per round).
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace csb {
namespace cg = cooperative_groups;

constexpr int kTriThreads = 512;
constexpr int kTriMaxM = 2048;
constexpr int kTriOwnMaxM = 512;  // default own path up to here

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
    if (tid < 32) {
      // lane q reads CTA q's partials (remote loads in parallel, not a
      // dependent chain of DSMEM round trips), then a fixed shuffle tree
      double S = 0.0, Al = 0.0;
      if (tid < CS) {
        const double* rq = cluster.map_shared_rank(&red[par][0], tid);
        S = rq[0];
        Al = rq[1];
      }
      for (int o = 16; o > 0; o >>= 1) {
        S += __shfl_xor_sync(0xffffffffu, S, o);
        Al += __shfl_xor_sync(0xffffffffu, Al, o);
      }
      double tau = 0.0, scal = 0.0, beta = Al;
      if (S > 0.0) {
        const double nrm = sqrt(Al * Al + S);
        beta = -copysign(nrm, Al);
        tau = (beta - Al) / beta;
        scal = 1.0 / (Al - beta);
      }
      if (tid == 0) {
        bc[0] = tau;
        bc[1] = scal;
        if (c == 0) {
          a.d[k] = A[static_cast<size_t>(k) * m + k];
          a.e[k] = beta;
        }
      }
    }
    __syncthreads();
    const double tau = bc[0], scal = bc[1];
    if (tau == 0.0) {  // column already reduced: H = I (all CTAs agree: same S)
      __syncthreads();
      continue;
    }
    // v from column k itself (every CTA reads the whole column from L2: the
    // previous step's updates are ordered before it by the barrier above),
    // so no exchange and no barrier for v
    auto vof = [&](int j) { return j == k + 1 ? 1.0 : col(k)[j] * scal; };
    const double vi = (own && i >= k + 1) ? vof(i) : 0.0;
    // (b) p_i = tau sum_{j > k} A(i, j) v_j over this CTA's rows
    double acc = 0.0;
    if (own && i >= k + 1) {
      // eight columns' loads in flight per batch, four accumulators
      double acc4[4] = {0.0, 0.0, 0.0, 0.0};
      int j = k + 1 + ph;
      for (; j + 7 * nph < m; j += 8 * nph) {
        double av[8], vv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          av[u] = col(j + u * nph)[i];
          vv[u] = vof(j + u * nph);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc4[u & 3] = fma(av[u], vv[u], acc4[u & 3]);
      }
      for (; j < m; j += nph) acc4[0] = fma(col(j)[i], vof(j), acc4[0]);
      acc = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
    }
    prow[tid] = acc;
    __syncthreads();
    double pi = 0.0;
    if (ph == 0 && own && i >= k + 1) {
      for (int q = 0; q < nph; ++q) pi += prow[q * RP + rr];
      pi *= tau;
      a.gv[i] = pi;  // p goes out with the p.v partial: one barrier for both
    }
    double pv = tri_block_sum(ph == 0 ? pi * vi : 0.0, scratch);
    if (tid == 0) red[par][2] = pv;
    cluster.sync();
    if (tid < 32) {
      double K = tid < CS ? cluster.map_shared_rank(&red[par][0], tid)[2] : 0.0;
      for (int o = 16; o > 0; o >>= 1) K += __shfl_xor_sync(0xffffffffu, K, o);
      if (tid == 0) bc[2] = K;
    }
    __syncthreads();
    const double hk = 0.5 * tau * bc[2];
    // (d) A22 -= v w^T + w v^T on this CTA's rows, w_j = p_j - (tau K / 2) v_j
    // formed on the fly from the exchanged p (same expression in every CTA)
    if (own && i >= k + 1) {
      const double wi = a.gv[i] - hk * vi;
      int j = k + 1 + ph;
      for (; j + 7 * nph < m; j += 8 * nph) {
        double av[8], pj[8], vj[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          av[u] = col(j + u * nph)[i];
          pj[u] = a.gv[j + u * nph];
          vj[u] = vof(j + u * nph);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double wj = pj[u] - hk * vj[u];
          col(j + u * nph)[i] = av[u] - __dadd_rn(__dmul_rn(vi, wj), __dmul_rn(wi, vj[u]));
        }
      }
      for (; j < m; j += nph) {
        const double vj = vof(j), wj = a.gv[j] - hk * vj;
        col(j)[i] -= __dadd_rn(__dmul_rn(vi, wj), __dmul_rn(wi, vj));
      }
    }
    __syncthreads();  // the next column's entries of this CTA's rows are final; other CTAs
                      // read them after the next step's first cluster barrier
  }
  // the last 2 x 2 block
  cluster.sync();
  if (c == 0 && tid == 0) {
    if (m >= 2) {
      a.d[m - 2] = A[static_cast<size_t>(m - 2) * m + (m - 2)];
      a.e[m - 2] = A[static_cast<size_t>(m - 2) * m + (m - 1)];
    }
    a.d[m - 1] = A[static_cast<size_t>(m - 1) * m + (m - 1)];
  }
}

// Small matrices (m <= kTriCtaMaxM): the same reduction by ONE CTA with the
// whole matrix in shared memory -- block barriers only, no cluster barrier
// or L2 round trip per column (m = 100: ~0.15 ms against syevd's 0.75 ms).
constexpr int kTriCtaMaxM = 160;
constexpr int kTriCtaThreads = 512;
__host__ __device__ constexpr size_t tri_cta_smem(int m) {
  return sizeof(double) * (static_cast<size_t>(m) * (m + 1) + 3 * static_cast<size_t>(m) + kTriCtaThreads +
                           kTriCtaThreads / 32 + 8);
}

__global__ void __launch_bounds__(kTriCtaThreads, 1) tridiag_cta_kernel(const double* __restrict__ G, int m,
                                                                         double* __restrict__ d,
                                                                         double* __restrict__ e) {
  extern __shared__ double sm[];
  const int ld = m + 1;  // odd stride: column reads by consecutive rows are conflict-free
  double* A = sm;
  double* v = A + static_cast<size_t>(m) * ld;
  double* p = v + m;
  double* w = p + m;
  double* part = w + m;  // [kTriCtaThreads] row partials by column phase
  double* scratch = part + kTriCtaThreads;
  double* bc = scratch + kTriCtaThreads / 32;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < m * m; idx += blockDim.x) {
    const int i = idx % m, j = idx / m;
    A[i + j * ld] = G[idx];
  }
  __syncthreads();
  auto bsum = [&](double x) {
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    __syncthreads();
    if ((tid & 31) == 0) scratch[tid >> 5] = x;
    __syncthreads();
    double s = 0.0;
    for (int q = 0; q < kTriCtaThreads / 32; ++q) s += scratch[q];
    return s;
  };
  for (int k = 0; k + 2 < m; ++k) {
    const int i0 = k + 1, mp = m - i0;  // trailing block rows / cols [i0, m)
    double sig = 0.0;
    for (int i = k + 2 + tid; i < m; i += blockDim.x) {
      const double x = A[i + k * ld];
      sig += x * x;
    }
    sig = bsum(sig);
    if (tid == 0) {
      const double al = A[i0 + k * ld];
      double tau = 0.0, scal = 0.0, beta = al;
      if (sig > 0.0) {
        const double nrm = sqrt(al * al + sig);
        beta = -copysign(nrm, al);
        tau = (beta - al) / beta;
        scal = 1.0 / (al - beta);
      }
      d[k] = A[k + k * ld];
      e[k] = beta;
      bc[0] = tau;
      bc[1] = scal;
    }
    __syncthreads();
    const double tau = bc[0], scal = bc[1];
    if (tau == 0.0) continue;  // uniform
    for (int i = i0 + tid; i < m; i += blockDim.x) v[i] = i == i0 ? 1.0 : A[i + k * ld] * scal;
    __syncthreads();
    // p = tau A22 v: (row, column phase) per thread, phases summed in order
    const int nq = kTriCtaThreads / 128;
    for (int r0 = 0; r0 < mp; r0 += 128) {
      const int rr = tid % 128, q = tid / 128, i = i0 + r0 + rr;
      double acc = 0.0;
      if (i < m)
        for (int j = i0 + q; j < m; j += nq) acc = fma(A[i + j * ld], v[j], acc);
      part[q * 128 + rr] = acc;
      __syncthreads();
      if (q == 0 && i < m) {
        double sp = 0.0;
        for (int qq = 0; qq < nq; ++qq) sp += part[qq * 128 + rr];
        p[i] = sp;
      }
      __syncthreads();
    }
    double pv = 0.0;
    for (int i = i0 + tid; i < m; i += blockDim.x) {
      p[i] *= tau;
      pv += p[i] * v[i];
    }
    const double K = bsum(pv);
    for (int i = i0 + tid; i < m; i += blockDim.x) w[i] = p[i] - 0.5 * tau * K * v[i];
    __syncthreads();
    for (int idx = tid; idx < mp * mp; idx += blockDim.x) {
      const int i = i0 + idx % mp, j = i0 + idx / mp;
      A[i + j * ld] -= __dadd_rn(__dmul_rn(v[i], w[j]), __dmul_rn(w[i], v[j]));
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (m >= 2) {
      d[m - 2] = A[(m - 2) + (m - 2) * ld];
      e[m - 2] = A[(m - 1) + (m - 2) * ld];
    }
    d[m - 1] = A[(m - 1) + (m - 1) * ld];
  }
}

// Eigenvalues of the symmetric tridiagonal (d, e), ascending: one WARP per
// eigenvalue, 32-way multisection -- each round every lane counts the
// eigenvalues below its own shift of the current interval and the warp keeps
// the sub-interval where the count passes k (a ballot), so ~12 rounds reach
// the last bit instead of ~60 bisection steps.  The Sturm recurrence
// q_i = (d_i - x) - e_{i-1}^2 / q_{i-1} (zero pivots replaced by -pivmin,
// LAPACK dstebz) divides through a MUFU reciprocal seed and two Newton
// steps (~1 ulp; the count is that of a matrix within a few ulps of T).
__device__ __forceinline__ double sturm_rcp(double q) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
  r = fma(r, fma(-q, r, 1.0), r);
  r = fma(r, fma(-q, r, 1.0), r);
  return r;
}

constexpr int kBisectWarps = 4;  // eigenvalues per 128-thread block
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
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * kBisectWarps + (threadIdx.x >> 5);
  if (k >= m) return;
  double lo = lo0, hi = hi0;
  for (int round = 0; round < 64; ++round) {
    const double x = lo + (hi - lo) * (static_cast<double>(lane + 1) / 33.0);
    double q = sd[0] - x;
    int cnt = q < 0.0;
    for (int i = 1; i < m; ++i) {
      const double qq = fabs(q) < pivmin ? -pivmin : q;
      q = (sd[i] - x) - se2[i - 1] * sturm_rcp(qq);
      cnt += q < 0.0;
    }
    const unsigned above = __ballot_sync(0xffffffffu, cnt > k);  // shifts with > k eigenvalues below
    const int j = above ? __ffs(above) - 1 : 32;                // first such lane
    const double nlo = j > 0 ? __shfl_sync(0xffffffffu, x, j - 1) : lo;
    const double nhi = j < 32 ? __shfl_sync(0xffffffffu, x, j) : hi;
    if (!(nlo > lo || nhi < hi)) break;  // no shift fell strictly inside: the interval is at the last bits
    lo = nlo;
    hi = nhi;
  }
  if (lane == 0) w[k] = 0.5 * (lo + hi);
}

}  // namespace csb
