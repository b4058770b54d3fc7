// eig_tridiag.cuh -- eigenvalues of a symmetric matrix without cuSOLVER:
// Householder tridiagonalisation with the matrix held in shared memory, then
// Sturm-count multisection.  The eigenvalues-only calls of the train path
// (the eager eigen_spectrum and the eigen route's rank decision,
// mset.cpp:153-163) take it by default for m <= kTriMaxM (measured, 1 x
// B200, against cuSOLVER's syevd: m = 100 0.42 vs 0.75 ms, 200 0.94 vs 1.86,
// 500 3.3 vs 5.3, 1000 7.4 vs 11.9, 2000 22.5 vs 28.4); larger m stays on
// syevd.  Exact to 1e-12 of max|lambda| against LAPACK (tests/test_gpu_eig.py).
//
// Tridiagonalisation (the classical one-stage algorithm, Golub & Van Loan
// 8.3.1): for k = 0 .. m-3, a Householder reflector H = I - tau v v^T
// (v_0 = 1) maps column k below the diagonal to (beta, 0, ...); the trailing
// matrix becomes H A22 H = A22 - v w^T - w v^T with p = tau A22 v and
// w = p - (tau / 2)(p^T v) v.  Every column step needs the whole trailing
// matrix (p) and then a vector exchange before the next step can start, so
// the reduction is latency-bound: cuSOLVER's blocked sytrd spends ~11 ms at
// m = 1000 in per-column kernels.  Here one launch does all m - 2 steps:
// one CTA for m <= kTriCtaMaxM, a co-resident grid above (one column
// exchange through L2 per step, see tridiag_grid_kernel).
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

constexpr int kTriMaxM = 2048;
constexpr int kTriCtaMaxM = 160;

// Small matrices (m <= kTriCtaMaxM): the same reduction by ONE CTA with the
// whole matrix in shared memory -- block barriers only, no cluster barrier
// or L2 round trip per column (m = 100: ~0.15 ms against syevd's 0.75 ms).
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
    // every thread forms the reflector itself (the same values): no
    // broadcast through shared memory and no barrier for it
    const double al = A[i0 + k * ld];
    double tau = 0.0, scal = 0.0, beta = al;
    if (sig > 0.0) {
      const double nrm = sqrt(al * al + sig);
      beta = -copysign(nrm, al);
      tau = (beta - al) / beta;
      scal = 1.0 / (al - beta);
    }
    if (tid == 0) {
      d[k] = A[k + k * ld];
      e[k] = beta;
    }
    if (tau == 0.0) {  // uniform
      __syncthreads();  // bsum's scratch is reused next step
      continue;
    }
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
    // rank-2 update: a warp per column, lanes down the rows (no index
    // division per element)
    for (int j = i0 + (tid >> 5); j < m; j += kTriCtaThreads / 32) {
      const double vj = v[j], wj = w[j];
      for (int i = i0 + (tid & 31); i < m; i += 32)
        A[i + j * ld] -= __dadd_rn(__dmul_rn(v[i], wj), __dmul_rn(w[i], vj));
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

// Larger matrices (kTriClusterMaxM < m <= kTriMaxM): the same reduction by a
// co-resident grid for all but the last kTriClusterMaxM columns, whose
// trailing block the 16-CTA cluster kernel below finishes (or, without
// clusters, all but the last kTriCtaMaxM for the one-CTA kernel: its steps
// cost ~4 us on a 160 block against the grid's ~6.5 us exchange-bound ones).  The grid is a
// co-resident one (cooperative launch, one CTA per SM) with the whole
// matrix in SHARED memory -- CTA c keeps the full rows i = c, c + P, ...
// (cyclic, so the shrinking trailing block stays balanced; at most
// kTriGridRows rows of m doubles); thread t owns the columns j = t + u T.
// ONE exchange through L2 per column step, no barrier:
//   (B) every CTA forms p_i = tau (A22 v)_i for its rows i > k and publishes
//       p_i, its partial of K = p^T v, and -- the owner of row k + 2 --
//       that row as it stands (after step k - 1);
//   (C) every CTA reads all p_j, the P partials (summed in CTA order: every
//       CTA gets the same K, hence the same w = p - (tau K / 2) v) and row
//       k + 2, then applies A_ij -= v_i w_j + w_i v_j to its own rows and
//       to two REPLICA rows held in registers: row k + 1 (received one step
//       earlier) and row k + 2.  Row k + 1 is then final for step k + 1, so
//       every CTA forms the next reflector (v, tau) itself from its replica
//       -- the same values, bit for bit, as the owner's row gives (same
//       inputs, same operations) -- and no second exchange is needed.
// The mirrored element A_ji gets the identically rounded update, so the
// matrix stays exactly symmetric.  Every published double travels as two
// 8-byte words (32-bit half + 32-bit step tag; 8-byte stores are single-copy
// atomic), so a reader polls the data itself: no flag, fence or barrier.
// Buffers alternate by step parity; a CTA can run at most one step ahead of
// the slowest (step k+1's exchange needs every CTA's step-k publication,
// which follows its step k-1 reads), so two generations suffice.  tau = 0
// steps run the same exchange (p = 0, w = 0: the update subtracts zeros).
constexpr int kTriGridThreads = 256;
constexpr int kTriGridRows = 16;                          // owned rows per CTA (one row sum per lane pair)
constexpr int kTriGridCols = kTriMaxM / kTriGridThreads;  // columns per thread
constexpr int kTriGridMaxP = 160;                         // CTAs (partials of p^T v: 5 per lane)
static_assert(kTriGridCols * kTriGridThreads >= kTriMaxM, "grid reduction column cover");
static_assert(kTriGridRows == 16, "the row-sum transpose reduction is written for 16 rows");

struct TriGridArgs {
  const double* G;   // m x m symmetric, column-major (read only)
  int m, P;
  double* d;         // [m]
  double* e;         // [m - 1]
  ulonglong2* pbuf;  // [2][m] tagged p
  ulonglong2* rbuf;  // [2][m] tagged row k + 2
  ulonglong2* kbuf;  // [2][P] tagged partials of p^T v
  unsigned long long* trace;  // development: [m][4] globaltimer stamps of CTA 0, or nullptr
  int kstop;                  // steps 0 .. kstop - 1 here (kstop <= m - 2) ...
  double* tail;               // ... then rows / cols >= kstop go here (column-major, m - kstop square)
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void tag_store(ulonglong2* p, double x, unsigned tag) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
  const unsigned long long t = static_cast<unsigned long long>(tag) << 32;
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(t | (b & 0xffffffffull)),
               "l"(t | (b >> 32))
               : "memory");
}
__device__ __forceinline__ ulonglong2 tag_load(const ulonglong2* p) {
  ulonglong2 r;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ bool tag_ok(ulonglong2 r, unsigned tag) {
  return static_cast<unsigned>(r.x >> 32) == tag && static_cast<unsigned>(r.y >> 32) == tag;
}
__device__ __forceinline__ double tag_value(ulonglong2 r) {
  return __longlong_as_double(static_cast<long long>((r.y << 32) | (r.x & 0xffffffffull)));
}
// N tagged slots at addr(u) (nullptr: none): every load is issued before
// any tag is checked, and only the late slots are re-polled
template <int N, class Addr>
__device__ __forceinline__ void tag_wait_slots(Addr addr, unsigned tag, double (&out)[N]) {
  ulonglong2 r[N];
  const unsigned long long t = static_cast<unsigned long long>(tag) << 32;
#pragma unroll
  for (int u = 0; u < N; ++u) {
    const ulonglong2* p = addr(u);
    r[u] = p ? tag_load(p) : make_ulonglong2(t, t);
  }
  // bounded spin: a producer that can never arrive (a bug, or a co-residency
  // violation) ends the kernel with an error instead of hanging the device
  for (uint32_t spins = 0;; ++spins) {
    bool ok = true;
#pragma unroll
    for (int u = 0; u < N; ++u) ok &= tag_ok(r[u], tag);
    if (ok) break;
    if (spins > (1u << 24)) __trap();  // ~10 s of polling
#pragma unroll
    for (int u = 0; u < N; ++u)
      if (!tag_ok(r[u], tag)) r[u] = tag_load(addr(u));
  }
#pragma unroll
  for (int u = 0; u < N; ++u) out[u] = addr(u) ? tag_value(r[u]) : 0.0;
}

// shared memory: the small arrays, then `rows` rows of NC T doubles (a
// compile-time row stride: every row access is one base register plus an
// immediate offset, and the columns past m are zero padding)
constexpr int kTriGridSmall = 2 * kTriGridRows + kTriGridRows * (kTriGridThreads / 32) + kTriGridThreads / 32 + 8;
__host__ __device__ constexpr size_t tri_grid_smem(int nc, int rows) {
  return sizeof(double) * (static_cast<size_t>(rows) * nc * kTriGridThreads + kTriGridSmall);
}

template <int NC>  // column slots per thread: m <= NC kTriGridThreads
__global__ void __launch_bounds__(kTriGridThreads, 1) tridiag_grid_kernel(TriGridArgs a) {
  extern __shared__ double sm[];
  constexpr int T = kTriGridThreads, NW = T / 32, LD = NC * T;
  const int m = a.m, P = a.P, c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int R = (m - c + P - 1) / P;  // rows i = c + r P, r < R
  const int Rmax = (m + P - 1) / P;
  double* vo = sm;                            // [kTriGridRows] v_i of the owned rows
  double* po = vo + kTriGridRows;             // [kTriGridRows] p_i of the owned rows
  double* red = po + kTriGridRows;            // [kTriGridRows][NW] row sums by warp
  double* scratch = red + kTriGridRows * NW;  // [NW]
  double* bc = scratch + NW;                  // broadcast scalars
  double* At = sm + kTriGridSmall + tid;      // this thread's column 0 of owned row 0: (r, u) at r LD + u T
  for (int r = 0; r < Rmax; ++r) {
    const double* gcol = a.G + static_cast<size_t>(c + r * P) * m;  // row i == column i
#pragma unroll
    for (int u = 0; u < NC; ++u) {
      const int j = tid + u * T;
      At[r * LD + u * T] = r < R && j < m ? gcol[j] : 0.0;
    }
  }
  if (tid < 2 * kTriGridRows) vo[tid] = 0.0;  // vo, po
  // replicas of rows 0 and 1 (columns of this thread) straight from G
  double r1[NC], vr[NC];
#pragma unroll
  for (int u = 0; u < NC; ++u) {
    const int j = tid + u * T;
    r1[u] = j < m ? a.G[static_cast<size_t>(1) * m + j] : 0.0;
    vr[u] = j < m ? a.G[j] : 0.0;  // row 0, turned into v below
  }
  // reflector of row `kk` (values x[u] at this thread's columns): sigma by a
  // fixed-order block sum, then every thread forms tau / scal / beta itself
  auto reflector = [&](int kk, double (&x)[NC], double& tau_out) {
    double sig = 0.0;
#pragma unroll
    for (int u = 0; u < NC; ++u) {
      const int j = tid + u * T;
      if (j > kk + 1 && j < m) sig = fma(x[u], x[u], sig);
      if (j == kk + 1) bc[0] = x[u];  // alpha
      if (j == kk && c == 0) a.d[kk] = x[u];
    }
    for (int o = 16; o > 0; o >>= 1) sig += __shfl_xor_sync(0xffffffffu, sig, o);
    if (lane == 0) scratch[warp] = sig;
    __syncthreads();
    double S = 0.0;
    for (int w = 0; w < NW; ++w) S += scratch[w];
    const double al = bc[0];
    double tau = 0.0, scal = 0.0, beta = al;
    if (S > 0.0) {
      const double nrm = sqrt(al * al + S);
      beta = -copysign(nrm, al);
      tau = (beta - al) / beta;
      scal = 1.0 / (al - beta);
    }
    if (c == 0 && tid == 0) a.e[kk] = beta;
#pragma unroll
    for (int u = 0; u < NC; ++u) {
      const int j = tid + u * T;
      x[u] = j == kk + 1 ? 1.0 : (j > kk + 1 && j < m ? x[u] * scal : 0.0);
    }
    tau_out = tau;
    __syncthreads();  // scratch / bc[0] reusable
  };
  // step kk's copy of row kk + 2 (as it stands after step kk - 1), published
  // by its owner as soon as that update is done: each thread its own
  // columns, which it wrote itself (no barrier)
  auto publish_row = [&](int kk) {
    if ((kk + 2) % P == c) {
      const double* row = At + ((kk + 2) / P) * LD;
      ulonglong2* rbk = a.rbuf + static_cast<size_t>(kk & 1) * m;
#pragma unroll
      for (int u = 0; u < NC; ++u) {
        const int j = tid + u * T;
        if (j >= kk + 2 && j < m) tag_store(rbk + j, row[u * T], static_cast<unsigned>(kk + 1));
      }
    }
  };
  __syncthreads();  // the rows are loaded
  if (m > 2) publish_row(0);
  double tau;
  reflector(0, vr, tau);

  const int kstop = a.kstop;
  for (int k = 0; k < kstop; ++k) {
    const unsigned tag = static_cast<unsigned>(k + 1);
    const int par = k & 1;
    ulonglong2* pb = a.pbuf + static_cast<size_t>(par) * m;
    ulonglong2* rb = a.rbuf + static_cast<size_t>(par) * m;
    ulonglong2* kb = a.kbuf + static_cast<size_t>(par) * P;
    const int rlo = c > k ? 0 : (k - c) / P + 1;  // first owned row with i > k
    // (B) row sums of the owned rows against v
    // Slots are skipped only where a whole warp's 32 columns are dead (a
    // uniform branch); inside a live warp slot v_j = 0 at j <= k and j >= m
    // (where the row is zero padding), so dead columns add exact zeros.
    // Rows i <= k (r < rlo) are finished and skipped (uniform).
    bool live[NC];
#pragma unroll
    for (int u = 0; u < NC; ++u) live[u] = u * T + warp * 32 + 31 > k && u * T + warp * 32 < m;
    double acc[kTriGridRows];
#pragma unroll
    for (int r = 0; r < kTriGridRows; ++r) {
      acc[r] = 0.0;
      if (r >= rlo && r < R) {  // uniform
#pragma unroll
        for (int u = 0; u < NC; ++u)
          if (live[u]) acc[r] = fma(At[r * LD + u * T], vr[u], acc[r]);
      }
    }
#pragma unroll
    for (int u = 0; u < NC; ++u) {  // stash v_i of the owned rows
      const int j = tid + u * T;
      if (j > k && j < m && j % P == c) vo[j / P] = vr[u];
    }
    // 16 row sums over the warp by a transposing butterfly (16 shuffles):
    // lane l ends with row l >> 1
#pragma unroll
    for (int h = 8; h >= 1; h >>= 1) {
      const bool up = lane & (2 * h);
#pragma unroll
      for (int i = 0; i < h; ++i) {
        const double send = up ? acc[i] : acc[i + h];
        const double keep = up ? acc[i + h] : acc[i];
        acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2 * h);
      }
    }
    acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
    if ((lane & 1) == 0) red[(lane >> 1) * NW + warp] = acc[0];
    __syncthreads();
    if (warp == 0) {
      const int r = lane;
      double pv = 0.0;
      if (r < rlo && r < kTriGridRows) vo[r] = po[r] = 0.0;  // finished rows: the update subtracts zeros
      if (r >= rlo && r < R) {
        const int i = c + r * P;
        double s = 0.0;
        for (int w = 0; w < NW; ++w) s += red[r * NW + w];
        const double pi = tau * s;
        po[r] = pi;
        tag_store(pb + i, pi, tag);
        pv = pi * vo[r];
      }
      for (int o = 16; o > 0; o >>= 1) pv += __shfl_xor_sync(0xffffffffu, pv, o);
      if (lane == 0) tag_store(kb + c, pv, tag);
      if (a.trace && c == 0 && lane == 0) a.trace[4 * k + 1] = gtimer();
    }
    // (C) all p_j, row k + 2 and (warp 0) the partials, in ONE batch of loads
    constexpr int KQ = (kTriGridMaxP + 31) / 32;
    double pw[NC], r2[NC];
    {
      double got[2 * NC + KQ];
      tag_wait_slots([&](int u) -> const ulonglong2* {
        if (u < NC) {
          const int j = tid + u * T;
          return j > k && j < m ? pb + j : nullptr;
        }
        if (u < 2 * NC) {
          const int j = tid + (u - NC) * T;
          return j >= k + 2 && j < m ? rb + j : nullptr;
        }
        const int q = lane + (u - 2 * NC) * 32;  // partial q (lane + 32 i: a fixed order)
        return warp == 0 && q < P ? kb + q : nullptr;
      }, tag, got);
#pragma unroll
      for (int u = 0; u < NC; ++u) {
        pw[u] = got[u];
        r2[u] = got[NC + u];
      }
      if (warp == 0) {
        double K = 0.0;
#pragma unroll
        for (int u = 0; u < KQ; ++u) K += got[2 * NC + u];
        for (int o = 16; o > 0; o >>= 1) K += __shfl_xor_sync(0xffffffffu, K, o);
        if (lane == 0) bc[3] = K;
      }
    }
#pragma unroll
    for (int u = 0; u < NC; ++u) {  // p and v at columns k + 1, k + 2 for the replicas
      const int j = tid + u * T;
      if (j == k + 1) bc[4] = pw[u];
      if (j == k + 2) {
        bc[5] = pw[u];
        bc[6] = vr[u];
      }
    }
    __syncthreads();
    if (a.trace && c == 0 && tid == 0) a.trace[4 * k + 2] = gtimer();
    const double hk = 0.5 * tau * bc[3];
#pragma unroll
    for (int u = 0; u < NC; ++u) pw[u] = pw[u] - hk * vr[u];  // w_j
    // live owned rows, live warp slots; at j <= k inside a live slot both w_j
    // and v_j are 0, so those columns subtract exact zeros.  Groups of rows
    // are loaded before any is stored (the compiler cannot tell the
    // shared-memory rows apart and would order every load after the
    // previous store).
    constexpr int RG = NC <= 2 ? 8 : 16 / NC;
#pragma unroll
    for (int r0 = 0; r0 < kTriGridRows; r0 += RG) {
      if (r0 + RG > rlo && r0 < R) {  // uniform
        double x[RG][NC], vi[RG], wi[RG];
#pragma unroll
        for (int g = 0; g < RG; ++g) {
          vi[g] = vo[r0 + g];
          wi[g] = po[r0 + g] - hk * vi[g];
          const bool rl = r0 + g >= rlo && r0 + g < R;  // uniform
#pragma unroll
          for (int u = 0; u < NC; ++u) x[g][u] = rl && live[u] ? At[(r0 + g) * LD + u * T] : 0.0;
        }
#pragma unroll
        for (int g = 0; g < RG; ++g) {
          if (r0 + g >= rlo && r0 + g < R) {  // uniform
#pragma unroll
            for (int u = 0; u < NC; ++u)
              if (live[u] && tid + u * T < m)
                At[(r0 + g) * LD + u * T] = x[g][u] - __dadd_rn(__dmul_rn(vi[g], pw[u]), __dmul_rn(wi[g], vr[u]));
          }
        }
      }
    }
    {
      // replica rows k + 1 (v_{k+1} = 1) and k + 2, updated exactly as their owners do
      const double w1 = bc[4] - hk * 1.0;
      const double v2 = bc[6], w2 = bc[5] - hk * v2;
#pragma unroll
      for (int u = 0; u < NC; ++u) {
        const int j = tid + u * T;
        if (j > k && j < m) {
          r1[u] -= __dadd_rn(__dmul_rn(1.0, pw[u]), __dmul_rn(w1, vr[u]));
          r2[u] -= __dadd_rn(__dmul_rn(v2, pw[u]), __dmul_rn(w2, vr[u]));
        }
      }
    }
    if (k + 1 < kstop) {
      publish_row(k + 1);
      // the next reflector from row k + 1, which is final now
#pragma unroll
      for (int u = 0; u < NC; ++u) vr[u] = r1[u];
      reflector(k + 1, vr, tau);
    } else if (kstop == m - 2) {
      // the last 2 x 2 block: rows m - 2 (= k + 1) and m - 1 (= k + 2)
#pragma unroll
      for (int u = 0; u < NC; ++u) {
        const int j = tid + u * T;
        if (c == 0 && j == m - 2) a.d[m - 2] = r1[u];
        if (c == 0 && j == m - 1) {
          a.e[m - 2] = r1[u];
          a.d[m - 1] = r2[u];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < NC; ++u) r1[u] = r2[u];
    if (a.trace && c == 0 && tid == 0) a.trace[4 * k + 3] = gtimer();
  }
  if (kstop < m - 2) {
    // hand the trailing block (as updated by step kstop - 1) to the one-CTA
    // kernel: each thread its own columns of the owned rows i >= kstop
    const int nt = m - kstop;
    for (int r = 0; r < R; ++r) {
      const int i = c + r * P;
      if (i < kstop) continue;
#pragma unroll
      for (int u = 0; u < NC; ++u) {
        const int j = tid + u * T;
        if (j >= kstop && j < m) a.tail[static_cast<size_t>(j - kstop) * nt + (i - kstop)] = At[r * LD + u * T];
      }
    }
  }
}

// Trailing blocks up to kTriClusterMaxM (and whole matrices of that size):
// the same one-exchange-per-step reduction by ONE 16-CTA cluster, the
// exchange through distributed shared memory and one cluster barrier per
// step instead of tagged L2 words (a cluster barrier plus DSMEM reads cost
// well under the ~2.5 us L2 round trip of the grid).  CTA c keeps rows
// i = c, c + 16, ... (at most kTriClusterRows) of the block in shared memory.
// Per step: the owned rows' p_i and the CTA's partial of p^T v go to this
// CTA's shared memory (by step parity); cluster barrier; every CTA reads the
// p_j of its columns, row k + 2 (published by its owner at the end of the
// previous step) and the 16 partials from the other CTAs' shared memory.  A
// CTA can run at most one step ahead (the barrier), so two generations of
// every buffer suffice.
constexpr int kTriClusterSize = 16;
constexpr int kTriClusterRows = 32;
constexpr int kTriClusterNC = 2;  // column slots per thread (256 threads)
constexpr int kTriClusterMaxM = kTriClusterNC * kTriGridThreads;  // 512
constexpr int kTriClusterSmall = 2 * kTriClusterRows /*pbuf*/ + 2 /*kpart*/ + 2 * kTriClusterRows /*vo, po*/ +
                                 kTriClusterRows * (kTriGridThreads / 32) /*red*/ + kTriGridThreads / 32 + 8;
__host__ __device__ constexpr size_t tri_cluster_smem() {
  return sizeof(double) * (static_cast<size_t>(kTriClusterRows + 2) * kTriClusterMaxM + kTriClusterSmall);
}

__global__ void __launch_bounds__(kTriGridThreads, 1) tridiag_cluster_kernel(const double* __restrict__ G, int m,
                                                                             double* __restrict__ dout,
                                                                             double* __restrict__ eout) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ double sm[];
  constexpr int T = kTriGridThreads, NW = T / 32, NC = kTriClusterNC, LD = NC * T, P = kTriClusterSize;
  const int c = static_cast<int>(cluster.block_rank());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int R = (m - c + P - 1) / P;  // rows i = c + r P, r < R
  double* pbuf = sm;                            // [2][kTriClusterRows] p of the owned rows (read remotely)
  double* kpart = pbuf + 2 * kTriClusterRows;   // [2] this CTA's partial of p^T v (read remotely)
  double* vo = kpart + 2;                       // [kTriClusterRows]
  double* po = vo + kTriClusterRows;            // [kTriClusterRows]
  double* red = po + kTriClusterRows;           // [kTriClusterRows][NW]
  double* scratch = red + kTriClusterRows * NW;  // [NW]
  double* bc = scratch + NW;
  double* rowbuf = sm + kTriClusterSmall;       // [2][LD] row k + 2 by step parity (read remotely)
  double* At = rowbuf + 2 * LD + tid;           // owned rows: (r, u) at r LD + u T
  for (int r = 0; r < kTriClusterRows; ++r) {
    const double* gcol = G + static_cast<size_t>(min(c + r * P, m - 1)) * m;
#pragma unroll
    for (int u = 0; u < NC; ++u) {
      const int j = tid + u * T;
      At[r * LD + u * T] = r < R && j < m ? gcol[j] : 0.0;
    }
  }
  if (tid < 2 * kTriClusterRows) vo[tid] = 0.0;  // vo, po
  double r1[NC], vr[NC];
#pragma unroll
  for (int u = 0; u < NC; ++u) {
    const int j = tid + u * T;
    r1[u] = j < m ? G[static_cast<size_t>(1) * m + j] : 0.0;
    vr[u] = j < m ? G[j] : 0.0;
  }
  auto reflector = [&](int kk, double (&x)[NC], double& tau_out) {
    double sig = 0.0;
#pragma unroll
    for (int u = 0; u < NC; ++u) {
      const int j = tid + u * T;
      if (j > kk + 1 && j < m) sig = fma(x[u], x[u], sig);
      if (j == kk + 1) bc[0] = x[u];
      if (j == kk && c == 0) dout[kk] = x[u];
    }
    for (int o = 16; o > 0; o >>= 1) sig += __shfl_xor_sync(0xffffffffu, sig, o);
    if (lane == 0) scratch[warp] = sig;
    __syncthreads();
    double S = 0.0;
    for (int w = 0; w < NW; ++w) S += scratch[w];
    const double al = bc[0];
    double tau = 0.0, scal = 0.0, beta = al;
    if (S > 0.0) {
      const double nrm = sqrt(al * al + S);
      beta = -copysign(nrm, al);
      tau = (beta - al) / beta;
      scal = 1.0 / (al - beta);
    }
    if (c == 0 && tid == 0) eout[kk] = beta;
#pragma unroll
    for (int u = 0; u < NC; ++u) {
      const int j = tid + u * T;
      x[u] = j == kk + 1 ? 1.0 : (j > kk + 1 && j < m ? x[u] * scal : 0.0);
    }
    tau_out = tau;
    __syncthreads();
  };
  // row kk + 2 as it stands after step kk - 1 into this CTA's rowbuf (kk & 1)
  auto publish_row = [&](int kk) {
    if ((kk + 2) % P == c) {
      const double* row = At + ((kk + 2) / P) * LD;
      double* rb = rowbuf + (kk & 1) * LD + tid;
#pragma unroll
      for (int u = 0; u < NC; ++u) rb[u * T] = row[u * T];
    }
  };
  __syncthreads();
  if (m > 2) publish_row(0);
  double tau;
  reflector(0, vr, tau);
  for (int k = 0; k + 2 < m; ++k) {
    const int par = k & 1;
    const int rlo = c > k ? 0 : (k - c) / P + 1;
    bool live[NC];
#pragma unroll
    for (int u = 0; u < NC; ++u) live[u] = u * T + warp * 32 + 31 > k && u * T + warp * 32 < m;
#pragma unroll
    for (int u = 0; u < NC; ++u) {
      const int j = tid + u * T;
      if (j > k && j < m && j % P == c) vo[j / P] = vr[u];
    }
    // row sums in two passes of 16 rows (transposing butterfly)
#pragma unroll
    for (int r0 = 0; r0 < kTriClusterRows; r0 += 16) {
      double acc[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int r = r0 + q;
        acc[q] = 0.0;
        if (r >= rlo && r < R) {
#pragma unroll
          for (int u = 0; u < NC; ++u)
            if (live[u]) acc[q] = fma(At[r * LD + u * T], vr[u], acc[q]);
        }
      }
#pragma unroll
      for (int h = 8; h >= 1; h >>= 1) {
        const bool up = lane & (2 * h);
#pragma unroll
        for (int i = 0; i < h; ++i) {
          const double send = up ? acc[i] : acc[i + h];
          const double keep = up ? acc[i + h] : acc[i];
          acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2 * h);
        }
      }
      acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
      if ((lane & 1) == 0) red[(r0 + (lane >> 1)) * NW + warp] = acc[0];
    }
    __syncthreads();
    if (warp == 0) {
      const int r = lane;  // kTriClusterRows == 32
      double pv = 0.0;
      if (r < rlo) vo[r] = po[r] = 0.0;
      if (r >= rlo && r < R) {
        double s = 0.0;
        for (int w = 0; w < NW; ++w) s += red[r * NW + w];
        const double pi = tau * s;
        po[r] = pi;
        pbuf[par * kTriClusterRows + r] = pi;
        pv = pi * vo[r];
      }
      for (int o = 16; o > 0; o >>= 1) pv += __shfl_xor_sync(0xffffffffu, pv, o);
      if (lane == 0) kpart[par] = pv;
    }
    cluster.sync();  // every CTA's p, partial and row k + 2 are published
    double pw[NC], r2[NC];
#pragma unroll
    for (int u = 0; u < NC; ++u) {
      const int j = tid + u * T;
      pw[u] = 0.0;
      r2[u] = 0.0;
      if (j > k && j < m) {
        const double* rp = cluster.map_shared_rank(pbuf, j % P);
        pw[u] = rp[par * kTriClusterRows + j / P];
      }
      if (j >= k + 2 && j < m) {
        const double* rr = cluster.map_shared_rank(rowbuf, (k + 2) % P);
        r2[u] = rr[par * LD + j];
      }
    }
    if (warp == 0) {
      double K = lane < P ? cluster.map_shared_rank(kpart, lane)[par] : 0.0;
      for (int o = 16; o > 0; o >>= 1) K += __shfl_xor_sync(0xffffffffu, K, o);
      if (lane == 0) bc[3] = K;
    }
#pragma unroll
    for (int u = 0; u < NC; ++u) {
      const int j = tid + u * T;
      if (j == k + 1) bc[4] = pw[u];
      if (j == k + 2) {
        bc[5] = pw[u];
        bc[6] = vr[u];
      }
    }
    __syncthreads();
    const double hk = 0.5 * tau * bc[3];
#pragma unroll
    for (int u = 0; u < NC; ++u) pw[u] = pw[u] - hk * vr[u];
#pragma unroll 4
    for (int r = 0; r < kTriClusterRows; ++r) {
      if (r >= rlo && r < R) {
        const double vi = vo[r], wi = po[r] - hk * vi;
        double x[NC];
#pragma unroll
        for (int u = 0; u < NC; ++u) x[u] = live[u] ? At[r * LD + u * T] : 0.0;
#pragma unroll
        for (int u = 0; u < NC; ++u)
          if (live[u] && tid + u * T < m) At[r * LD + u * T] = x[u] - __dadd_rn(__dmul_rn(vi, pw[u]), __dmul_rn(wi, vr[u]));
      }
    }
    {
      const double w1 = bc[4] - hk * 1.0;
      const double v2 = bc[6], w2 = bc[5] - hk * v2;
#pragma unroll
      for (int u = 0; u < NC; ++u) {
        const int j = tid + u * T;
        if (j > k && j < m) {
          r1[u] -= __dadd_rn(__dmul_rn(1.0, pw[u]), __dmul_rn(w1, vr[u]));
          r2[u] -= __dadd_rn(__dmul_rn(v2, pw[u]), __dmul_rn(w2, vr[u]));
        }
      }
    }
    if (k + 3 < m) {
      publish_row(k + 1);
#pragma unroll
      for (int u = 0; u < NC; ++u) vr[u] = r1[u];
      reflector(k + 1, vr, tau);
    } else {
#pragma unroll
      for (int u = 0; u < NC; ++u) {
        const int j = tid + u * T;
        if (c == 0 && j == m - 2) dout[m - 2] = r1[u];
        if (c == 0 && j == m - 1) {
          eout[m - 2] = r1[u];
          dout[m - 1] = r2[u];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < NC; ++u) r1[u] = r2[u];
  }
  cluster.sync();  // no CTA leaves while peers may still read its shared memory
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

// Gershgorin interval of T widened by dstebz's pad, and its pivmin:
// prm = {lo, hi, pivmin} (min / max reductions: order-independent)
__global__ void __launch_bounds__(1024) gershgorin_kernel(const double* __restrict__ d,
                                                          const double* __restrict__ e, int m,
                                                          double* __restrict__ prm) {
  __shared__ double slo[32], shi[32], se2[32];
  double lo = INFINITY, hi = -INFINITY, e2 = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const double r = __dadd_rn(i > 0 ? fabs(e[i - 1]) : 0.0, i + 1 < m ? fabs(e[i]) : 0.0);
    lo = fmin(lo, __dsub_rn(d[i], r));
    hi = fmax(hi, __dadd_rn(d[i], r));
    if (i + 1 < m) e2 = fmax(e2, __dmul_rn(e[i], e[i]));
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    e2 = fmax(e2, __shfl_xor_sync(0xffffffffu, e2, o));
  }
  if ((threadIdx.x & 31) == 0) {
    slo[threadIdx.x >> 5] = lo;
    shi[threadIdx.x >> 5] = hi;
    se2[threadIdx.x >> 5] = e2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < static_cast<int>(blockDim.x >> 5); ++q) {
      lo = fmin(lo, slo[q]);
      hi = fmax(hi, shi[q]);
      e2 = fmax(e2, se2[q]);
    }
    const double tnorm = fmax(fabs(lo), fabs(hi));
    const double pivmin = __dmul_rn(2.2250738585072014e-308, fmax(1.0, e2));
    const double pad = __dadd_rn(__dmul_rn(__dmul_rn(2.0 * 2.220446049250313e-16, tnorm), static_cast<double>(m)),
                                 __dmul_rn(2.0, pivmin));
    prm[0] = __dsub_rn(lo, pad);
    prm[1] = __dadd_rn(hi, pad);
    prm[2] = pivmin;
  }
}

constexpr int kBisectWarps = 4;  // eigenvalues per 128-thread block
__global__ void __launch_bounds__(128) tridiag_bisect_kernel(const double* __restrict__ d,
                                                             const double* __restrict__ e, int m,
                                                             const double* __restrict__ prm,
                                                             double* __restrict__ w) {
  const double lo0 = prm[0], hi0 = prm[1], pivmin = prm[2];
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
