// dmma_f64.cuh -- FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) kernels of
// the train path: a grouped GEMM with triangle-aware K clipping and two
// epilogues (plain alpha/beta, and the Gram similarity map), and the
// single-CTA Cholesky + triangular-inverse leaf of the recursive
// factorisation in train_f64.cu.
//
// The reference's train arithmetic is FP64 throughout (types.hpp:13); B200
// has no tcgen05 f64 kind, so the FP64 tensor path is the legacy DMMA
// instruction (SASS `DMMA.884`).  Fragment layout of m8n8k4 (.row.col):
// lane l = 4 g + t holds A[g][t], B[t][g] and C[g][2t .. 2t+1].
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace csb {

// ------------------------------------------------------------------ GEMM
// One product C = alpha op(A) op(B) + beta C of a grouped launch.
// op(A) is M x K, op(B) is K x N, C is M x N, all column-major.
// Flags describe zero structure of the (logical) operands so a tile skips
// the K range that cannot contribute, and which output tiles to compute.
enum DgemmFlags : int {
  kALower = 1,    // op(A)(i, k) == 0 for k > i
  kAUpper = 2,    // op(A)(i, k) == 0 for k < i
  kBLower = 4,    // op(B)(k, j) == 0 for k < j
  kBUpper = 8,    // op(B)(k, j) == 0 for k > j
  kCLower = 16,   // compute only the lower triangle (i >= j); requires M == N
  kCMirror = 32,  // with kCLower: also write C(j, i) = C(i, j) (symmetric output)
};

struct DgemmProblem {
  const double* A;
  const double* B;
  double* C;
  int64_t lda, ldb, ldc;
  int M, N, K;
  int flags;
  double alpha, beta;
  int tiles_m, tiles;  // output tiles of this problem (filled by the host)
};

constexpr int kDgemmMaxGroup = 16;

struct DgemmGroup {
  DgemmProblem p[kDgemmMaxGroup];
  int count;
  int tile_start[kDgemmMaxGroup + 1];
};

// Gram epilogue (mset.cpp:151-152 via the GEMM form ||a||^2+||b||^2-2a.b):
// G(i, j) = k(d2), exact 1 on the diagonal (d2(x, x) = 0 exactly in the
// reference), and entries whose GEMM-form d2 is small relative to the norms
// (d2 < tau (dd_i + dd_j), where cancellation would dominate -- SURVEY H2)
// recomputed by direct differences in the reference's order
// (backends.cpp:139-150).
struct GramEpi {
  const double* Dn;  // n x m column-major (normalised memory vectors)
  const double* dd;  // ||Dn(:, i)||^2
  int64_t n;
  int kind;          // CS_KERNEL_INVERSE_DISTANCE / CS_KERNEL_GAUSSIAN
  double h;
  double tau;
};

namespace dmma {

__device__ __forceinline__ void mma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int sz = valid ? 8 : 0;  // src-size 0: zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ double kernel_from_d2(double d2, int kind, double h) {
  // kernels.hpp:54-57
  if (kind == 0) return 1.0 / (1.0 + sqrt(d2) / h);
  return exp(-d2 / (2.0 * h * h));
}

}  // namespace dmma

// Tile shape: BM x BN output per CTA, BK-deep shared-memory stages, warps of
// WM x WN.  Shared rows are padded by 8 doubles so a fragment load (4 k-rows
// x 8 consecutive i) touches all 32 banks twice (2 wavefronts, the minimum
// for 256 bytes).
template <int BM, int BN, int BK, int WM, int WN, int STAGES>
struct DgemmCfg {
  static constexpr int kWarps = (BM / WM) * (BN / WN);
  static constexpr int kThreads = kWarps * 32;
  static constexpr int kPadA = BM + 8, kPadB = BN + 8;
  static constexpr int kStageDoubles = BK * (kPadA + kPadB);
  static constexpr size_t kSmem = sizeof(double) * STAGES * kStageDoubles;
  static constexpr int MI = WM / 8, NI = WN / 8;
};

// Grouped FP64 GEMM.  TA: op(A) = A^T (A stored K x M); TB: op(B) = B^T.
// EPI 0: C = alpha acc + beta C.  EPI 1: Gram map (GramEpi), problem 0 only.
template <class Cfg, int BM, int BN, int BK, int WM, int WN, int STAGES, bool TA, bool TB, int EPI>
__global__ void __launch_bounds__(Cfg::kThreads)
dgemm_dmma_kernel(const __grid_constant__ DgemmGroup grp, const __grid_constant__ GramEpi gram) {
  extern __shared__ __align__(16) double smem[];
  // ---- which problem / tile
  int pi = 0;
  const int bid = blockIdx.x;
  while (pi + 1 < grp.count && bid >= grp.tile_start[pi + 1]) ++pi;
  const DgemmProblem& P = grp.p[pi];
  int t = bid - grp.tile_start[pi];
  int bm, bn;
  if (P.flags & kCLower) {
    // lower-triangle tile enumeration: t -> (bm >= bn)
    bm = static_cast<int>((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((bm + 1) * (bm + 2) / 2 <= t) ++bm;
    while (bm * (bm + 1) / 2 > t) --bm;
    bn = t - bm * (bm + 1) / 2;
  } else {
    bm = t % P.tiles_m;
    bn = t / P.tiles_m;
  }
  const int i0 = bm * BM, j0 = bn * BN;
  // ---- K range this tile needs
  int k_lo = 0, k_hi = P.K;
  if (P.flags & kALower) k_hi = min(k_hi, i0 + BM);
  if (P.flags & kBUpper) k_hi = min(k_hi, j0 + BN);
  if (P.flags & kAUpper) k_lo = max(k_lo, i0);
  if (P.flags & kBLower) k_lo = max(k_lo, j0);
  k_lo = (k_lo / BK) * BK;
  const int ktiles = k_hi > k_lo ? (k_hi - k_lo + BK - 1) / BK : 0;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp % (BM / WM)) * WM, wn0 = (warp / (BM / WM)) * WN;
  const int g = lane >> 2, tq = lane & 3;

  const double* __restrict__ A = P.A;
  const double* __restrict__ B = P.B;
  auto As = [&](int s) { return smem + s * Cfg::kStageDoubles; };
  auto Bs = [&](int s) { return smem + s * Cfg::kStageDoubles + BK * Cfg::kPadA; };

  auto load_stage = [&](int s, int kt) {
    const int kb = k_lo + kt * BK;
    double* as = As(s);
    double* bs = Bs(s);
    for (int e = tid; e < BM * BK; e += Cfg::kThreads) {
      int i, k;
      if (TA) { k = e % BK; i = e / BK; } else { i = e % BM; k = e / BM; }
      const int gi = i0 + i, gk = kb + k;
      const bool ok = gi < P.M && gk < k_hi;
      const double* src = TA ? A + (static_cast<int64_t>(gi) * P.lda + gk) : A + (gi + static_cast<int64_t>(gk) * P.lda);
      dmma::cp_async8(as + k * Cfg::kPadA + i, ok ? src : A, ok);
    }
    for (int e = tid; e < BN * BK; e += Cfg::kThreads) {
      int j, k;
      if (TB) { j = e % BN; k = e / BN; } else { k = e % BK; j = e / BK; }
      const int gj = j0 + j, gk = kb + k;
      const bool ok = gj < P.N && gk < k_hi;
      const double* src = TB ? B + (gj + static_cast<int64_t>(gk) * P.ldb) : B + (gk + static_cast<int64_t>(gj) * P.ldb);
      dmma::cp_async8(bs + k * Cfg::kPadB + j, ok ? src : B, ok);
    }
  };

  double acc[Cfg::MI][Cfg::NI][2];
#pragma unroll
  for (int a = 0; a < Cfg::MI; ++a)
#pragma unroll
    for (int b = 0; b < Cfg::NI; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_stage(s, s);
    dmma::cp_commit();
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    dmma::cp_wait<STAGES - 2>();
    __syncthreads();
    const int s = kt % STAGES;
    const double* as = As(s);
    const double* bs = Bs(s);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[Cfg::MI], bf[Cfg::NI];
#pragma unroll
      for (int a = 0; a < Cfg::MI; ++a) af[a] = as[(kk + tq) * Cfg::kPadA + wm0 + a * 8 + g];
#pragma unroll
      for (int b = 0; b < Cfg::NI; ++b) bf[b] = bs[(kk + tq) * Cfg::kPadB + wn0 + b * 8 + g];
#pragma unroll
      for (int a = 0; a < Cfg::MI; ++a)
#pragma unroll
        for (int b = 0; b < Cfg::NI; ++b) dmma::mma884(acc[a][b], af[a], bf[b]);
    }
    const int nk = kt + STAGES - 1;
    if (nk < ktiles) load_stage(nk % STAGES, nk);
    dmma::cp_commit();
  }
  dmma::cp_wait<0>();

  // ---- epilogue
#pragma unroll
  for (int a = 0; a < Cfg::MI; ++a) {
    const int i = i0 + wm0 + a * 8 + g;
#pragma unroll
    for (int b = 0; b < Cfg::NI; ++b) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int j = j0 + wn0 + b * 8 + 2 * tq + c;
        if (i >= P.M || j >= P.N) continue;
        if ((P.flags & kCLower) && i < j) continue;
        double v;
        if (EPI == 1) {
          if (i == j) {
            v = 1.0;  // d2(x, x) == 0 exactly: k(0) = 1 for both kernels
          } else {
            const double di = gram.dd[i], dj = gram.dd[j];
            double d2 = di + dj - 2.0 * acc[a][b][c];
            if (d2 < gram.tau * (di + dj)) {
              // cancellation-prone: direct differences, reference order
              const double* x = gram.Dn + static_cast<int64_t>(i) * gram.n;
              const double* y = gram.Dn + static_cast<int64_t>(j) * gram.n;
              double s = 0.0;
              for (int64_t k = 0; k < gram.n; ++k) {
                const double d = __dsub_rn(x[k], y[k]);
                s = __dadd_rn(s, __dmul_rn(d, d));
              }
              d2 = s;
            }
            v = dmma::kernel_from_d2(d2, gram.kind, gram.h);
          }
        } else {
          v = P.alpha * acc[a][b][c];
          if (P.beta != 0.0) v += P.beta * P.C[i + static_cast<int64_t>(j) * P.ldc];
        }
        P.C[i + static_cast<int64_t>(j) * P.ldc] = v;
        if ((P.flags & kCMirror) && i != j) P.C[j + static_cast<int64_t>(i) * P.ldc] = v;
      }
    }
  }
}

// ------------------------------------------------------ Cholesky leaf
// Factor the b x b (b <= kLeaf) diagonal block at (r0, r0) of the
// lower-triangular work matrix L (ld m) in shared memory, G_bb = L_bb L_bb^T,
// then invert L_bb in place (column by column from the right,
// X(j+1:, j) = -X(j+1:, j+1:) L(j+1:, j) / L(j, j)), and write X_bb = L_bb^-1
// into X.  A non-positive or non-finite pivot sets *fail (the caller then
// takes the reference's eigen route).  One CTA of kLeafThreads.
constexpr int kLeaf = 128;
constexpr int kLeafThreads = 512;
constexpr int kLeafLd = kLeaf;  // column stride 129 doubles in the trailing update: conflict-free

__global__ void __launch_bounds__(kLeafThreads)
chol_leaf_kernel(const double* __restrict__ L, int64_t m, int64_t r0, int b, double* __restrict__ X,
                 int* __restrict__ fail) {
  extern __shared__ double S[];  // [kLeaf cols][kLeafLd] column-major, + kLeaf temp
  double* col = S + kLeaf * kLeafLd;
  __shared__ int bad;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  for (int e = tid; e < b * b; e += kLeafThreads) {
    const int i = e % b, j = e / b;
    S[j * kLeafLd + i] = i >= j ? L[(r0 + i) + (r0 + j) * m] : 0.0;
  }
  __syncthreads();
  // right-looking Cholesky: thread (jc, q) owns column jc, rows i = q (mod 4)
  const int jc = tid % kLeaf, q = tid / kLeaf;
  for (int k = 0; k < b; ++k) {
    if (tid == 0) {
      const double d = S[k * kLeafLd + k];
      if (!(d > 0.0) || !isfinite(d)) bad = 1;
      S[k * kLeafLd + k] = sqrt(fmax(d, 0.0));
    }
    __syncthreads();
    const double piv = S[k * kLeafLd + k];
    for (int i = k + 1 + tid; i < b; i += kLeafThreads) S[k * kLeafLd + i] /= piv;
    __syncthreads();
    if (jc > k && jc < b) {
      const double ljk = S[k * kLeafLd + jc];
      for (int i = jc + q; i < b; i += kLeafThreads / kLeaf) S[jc * kLeafLd + i] -= S[k * kLeafLd + i] * ljk;
    }
    __syncthreads();
  }
  // in-place inverse, columns right to left; 4 threads per row share the sum
  const int row = tid / 4, part = tid % 4;
  for (int j = b - 1; j >= 0; --j) {
    if (tid < b) col[tid] = S[j * kLeafLd + tid];  // L(:, j) (rows > j) before it is overwritten
    __syncthreads();
    const double ljj = col[j];
    double s = 0.0;
    if (row > j && row < b) {
      for (int k = j + 1 + part; k <= row; k += 4) s += S[k * kLeafLd + row] * col[k];
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    __syncthreads();
    if (part == 0 && row > j && row < b) S[j * kLeafLd + row] = -s / ljj;
    if (tid == 0) S[j * kLeafLd + j] = 1.0 / ljj;
    __syncthreads();
  }
  for (int e = tid; e < b * b; e += kLeafThreads) {
    const int i = e % b, jj = e / b;
    X[(r0 + i) + (r0 + jj) * m] = i >= jj ? S[jj * kLeafLd + i] : 0.0;
  }
  if (tid == 0 && bad) atomicExch(fail, 1);
}

}  // namespace csb
