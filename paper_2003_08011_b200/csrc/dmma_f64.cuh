// dmma_f64.cuh -- FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) kernels of
// the train path (train_f64.cu): a grouped GEMM with triangle-aware K
// clipping and two epilogues (alpha/beta, and the Gram similarity map), and
// the single-CTA Cholesky + triangular-inverse leaf of the recursive
// factorisation.
//
// The reference's train arithmetic is FP64 throughout (types.hpp:13); B200
// has no tcgen05 f64 kind, so the FP64 tensor path is the DMMA instruction
// (SASS `DMMA.884`, 37 TFLOP/s measured, profiles/peaks_probe.json).
// Fragment layout of m8n8k4 (.row.col): lane l = 4 g + t holds A[g][t],
// B[t][g] and C[g][2t .. 2t+1].
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace csb {

// ------------------------------------------------------------------ GEMM
// One product C = alpha op(A) op(B) + beta C of a grouped launch; op(A) is
// M x K, op(B) is K x N, C is M x N, all column-major.  Flags give the
// transposes and the zero structure of the logical operands, so a tile skips
// the K range that cannot contribute, and which output tiles to compute.
enum DgemmFlags : int {
  kALower = 1,    // op(A)(i, k) == 0 for k > i
  kAUpper = 2,    // op(A)(i, k) == 0 for k < i
  kBLower = 4,    // op(B)(k, j) == 0 for k < j
  kBUpper = 8,    // op(B)(k, j) == 0 for k > j
  kCLower = 16,   // compute only the lower triangle (i >= j); requires M == N
  kCMirror = 32,  // with kCLower: also write C(j, i) = C(i, j) (symmetric output)
  kTransA = 64,   // op(A) = A^T (A stored K x M)
  kTransB = 128,  // op(B) = B^T (B stored N x K)
  kReverse = 256, // enumerate tiles in reverse (heaviest K ranges first under kALower / kBUpper)
};

struct DgemmProblem {
  const double* A;
  const double* B;
  double* C;
  int64_t lda, ldb, ldc;
  int M, N, K;
  int flags;
  double alpha, beta;
  int tiles_m, pad_;
};

// small: the group is a kernel parameter, copied into every launch
constexpr int kDgemmMaxGroup = 4;

struct DgemmGroup {
  DgemmProblem p[kDgemmMaxGroup];
  int count;
  int tile_start[kDgemmMaxGroup + 1];
};

// Gram epilogue (mset.cpp:151-152 through the GEMM form ||a||^2 + ||b||^2 -
// 2 a.b): G(i, j) = k(d2) with the exact 1 on the diagonal (d2(x, x) = 0
// exactly in the reference), and any entry whose GEMM-form d2 is small
// relative to the norms (d2 < tau (dd_i + dd_j), where cancellation would
// dominate -- SURVEY H2) recomputed by direct differences in the reference's
// order (backends.cpp:139-150), so duplicate and near-duplicate memory
// vectors get the reference's values.
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
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(src) : "memory");
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
// WM x WN.  Shared rows are padded to a stride of 4 (mod 16) doubles: a
// 64-bit fragment load is served per half-warp (lanes g = 0..3 or 4..7,
// t = 0..3 reading k-row t, column g), and with that stride the 16 doubles of
// a half-warp land on 16 distinct bank pairs -- 2 wavefronts per load, the
// minimum.  (A stride of 8 mod 16 put k-rows t and t + 2 on the same banks:
// ncu measured 4.1-way conflicts and an L1-bound GEMM.)
template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_>
struct DgemmCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr int kWarps = (BM / WM) * (BN / WN);
  static constexpr int kThreads = kWarps * 32;
  static constexpr int kPadA = BM + 4, kPadB = BN + 4;
  static constexpr int kStageDoubles = BK * (kPadA + kPadB);
  static constexpr size_t kSmem = sizeof(double) * STAGES * kStageDoubles;
  static constexpr int MI = WM / 8, NI = WN / 8;
};

// Grouped FP64 GEMM.  EPI 0: C = alpha acc + beta C.  EPI 1: Gram map
// (GramEpi) for every problem of the group.
template <class Cfg, int EPI>
__global__ void __launch_bounds__(Cfg::kThreads)
dgemm_dmma_kernel(const __grid_constant__ DgemmGroup grp, const __grid_constant__ GramEpi gram) {
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, STAGES = Cfg::STAGES;
  extern __shared__ __align__(16) double smem[];
  // ---- which problem / tile
  int pi = 0;
  const int bid = blockIdx.x;
  while (pi + 1 < grp.count && bid >= grp.tile_start[pi + 1]) ++pi;
  const DgemmProblem& P = grp.p[pi];
  const int nt = grp.tile_start[pi + 1] - grp.tile_start[pi];
  const int t = (P.flags & kReverse) ? nt - 1 - (bid - grp.tile_start[pi]) : bid - grp.tile_start[pi];
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
  const bool ta = P.flags & kTransA, tb = P.flags & kTransB;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp % (BM / Cfg::WM)) * Cfg::WM, wn0 = (warp / (BM / Cfg::WM)) * Cfg::WN;
  const int g = lane >> 2, tq = lane & 3;

  const double* __restrict__ A = P.A;
  const double* __restrict__ B = P.B;
  auto As = [&](int s) { return smem + s * Cfg::kStageDoubles; };
  auto Bs = [&](int s) { return smem + s * Cfg::kStageDoubles + BK * Cfg::kPadA; };

  // stage loads: element (i, k) of op(A) goes to as[k * kPadA + i]; the
  // thread -> element map walks the contiguous dimension of the stored
  // operand so global reads coalesce
  auto load_stage = [&](int s, int kt) {
    const int kb = k_lo + kt * BK;
    double* as = As(s);
    double* bs = Bs(s);
    for (int e = tid; e < BM * BK; e += Cfg::kThreads) {
      int i, k;
      if (ta) { k = e % BK; i = e / BK; } else { i = e % BM; k = e / BM; }
      const int gi = i0 + i, gk = kb + k;
      const bool ok = gi < P.M && gk < k_hi;
      const double* src = ta ? A + (static_cast<int64_t>(gi) * P.lda + gk) : A + (gi + static_cast<int64_t>(gk) * P.lda);
      dmma::cp_async8(as + k * Cfg::kPadA + i, ok ? src : A, ok);
    }
    for (int e = tid; e < BN * BK; e += Cfg::kThreads) {
      int j, k;
      if (tb) { j = e % BN; k = e / BN; } else { k = e % BK; j = e / BK; }
      const int gj = j0 + j, gk = kb + k;
      const bool ok = gj < P.N && gk < k_hi;
      const double* src = tb ? B + (gj + static_cast<int64_t>(gk) * P.ldb) : B + (gk + static_cast<int64_t>(gj) * P.ldb);
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
// One CTA factors the b x b (b <= kLeaf) diagonal block at (r0, r0) of A
// (lower triangle read, ld lda), A_bb = L L^T, and writes X_bb = L^-1 (lower)
// into X.  Blocked by 32 inside the CTA:
//   factor:  for each 32-column block k: one warp factors L_kk in registers
//            (shuffle broadcasts; one reciprocal square root per pivot, no
//            FP64 division on the chain) and inverts it column-parallel
//            (X_kk, kept in place of L_kk); the panel below becomes
//            L_ik = A_ik X_kk^T and the trailing lower triangle takes the
//            rank-32 update A_ij -= L_ik L_jk^T -- both as warp-level DMMA
//            products over 16 x 16 output quadrants;
//   inverse: X_IJ = -X_II (sum_{K=J..I-1} L_IK X_KJ) by block distance
//            I - J = 1, 2, 3 (DMMA quadrants again); the diagonal X blocks
//            replace L's, the off-diagonal ones go to a second buffer.
// Column stride kLeafLd = 132 (4 mod 16): DMMA fragment loads are 2
// wavefronts (see DgemmCfg).  Padding rows / columns (b .. 32 nb) are the
// identity.  A non-positive or non-finite pivot sets *fail (the caller then
// takes the reference's eigen route).
constexpr int kLeaf = 128;
constexpr int kLeafThreads = 256;
constexpr int kLeafLd = 132;
constexpr int kLeafTLd = 36;
// S (the factor, 128 x 132) + Tm (3 pair products) + Xo (6 off-diagonal X blocks)
constexpr size_t kLeafSmem = sizeof(double) * (kLeaf * kLeafLd + 9 * 32 * kLeafTLd);
#ifdef CSB_LEAF_PROFILE
__device__ long long g_leaf_clk[64];
#define LEAF_MARK(slot) \
  if (threadIdx.x == 0) g_leaf_clk[slot] = clock64();
#else
#define LEAF_MARK(slot)
#endif

namespace dmma {
// 16 x 16 output quadrant of a warp: acc[a][b] is the m8n8 subtile (8a.., 8b..);
// lane (g, t) holds rows 8a + g, columns 8b + 2t, 8b + 2t + 1
template <class FA, class FB>
__device__ __forceinline__ void warp_mma16(double (&acc)[2][2][2], int K, FA a_at, FB b_at, int g, int t) {
  for (int k0 = 0; k0 < K; k0 += 4) {
    const double a0 = a_at(g, k0 + t), a1 = a_at(8 + g, k0 + t);
    const double b0 = b_at(k0 + t, g), b1 = b_at(k0 + t, 8 + g);
    mma884(acc[0][0], a0, b0);
    mma884(acc[0][1], a0, b1);
    mma884(acc[1][0], a1, b0);
    mma884(acc[1][1], a1, b1);
  }
}
}  // namespace dmma

__global__ void __launch_bounds__(kLeafThreads)
chol_inv_leaf_kernel(const double* __restrict__ A, int64_t lda, int64_t r0, int b, double* __restrict__ X,
                     int64_t ldx, int* __restrict__ fail) {
  extern __shared__ __align__(16) double S[];  // [kLeaf cols][kLeafLd]
  double* Tm = S + kLeaf * kLeafLd;            // [3][32 cols][kLeafTLd] products of the inverse phase
  double* Xo = Tm + 3 * 32 * kLeafTLd;         // [6][32 cols][kLeafTLd] X_IJ, I > J (column-major)
  LEAF_MARK(0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  constexpr int kWarps = kLeafThreads / 32;
  const int nb = (b + 31) / 32, bp = nb * 32;
  auto at = [&](int i, int j) -> double& { return S[j * kLeafLd + i]; };
  // X_IJ (I > J) lives in Xo, block index I (I - 1) / 2 + J
  auto xo = [&](int I, int J) -> double* { return Xo + (I * (I - 1) / 2 + J) * 32 * kLeafTLd; };
  // load: the bp x bp block by cp.async (16-byte copies of row pairs when
  // lda is even), then zero the diagonal blocks' upper parts and put the
  // identity on the padding
  if ((lda & 1) == 0 && (b & 1) == 0) {
    for (int j = warp; j < bp; j += kLeafThreads / 32)
      for (int i = 2 * lane; i < bp; i += 64) {
        if (i < b && j < b) dmma::cp_async16(&at(i, j), A + (r0 + i) + (r0 + j) * lda);
        else at(i, j) = at(i + 1, j) = 0.0;
      }
  } else {
    for (int j = warp; j < bp; j += kLeafThreads / 32)
      for (int i = lane; i < bp; i += 32) {
        const bool ok = i < b && j < b;
        dmma::cp_async8(&at(i, j), ok ? A + (r0 + i) + (r0 + j) * lda : A, ok);
      }
  }
  dmma::cp_commit();
  dmma::cp_wait<0>();
  __syncthreads();
  for (int e = tid; e < nb * 1024; e += kLeafThreads) {
    const int blk = e >> 10, i = (e >> 5) & 31, j = e & 31;
    if (i < j) at(32 * blk + i, 32 * blk + j) = 0.0;
  }
  for (int i = b + tid; i < bp; i += kLeafThreads) at(i, i) = 1.0;
  __syncthreads();
  LEAF_MARK(1);
  int bad = 0;
  for (int kb = 0; kb < nb; ++kb) {
    const int c0 = 32 * kb;
    if (warp == 0) {
      // L_kk: lane i holds row i of the block
      double r[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) r[k] = k <= lane ? at(c0 + lane, c0 + k) : 0.0;
      // the pivot chain: rsqrt -> scale -> the next diagonal on its own lane
      // -> one shuffle; the other lanes' updates hang off the chain
      // (column j of L is broadcast through shared memory: one store per
      // lane and broadcast loads, half the instructions of 64-bit shuffles)
      double* lc = Tm;  // [2][32], free until the inverse phase
      double piv = __shfl_sync(0xffffffffu, r[0], 0);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (!(piv > 0.0) || !isfinite(piv)) bad = 1;
        const double inv = rsqrt(fmax(piv, 1e-300));
        const double lj = lane == j ? piv * inv : (lane > j ? r[j] * inv : 0.0);
        r[j] = lj;
        if (j < 31) {
          lc[(j & 1) * 32 + lane] = lj;
          const double dnext = fma(-lj, lj, r[j + 1]);  // lane j + 1: its diagonal after step j
          piv = __shfl_sync(0xffffffffu, dnext, j + 1);
          __syncwarp();
#pragma unroll
          for (int k = j + 1; k < 32; ++k) r[k] = fma(-lj, lc[(j & 1) * 32 + k], r[k]);
        }
      }
      __syncwarp();
#ifdef CSB_LEAF_PROFILE
      if (lane == 0) g_leaf_clk[20 + kb] = clock64();
#endif
      double dl = r[0];
#pragma unroll
      for (int k = 1; k < 32; ++k)
        if (k == lane) dl = r[k];
      const double my_inv = 1.0 / dl;  // 1 / L(lane, lane): one division per lane, in parallel
#pragma unroll
      for (int k = 0; k < 32; ++k)
        if (k <= lane) at(c0 + lane, c0 + k) = r[k];
      __syncwarp();
#ifdef CSB_LEAF_PROFILE
      if (lane == 0) g_leaf_clk[24 + kb] = clock64();
#endif
      // X_kk = L_kk^-1 column-parallel: lane j owns column j;
      // X(i, j) = -(sum_{k=j}^{i-1} L(i, k) X(k, j)) / L(i, i)
      double x[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const double ii = __shfl_sync(0xffffffffu, my_inv, i);
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < i; ++k) s = fma(at(c0 + i, c0 + k), x[k], s);
        x[i] = i < lane ? 0.0 : (i == lane ? ii : -s * ii);
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i >= lane) at(c0 + i, c0 + lane) = x[i];  // the block's upper part stays 0
    }
    __syncthreads();
    LEAF_MARK(2 + 3 * kb);
    const int rem = nb - kb - 1;  // 32-blocks below / right of this one
    if (rem == 0) break;
    // panel: L_Ik = A_Ik X_kk^T for I > kb; a task owns 16 full rows (both
    // column quadrants), so it reads its rows completely before writing them
    for (int task = warp; task < rem * 2; task += kWarps) {
      const int I = kb + 1 + (task >> 1), qi = (task & 1) * 16;
      double acc[2][2][2][2] = {};
#pragma unroll
      for (int h = 0; h < 2; ++h)
        dmma::warp_mma16(
            acc[h], 32, [&](int i, int k) { return at(32 * I + qi + i, c0 + k); },
            [&](int k, int j) { return at(c0 + 16 * h + j, c0 + k); }, g, tq);  // X_kk(j, k): 0 for k > j
      __syncwarp();
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int bb = 0; bb < 2; ++bb)
#pragma unroll
            for (int c = 0; c < 2; ++c)
              at(32 * I + qi + 8 * a + g, c0 + 16 * h + 8 * bb + 2 * tq + c) = acc[h][a][bb][c];
    }
    __syncthreads();
    LEAF_MARK(3 + 3 * kb);
    // trailing: A_IJ -= L_Ik L_Jk^T for I >= J > kb (lower blocks; diagonal
    // blocks keep their upper part untouched)
    {
      const int nblk = rem * (rem + 1) / 2;
      for (int task = warp; task < nblk * 4; task += kWarps) {
        const int q = task >> 2;
        int bi = 0;
        while ((bi + 1) * (bi + 2) / 2 <= q) ++bi;
        const int bj = q - bi * (bi + 1) / 2;
        const int I = kb + 1 + bi, J = kb + 1 + bj;
        const int qi = ((task >> 1) & 1) * 16, qj = (task & 1) * 16;
        if (I == J && qi < qj) continue;  // upper quadrant of a diagonal block
        double acc[2][2][2] = {};
        dmma::warp_mma16(
            acc, 32, [&](int i, int k) { return at(32 * I + qi + i, c0 + k); },
            [&](int k, int j) { return at(32 * J + qj + j, c0 + k); }, g, tq);
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int bb = 0; bb < 2; ++bb)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const int i = 32 * I + qi + 8 * a + g, j = 32 * J + qj + 8 * bb + 2 * tq + c;
              if (i >= j) at(i, j) -= acc[a][bb][c];
            }
      }
    }
    __syncthreads();
    LEAF_MARK(4 + 3 * kb);
  }
  // inverse phase: X_IJ for I - J = d.  Storage: X_II in place of L_II
  // (lower, upper part 0), X_IJ (I > J) column-major in Xo.  Quadrant
  // tasks: (pair p, 16 x 16 quadrant)
  for (int d = 1; d < nb; ++d) {
    const int npairs = nb - d;
    // T_p = sum_{K=J}^{I-1} L_IK X_KJ for pair p = (I = J + d, J = p)
    for (int task = warp; task < npairs * 4; task += kWarps) {
      const int p = task >> 2, I = p + d, J = p, qi = ((task >> 1) & 1) * 16, qj = (task & 1) * 16;
      double acc[2][2][2] = {};
      dmma::warp_mma16(
          acc, 32, [&](int i, int k) { return at(32 * I + qi + i, 32 * J + k); },
          [&](int k, int j) { return at(32 * J + k, 32 * J + qj + j); }, g, tq);  // X_JJ in place
      for (int K = J + 1; K < I; ++K)
        dmma::warp_mma16(
            acc, 32, [&](int i, int k) { return at(32 * I + qi + i, 32 * K + k); },
            [&](int k, int j) { return xo(K, J)[(qj + j) * kLeafTLd + k]; }, g, tq);  // X_KJ (K > J)
      double* t = Tm + p * 32 * kLeafTLd;
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int bb = 0; bb < 2; ++bb)
#pragma unroll
          for (int c = 0; c < 2; ++c) t[(qj + 8 * bb + 2 * tq + c) * kLeafTLd + qi + 8 * a + g] = acc[a][bb][c];
    }
    __syncthreads();
    // X_IJ = -X_II T_p
    for (int task = warp; task < npairs * 4; task += kWarps) {
      const int p = task >> 2, I = p + d, J = p, qi = ((task >> 1) & 1) * 16, qj = (task & 1) * 16;
      const double* t = Tm + p * 32 * kLeafTLd;
      double acc[2][2][2] = {};
      dmma::warp_mma16(
          acc, 32, [&](int i, int k) { return at(32 * I + qi + i, 32 * I + k); },
          [&](int k, int j) { return t[(qj + j) * kLeafTLd + k]; }, g, tq);
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int bb = 0; bb < 2; ++bb)
#pragma unroll
          for (int c = 0; c < 2; ++c)
            xo(I, J)[(qj + 8 * bb + 2 * tq + c) * kLeafTLd + qi + 8 * a + g] = -acc[a][bb][c];
    }
    __syncthreads();
    LEAF_MARK(14 + d);
  }
  for (int j = warp; j < b; j += kLeafThreads / 32)
    for (int i = lane; i < b; i += 32)
      X[(r0 + i) + (r0 + j) * ldx] =
          i < j ? 0.0 : ((i >> 5) == (j >> 5) ? at(i, j) : xo(i >> 5, j >> 5)[(j & 31) * kLeafTLd + (i & 31)]);
  if (warp == 0 && __any_sync(0xffffffffu, bad) && lane == 0) atomicExch(fail, 1);
  LEAF_MARK(18);
}

}  // namespace csb
