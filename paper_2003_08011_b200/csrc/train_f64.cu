// train_f64.cu -- FP64 train on the DMMA tensor pipe: Gram matrix with the
// similarity map fused in the GEMM epilogue, recursive blocked Cholesky
// inverse, and the plain GEMMs of the train path (P = D_norm G+).
//
// Reference: the Gram matrix is sim_matrix(Dn, Dn) (mset.cpp:151-152,
// backends.cpp:129-152); the pseudo-inverse is the eigen route of
// mset.cpp:153-170, which equals G^-1 when every eigenvalue passes the
// cutoff -- the certified full-rank fast path in cstress_b200.cu proves that
// from the 1-norm condition number of this inverse.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <vector>

#include "common.cuh"
#include "dmma_f64.cuh"
#include "train_f64.h"

namespace csb {
namespace {

// 64 x 64 tiles (4 warps of 32 x 32, 4 CTAs / SM) for large products;
// 32 x 32 tiles (4 warps of 16 x 16) when a launch has under two waves of
// 64-tiles -- the deep levels of the recursion, where parallelism, not DMMA
// issue, bounds the launch
using Cfg = DgemmCfg<64, 64, 16, 32, 32, 3>;
using CfgS = DgemmCfg<32, 32, 16, 16, 16, 4>;

__global__ void col_sqnorm_f64_kernel(const double* __restrict__ D, int64_t n, int64_t m, double* __restrict__ dd) {
  // one warp per column: coalesced reads, shuffle reduction
  const int64_t c = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= m) return;
  const double* x = D + c * n;
  double s = 0.0;
  for (int64_t k = lane; k < n; k += 32) s = fma(x[k], x[k], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) dd[c] = s;
}

// lower -> upper copy through 32 x 32 shared tiles (coalesced both ways)
__global__ void mirror_lower_kernel(double* __restrict__ A, int64_t m) {
  __shared__ double t[32][33];
  const int bi = blockIdx.y, bj = blockIdx.x;  // tile (bi, bj) of the lower triangle, bi >= bj
  if (bi < bj) return;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = 32 * bi + tx, j = 32 * bj + r;
    t[r][tx] = (i < m && j < m) ? A[i + j * m] : 0.0;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int64_t i = 32 * bj + tx, j = 32 * bi + r;  // upper element (i, j) = lower (j, i)
    if (i < m && j < m && j > i) A[i + j * m] = t[tx][r];
  }
}

template <class C>
int tiles_of(DgemmProblem& p) {
  p.tiles_m = (p.M + C::BM - 1) / C::BM;
  if (p.M <= 0 || p.N <= 0) return 0;
  if (p.flags & kCLower) return p.tiles_m * (p.tiles_m + 1) / 2;
  return p.tiles_m * ((p.N + C::BN - 1) / C::BN);
}

template <class C, int EPI>
void launch_cfg(cudaStream_t st, const std::vector<DgemmProblem>& probs, const GramEpi& ge) {
  static_assert(C::BM == C::BN, "lower-triangle tiling needs square tiles");
  thread_local unsigned attr_set = 0;  // per device bit: the attribute is per (function, device)
  int dev = 0;
  CSB_CUDA(cudaGetDevice(&dev));
  if (!(attr_set >> dev & 1u)) {
    CSB_CUDA(cudaFuncSetAttribute(dgemm_dmma_kernel<C, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(C::kSmem)));
    attr_set |= 1u << dev;
  }
  size_t i = 0;
  while (i < probs.size()) {
    DgemmGroup grp{};
    int total = 0;
    grp.count = 0;
    for (; i < probs.size() && grp.count < kDgemmMaxGroup; ++i) {
      DgemmProblem p = probs[i];
      const int t = tiles_of<C>(p);
      // the K range grows with the tile index under these structures: run
      // the heavy tiles first so the launch's tail is the light ones
      if (p.flags & (kALower | kBUpper)) p.flags |= kReverse;
      if (t == 0) continue;
      grp.tile_start[grp.count] = total;
      grp.p[grp.count++] = p;
      total += t;
    }
    grp.tile_start[grp.count] = total;
    if (total == 0) continue;
    dgemm_dmma_kernel<C, EPI><<<total, C::kThreads, C::kSmem, st>>>(grp, ge);
    CSB_LAUNCH_CHECK();
  }
}

template <int EPI>
void launch_group(cudaStream_t st, std::vector<DgemmProblem> probs, const GramEpi& ge = GramEpi{}) {
  std::stable_sort(probs.begin(), probs.end(), [](const DgemmProblem& a, const DgemmProblem& b) {
    return static_cast<double>(a.M) * a.N * a.K > static_cast<double>(b.M) * b.N * b.K;
  });
  int tiles64 = 0;
  for (DgemmProblem p : probs) tiles64 += tiles_of<Cfg>(p);
  if (tiles64 < 2 * 148) launch_cfg<CfgS, EPI>(st, probs, ge);
  else launch_cfg<Cfg, EPI>(st, probs, ge);
}

DgemmProblem prob(int flags, int M, int N, int K, double alpha, const double* A, int64_t lda, const double* B,
                  int64_t ldb, double beta, double* C, int64_t ldc) {
  DgemmProblem p{};
  p.A = A;
  p.B = B;
  p.C = C;
  p.lda = lda;
  p.ldb = ldb;
  p.ldc = ldc;
  p.M = M;
  p.N = N;
  p.K = K;
  p.flags = flags;
  p.alpha = alpha;
  p.beta = beta;
  return p;
}

// A second stream: the C = X^T X products of finished subtrees
// run there, in the gaps the latency-bound leaves leave on the first one.
struct SideStream {
  cudaStream_t s = nullptr;
  std::vector<cudaEvent_t> ev;
  size_t next = 0;
  bool leaf_attr = false;
  cudaEvent_t event() {
    if (next == ev.size()) {
      cudaEvent_t e;
      CSB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ev.push_back(e);
    }
    return ev[next++];
  }
};

// one per (host thread, device): a call's event pool is never shared
SideStream& side_stream() {
  thread_local std::map<int, SideStream> per_device;
  int dev = 0;
  CSB_CUDA(cudaGetDevice(&dev));
  SideStream& ss = per_device[dev];
  if (!ss.s) CSB_CUDA(cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking));
  return ss;
}

struct CholWork {
  cudaStream_t st;
  double* A;    // working copy of G: lower = trailing updates, upper = T^T scratch
  double* X;    // L^-1 (lower); L21 blocks parked in the X21 slots until replaced
  double* out;  // C = X^T X (lower)
  int64_t m;
  int* fail;
  SideStream* side;
};

// hand the finished part of X to the side stream and queue C products there
void side_products(const CholWork& w, std::vector<DgemmProblem> ps) {
  cudaEvent_t e = w.side->event();
  CSB_CUDA(cudaEventRecord(e, w.st));
  CSB_CUDA(cudaStreamWaitEvent(w.side->s, e, 0));
  launch_group<0>(w.side->s, std::move(ps));
}

// factor rows/cols [r0, r0 + b): L = chol(A_bb), X_bb = L^-1, and queue
// C_bb = X_bb^T X_bb (lower) on the side stream
void chol_rec(const CholWork& w, int64_t r0, int64_t b) {
  const int64_t m = w.m;
  auto a = [&](int64_t i, int64_t j) { return w.A + i + j * m; };
  auto x = [&](int64_t i, int64_t j) { return w.X + i + j * m; };
  auto c = [&](int64_t i, int64_t j) { return w.out + i + j * m; };
  if (b <= kLeaf) {
    chol_inv_leaf_kernel<<<1, kLeafThreads, kLeafSmem, w.st>>>(w.A, m, r0, static_cast<int>(b), w.X, m, w.fail);
    CSB_LAUNCH_CHECK();
    const int B = static_cast<int>(b);
    side_products(w, {prob(kTransA | kAUpper | kBLower | kCLower, B, B, B, 1.0, x(r0, r0), m, x(r0, r0), m, 0.0,
                           c(r0, r0), m)});
    return;
  }
  const int64_t b1 = ((b / 2 + kLeaf - 1) / kLeaf) * kLeaf, b2 = b - b1, r1 = r0 + b1;
  const int B1 = static_cast<int>(b1), B2 = static_cast<int>(b2);
  chol_rec(w, r0, b1);
  // L21 = A21 L11^-T = A21 X11^T  (parked in X21's slot)
  launch_group<0>(w.st, {prob(kTransB | kBUpper, B2, B1, B1, 1.0, a(r1, r0), m, x(r0, r0), m, 0.0, x(r1, r0), m)});
  // A22 -= L21 L21^T (lower) ; T^T = X11^T L21^T into A's unused upper block
  launch_group<0>(w.st, {prob(kTransB | kCLower, B2, B2, B1, -1.0, x(r1, r0), m, x(r1, r0), m, 1.0, a(r1, r1), m),
                         prob(kTransA | kAUpper | kTransB, B1, B2, B1, 1.0, x(r0, r0), m, x(r1, r0), m, 0.0,
                              a(r0, r1), m)});
  chol_rec(w, r1, b2);
  // X21 = -X22 (L21 X11) = -X22 T
  launch_group<0>(w.st, {prob(kALower | kTransB, B2, B1, B2, -1.0, x(r1, r1), m, a(r0, r1), m, 0.0, x(r1, r0), m)});
  // C = X^T X over this node (its children's C blocks are queued before):
  // C11 += X21^T X21, C21 = X22^T X21
  side_products(w, {prob(kTransA | kCLower, B1, B1, B2, 1.0, x(r1, r0), m, x(r1, r0), m, 1.0, c(r0, r0), m),
                    prob(kTransA | kAUpper, B2, B1, B2, 1.0, x(r1, r1), m, x(r1, r0), m, 0.0, c(r1, r0), m)});
}

}  // namespace

void dmma_gemm(cudaStream_t st, int flags, int M, int N, int K, double alpha, const double* A, int64_t lda,
               const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
  launch_group<0>(st, {prob(flags, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc)});
}

void dmma_gram(cudaStream_t st, const double* Dn, int64_t n, int64_t m, int kind, double h, double* G) {
  TmpBuf<double> dd(m);
  col_sqnorm_f64_kernel<<<ceil_div(m * 32, 256), 256, 0, st>>>(Dn, n, m, dd.get());
  CSB_LAUNCH_CHECK();
  GramEpi ge{Dn, dd.get(), n, kind, h, 1.0 / 64.0};
  const int mi = static_cast<int>(m), ni = static_cast<int>(n);
  launch_group<1>(st, {prob(kTransA | kCLower | kCMirror, mi, mi, ni, 1.0, Dn, n, Dn, n, 0.0, G, m)}, ge);
}

bool dmma_chol_inverse(cudaStream_t st, const double* G, int64_t m, double* out) {
  if (m == 0) return true;
  TmpBuf<double> A(static_cast<size_t>(m) * m), X(static_cast<size_t>(m) * m);
  TmpBuf<int> fail(1);
  CSB_CUDA(cudaMemcpyAsync(A.get(), G, m * m * sizeof(double), cudaMemcpyDeviceToDevice, st));
  CSB_CUDA(cudaMemsetAsync(X.get(), 0, m * m * sizeof(double), st));  // X's upper triangle stays 0
  CSB_CUDA(cudaMemsetAsync(fail.get(), 0, sizeof(int), st));
  SideStream& side = side_stream();
  if (!side.leaf_attr) {
    CSB_CUDA(cudaFuncSetAttribute(chol_inv_leaf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kLeafSmem)));
    side.leaf_attr = true;
  }
  side.next = 0;
  CholWork w{st, A.get(), X.get(), out, m, fail.get(), &side};
  chol_rec(w, 0, m);
  cudaEvent_t done = side.event();
  CSB_CUDA(cudaEventRecord(done, side.s));
  CSB_CUDA(cudaStreamWaitEvent(st, done, 0));
  const int tb = ceil_div(m, 32);
  mirror_lower_kernel<<<dim3(tb, tb), dim3(32, 8), 0, st>>>(out, m);
  CSB_LAUNCH_CHECK();
  int hf = 0;
  CSB_CUDA(cudaMemcpyAsync(&hf, fail.get(), sizeof hf, cudaMemcpyDeviceToHost, st));
  CSB_CUDA(cudaStreamSynchronize(st));
  return hf == 0;
}

}  // namespace csb
