// cstress_b200.cu -- C-ABI implementation (include/cstress_b200.h).
//
// Host orchestration of the B200 MSET2 path: contexts (device + streams +
// cuSOLVER handle + workspace), device-resident models, train (selection ->
// scale -> Gram -> eig -> pseudo-inverse -> FP32 operand packing) and the two
// surveillance paths.  Reference citations are path:line under
// /root/reference/proj.
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>
#include <chrono>
#include <map>
#include <functional>
#include <mutex>
#include <tuple>
#include <type_traits>
#include <cstdlib>

#include "common.cuh"
#include "estimate_tc.cuh"
#include "gemm_tc.cuh"
#include "sprt.cuh"
#include "kernels_f64.cuh"
#include "selection.cuh"
#include "solver.cuh"
#include "synth.cuh"
#include "train_f64.h"
#include "eig_tridiag.cuh"

using namespace csb;

namespace {
thread_local std::string g_last_error;

cs_status record(cs_status code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

template <typename F>
cs_status guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return CS_OK;
  } catch (const Failure& e) {
    return record(e.code, e.msg);
  } catch (const std::bad_alloc&) {
    return record(CS_ERROR, "host allocation failed");
  } catch (const std::exception& e) {
    return record(CS_ERROR, e.what());
  }
}

void solver_check(cusolverStatus_t s, const char* what) {
  if (s != CUSOLVER_STATUS_SUCCESS) {
    char buf[256];
    std::snprintf(buf, sizeof buf, "cuSOLVER error %d in %s", static_cast<int>(s), what);
    fail(CS_ERROR, buf);
  }
}

int grid_for(int64_t total, int threads = 256) {
  const int64_t b = (total + threads - 1) / threads;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32)));
}

}  // namespace

// ------------------------------------------------------------------ structs
struct cs_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
#ifndef CSB_IO_SLOTS
#define CSB_IO_SLOTS 3
#endif
  static constexpr int kSlots = CSB_IO_SLOTS;  // host-API pipeline depth (streams / buffer sets)
  cudaStream_t aux[kSlots] = {};
  cusolverDnHandle_t solver = nullptr;
  cublasHandle_t blas = nullptr;
  int sm_count = 148;
  std::string name;
  // workspace (grow-only)
  DevBuf<double> wsA, wsB, wsC, wsD;
  DevBuf<double> io_in[kSlots], io_est[kSlots], io_res[kSlots];
  DevBuf<unsigned char> wsBytes;
  DevBuf<__half> wsX[kSlots], wsS[kSlots];  // large-n surveillance (per stream slot): x, S operands
  DevBuf<float> wsXX[kSlots];                // ||x||^2
  // pinned host staging for the small per-call transfers (grow-only)
  void* pin = nullptr;
  size_t pin_bytes = 0;
  void* pinned(size_t bytes) {
    if (bytes > pin_bytes) {
      if (pin) cudaFreeHost(pin);
      pin = nullptr;
      pin_bytes = 0;
      if (cudaMallocHost(&pin, bytes) != cudaSuccess) throw std::bad_alloc();
      pin_bytes = bytes;
    }
    return pin;
  }
};

struct cs_model {
  int device = 0;
  int64_t n = 0, m = 0, rank = 0;
  int kind = CS_KERNEL_INVERSE_DISTANCE;
  double h = 0.0;
  int precision = CS_PRECISION_FP64;
  std::vector<int64_t> source_indices;
  // eigen_spectrum: computed at train time on the eigen paths; on the
  // certified-Cholesky path it is materialised on first export (one
  // eigenvalues-only solve of the re-formed Gram matrix)
  mutable std::vector<double> spectrum_host;
  mutable DevBuf<double> spectrum;
  mutable bool spectrum_ready = true;
  mutable std::mutex spectrum_mu;
  DevBuf<double> D, Dn, scale, pinv;
  // FP32 tensor-core operands (precision == CS_PRECISION_FP32)
  bool tc = false;
  int MT = 0, NB = 1, SB = 1, K1 = 0, N2 = 0, m_tiles = 0, n_stages = 2;
  DevBuf<__half> dn_tiles, p_tiles;  // 3xFP16 operand tiles (pack_tc.cuh)
  DevBuf<float> dd, dn32, inv_scale, scale_f, scale_out_f;
  DevBuf<double> p_shift, scale_out_d;  // per-signal 2^-k_s, scale_s * 2^(k_s - 14)
  float dd_max = 0.f;  // max ||D_norm(:, i)||^2 (near-zero guard prefilter)
  float s_center = 0.f;         // similarity centring of the two-GEMM path (gemm_tc.cuh EpiSim)
  DevBuf<float> add_f;          // n: scale_s * s_center * rowsum(P)_s
  DevBuf<double> add_d;
  float aug_x = 1.f;   // x's value in the ||d||^2 column (2^k_aug)
  // large-n two-GEMM path (gemm_tc.cuh), used when the fused kernel's TMEM
  // plan does not fit (n > ~130)
  bool gemm = false;
  int bnA = 256, ntA = 0, kcA = 0, bnB = 256, ntB = 0, kcB = 0;
  DevBuf<__half> dn_gemm, p_gemm;
};

namespace {

void set_device(int dev) { CSB_CUDA(cudaSetDevice(dev)); }

// ------------------------------------------------------------ FP64 launches
void launch_sim_exact(cudaStream_t st, const double* A, int64_t lda, const double* B, int64_t ldb,
                      int64_t n, int64_t p, int64_t q, int kind, double h, double* out,
                      int64_t ldo) {
  if (p == 0 || q == 0) return;
  dim3 grid(ceil_div(p, kTile), ceil_div(q, kTile));
  sim_exact_kernel<<<grid, kThreads, 0, st>>>(A, lda, B, ldb, n, p, q, kind, h, out, ldo);
  CSB_LAUNCH_CHECK();
}

template <bool TA, bool TB>
void launch_gemm_exact(cudaStream_t st, const double* A, int64_t lda, const double* B, int64_t ldb,
                       int64_t p, int64_t k, int64_t q, double* C, int64_t ldc) {
  if (p == 0 || q == 0) return;
  dim3 grid(ceil_div(p, kTile), ceil_div(q, kTile));
  gemm_exact_kernel<TA, TB><<<grid, kThreads, 0, st>>>(A, lda, B, ldb, p, k, q, C, ldc);
  CSB_LAUNCH_CHECK();
}

void check_kind(int kind) {
  if (kind != CS_KERNEL_INVERSE_DISTANCE && kind != CS_KERNEL_GAUSSIAN)
    fail(CS_CONFIG_ERROR, "unknown kernel kind");
}

double resolve_h(double h, int64_t n) {
  // KernelConfig::resolved (kernels.hpp:30-34); validate() (kernels.hpp:24-27)
  const double r = h > 0.0 ? h : std::sqrt(static_cast<double>(n));
  if (!(r > 0.0)) fail(CS_CONFIG_ERROR, "kernel bandwidth must be > 0");
  return r;
}

// --------------------------------------------------------------- selection
// select_memory_vectors (mset.cpp:72-137); X is device N x n col-major.
// picked_host == nullptr: the indices go to ctx's pinned block without a
// sync (train_device copies them out after its final synchronisation)
void select_device(cs_ctx* ctx, const double* X, int64_t N, int64_t n, int64_t m,
                   DevBuf<int64_t>& picked, std::vector<int64_t>* picked_host) {
  cudaStream_t st = ctx->stream;
  if (m < 2 * n) {
    char buf[160];
    std::snprintf(buf, sizeof buf, "select_memory_vectors: m=%lld violates m >= 2n with n=%lld",
                  static_cast<long long>(m), static_cast<long long>(n));
    fail(CS_CONSTRAINT_VIOLATED, buf);
  }
  if (m > N) {
    char buf[160];
    std::snprintf(buf, sizeof buf, "select_memory_vectors: m=%lld exceeds %lld training observations",
                  static_cast<long long>(m), static_cast<long long>(N));
    fail(CS_INSUFFICIENT_TRAINING, buf);
  }
  // byte workspace: hashes (2N u64), keys (2N u64), rows (2N i64), flags (N), misc
  TmpBuf<unsigned long long> h1(N), h2(N);
  TmpBuf<int64_t> r1(N), r2(N), imin(n), imax(n), npicked(1);
  TmpBuf<unsigned char> selected(N);
  TmpBuf<unsigned long long> count(1);
  picked.resize(m);

  row_hash_kernel<<<ceil_div(N, 256), 256, 0, st>>>(X, N, n, h1.get());
  CSB_LAUNCH_CHECK();
  size_t tmp_bytes = 0, tmp2 = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, h1.get(), h2.get(), static_cast<int>(N), 0, 64, st);
  cub::DeviceRadixSort::SortPairs(nullptr, tmp2, h1.get(), h2.get(), r1.get(), r2.get(),
                                  static_cast<int>(N), 0, 64, st);
  ctx->wsBytes.resize(std::max(tmp_bytes, tmp2) + 16);
  tmp_bytes = ctx->wsBytes.count;
  CSB_CUDA(cub::DeviceRadixSort::SortKeys(ctx->wsBytes.get(), tmp_bytes, h1.get(), h2.get(),
                                          static_cast<int>(N), 0, 64, st));
  CSB_CUDA(cudaMemsetAsync(count.get(), 0, sizeof(unsigned long long), st));
  count_distinct_kernel<<<grid_for(N), 256, 0, st>>>(h2.get(), N, count.get());
  CSB_LAUNCH_CHECK();
  unsigned long long distinct = 0;
  CSB_CUDA(cudaMemcpyAsync(&distinct, count.get(), sizeof distinct, cudaMemcpyDeviceToHost, st));
  CSB_CUDA(cudaStreamSynchronize(st));
  if (static_cast<unsigned long long>(m) > distinct) {
    char buf[160];
    std::snprintf(buf, sizeof buf,
                  "select_memory_vectors: m=%lld exceeds %llu distinct training observations",
                  static_cast<long long>(m), distinct);
    fail(CS_INSUFFICIENT_TRAINING, buf);
  }
  // stage 1
  col_extrema_kernel<<<static_cast<unsigned>(n), 256, 0, st>>>(X, N, imin.get(), imax.get());
  CSB_LAUNCH_CHECK();
  CSB_CUDA(cudaMemsetAsync(selected.get(), 0, N, st));
  TmpBuf<unsigned> first(N);
  CSB_CUDA(cudaMemsetAsync(first.get(), 0xff, N * sizeof(unsigned), st));
  stage1_dedupe_kernel<<<1, 1024, 0, st>>>(imin.get(), imax.get(), n, selected.get(), picked.get(),
                                           npicked.get(), first.get());
  CSB_LAUNCH_CHECK();
  // stage 2
  row_norm_key_kernel<<<ceil_div(N, 256), 256, 0, st>>>(X, N, n, selected.get(), h1.get(), r1.get());
  CSB_LAUNCH_CHECK();
  tmp_bytes = ctx->wsBytes.count;
  CSB_CUDA(cub::DeviceRadixSort::SortPairs(ctx->wsBytes.get(), tmp_bytes, h1.get(), h2.get(),
                                           r1.get(), r2.get(), static_cast<int>(N), 0, 64, st));
  stride_pick_kernel<<<grid_for(m), 256, 0, st>>>(r2.get(), N, m, npicked.get(), picked.get());
  CSB_LAUNCH_CHECK();
  if (!picked_host) {
    CSB_CUDA(cudaMemcpyAsync(ctx->pinned(m * sizeof(int64_t)), picked.get(), m * sizeof(int64_t),
                             cudaMemcpyDeviceToHost, st));
    return;
  }
  picked_host->resize(m);
  CSB_CUDA(cudaMemcpyAsync(picked_host->data(), picked.get(), m * sizeof(int64_t),
                           cudaMemcpyDeviceToHost, st));
  CSB_CUDA(cudaStreamSynchronize(st));
}

// ------------------------------------------- eigenvalues without cuSOLVER
// (eig_tridiag.cuh): shared-memory tridiagonalisation + bisection, m <= kTriMaxM.
// Returns false when the grid cannot be co-resident (the caller then uses
// syevd).  w is a device array (ascending).
bool bisect_eigvals(cudaStream_t st, const double* dd, const double* de, int64_t m, double* w);
// one 16-CTA cluster reduces the m x m block G (m <= kTriClusterMaxM) to
// (d, e); false when the device cannot launch such a cluster
bool tri_cluster_available(cs_ctx* ctx) {
  if (std::getenv("CSB_EIG_NO_CLUSTER")) return false;
  static int ok_by_dev[64] = {};  // 0 unknown, 1 yes, -1 no
  static std::mutex mu;
  {
    std::lock_guard<std::mutex> lock(mu);
    int& ok = ok_by_dev[ctx->device & 63];
    if (ok == 0) {
      ok = -1;
      if (cudaFuncSetAttribute(tridiag_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
              cudaSuccess &&
          cudaFuncSetAttribute(tridiag_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(tri_cluster_smem())) == cudaSuccess) {
        cudaLaunchConfig_t q{};
        q.gridDim = dim3(kTriClusterSize);
        q.blockDim = dim3(kTriGridThreads);
        q.dynamicSmemBytes = tri_cluster_smem();
        cudaLaunchAttribute at{};
        at.id = cudaLaunchAttributeClusterDimension;
        at.val.clusterDim.x = kTriClusterSize;
        at.val.clusterDim.y = 1;
        at.val.clusterDim.z = 1;
        q.attrs = &at;
        q.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, tridiag_cluster_kernel, &q) == cudaSuccess && n > 0) ok = 1;
      }
      cudaGetLastError();
    }
    return ok == 1;
  }
}
bool tri_cluster_reduce(cs_ctx* ctx, cudaStream_t st, const double* G, int64_t m, double* d, double* e) {
  if (m > kTriClusterMaxM || !tri_cluster_available(ctx)) return false;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kTriClusterSize);
  cfg.blockDim = dim3(kTriGridThreads);
  cfg.dynamicSmemBytes = tri_cluster_smem();
  cfg.stream = st;
  cudaLaunchAttribute at{};
  at.id = cudaLaunchAttributeClusterDimension;
  at.val.clusterDim.x = kTriClusterSize;
  at.val.clusterDim.y = 1;
  at.val.clusterDim.z = 1;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  CSB_CUDA(cudaLaunchKernelEx(&cfg, tridiag_cluster_kernel, G, static_cast<int>(m), d, e));
  CSB_LAUNCH_CHECK();
  return true;
}

bool tridiag_eigvals(cs_ctx* ctx, const double* G, int64_t m, double* w) {
  if (m < 1 || m > kTriMaxM) return false;
  // Default for m <= kTriMaxM, where it beats syevd: one CTA with the matrix
  // in shared memory up to kTriCtaMaxM, the co-resident grid above
  // (eig_tridiag.cuh has the measurements); CSB_EIG_OWN=0: never.
  const char* own = std::getenv("CSB_EIG_OWN");
  if (own && own[0] == '0') return false;
  cudaStream_t st = ctx->stream;
  StreamScope scope(st);
  TmpBuf<double> d(m), e(m + 1);
  if (m <= kTriCtaMaxM) {
    // the attribute is per (function, device)
    static std::atomic<unsigned long long> attr_dev{0};
    if (!(attr_dev.load() >> ctx->device & 1ull)) {
      CSB_CUDA(cudaFuncSetAttribute(tridiag_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(tri_cta_smem(kTriCtaMaxM))));
      attr_dev.fetch_or(1ull << ctx->device);
    }
    tridiag_cta_kernel<<<1, kTriCtaThreads, tri_cta_smem(static_cast<int>(m)), st>>>(G, static_cast<int>(m), d.get(),
                                                                                     e.get());
    CSB_LAUNCH_CHECK();
    return bisect_eigvals(st, d.get(), e.get(), m, w);
  }
  // one 16-CTA cluster with the whole matrix in distributed shared memory
  if (tri_cluster_reduce(ctx, st, G, m, d.get(), e.get())) return bisect_eigvals(st, d.get(), e.get(), m, w);
  // co-resident grid, rows in shared memory: up to kTriGridRows rows of
  // NC x kTriGridThreads doubles per CTA, as many CTAs as that takes (<= SMs)
  int sms = 0, optin = 0;
  CSB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
  CSB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
  const int nc = m <= kTriGridThreads ? 1 : m <= 2 * kTriGridThreads ? 2 : m <= 4 * kTriGridThreads ? 4 : 8;
  const void* fn = nc == 1   ? reinterpret_cast<const void*>(tridiag_grid_kernel<1>)
                   : nc == 2 ? reinterpret_cast<const void*>(tridiag_grid_kernel<2>)
                   : nc == 4 ? reinterpret_cast<const void*>(tridiag_grid_kernel<4>)
                             : reinterpret_cast<const void*>(tridiag_grid_kernel<8>);
  cudaFuncAttributes fa{};
  CSB_CUDA(cudaFuncGetAttributes(&fa, fn));
  const int64_t row_bytes = static_cast<int64_t>(tri_grid_smem(nc, 1) - tri_grid_smem(nc, 0));
  const int64_t room = static_cast<int64_t>(optin) - static_cast<int64_t>(tri_grid_smem(nc, 0) + fa.sharedSizeBytes);
  int rows = kTriGridRows;
  if (const char* r = std::getenv("CSB_EIG_GRID_ROWS")) rows = std::max(1, std::min(kTriGridRows, std::atoi(r)));
  rows = static_cast<int>(std::min<int64_t>(rows, room / row_bytes));
  if (rows < 1) return false;
  const int P = static_cast<int>((m + rows - 1) / rows);
  const int Rmax = static_cast<int>((m + P - 1) / P);
  const size_t smem = tri_grid_smem(nc, Rmax);
  CSB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  CSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kTriGridThreads, smem));
  if (P > kTriGridMaxP || P > per_sm * sms) return false;  // cannot be co-resident: syevd
  TmpBuf<ulonglong2> pb(2 * m), rb(2 * m), kb(2 * static_cast<size_t>(P));
  // stale tags from an earlier call must not match this call's steps
  CSB_CUDA(cudaMemsetAsync(pb.get(), 0, 2 * m * sizeof(ulonglong2), st));
  CSB_CUDA(cudaMemsetAsync(rb.get(), 0, 2 * m * sizeof(ulonglong2), st));
  CSB_CUDA(cudaMemsetAsync(kb.get(), 0, 2 * static_cast<size_t>(P) * sizeof(ulonglong2), st));
  const bool trace = std::getenv("CSB_EIG_TRACE") != nullptr;  // development: per-step timeline
  TmpBuf<unsigned long long> tr(trace ? 4 * m : 1);
  // the last kTriCtaMaxM columns go to the one-CTA kernel (~4 us per step
  // there against ~6.5 us per grid step: the exchange latency)
  // (measured: -7..-10% at m = 500 .. 2000; at m <= 2 kTriCtaMaxM the grid
  // part is too short to pay for the hand-off)
  const bool cl_tail = m > kTriClusterMaxM + 2 && tri_cluster_available(ctx);
  const int nt = std::getenv("CSB_EIG_NO_TAIL") ? 2
                 : cl_tail                       ? kTriClusterMaxM
                 : (m <= 2 * kTriCtaMaxM)        ? 2
                                                 : kTriCtaMaxM;
  const int kstop = static_cast<int>(m) - nt;
  TmpBuf<double> tail(static_cast<size_t>(nt) * nt);
  TriGridArgs ga{G, static_cast<int>(m), P, d.get(), e.get(), pb.get(), rb.get(), kb.get(), trace ? tr.get() : nullptr,
                 kstop, tail.get()};
  void* args[] = {&ga};
  const cudaError_t launched = cudaLaunchCooperativeKernel(fn, dim3(P), dim3(kTriGridThreads), args, smem, st);
  if (launched == cudaErrorCooperativeLaunchTooLarge || launched == cudaErrorNotSupported) {
    cudaGetLastError();  // the grid cannot be co-resident here (e.g. a partitioned device): syevd
    return false;
  }
  CSB_CUDA(launched);
  CSB_LAUNCH_CHECK();
  if (trace) {
    std::vector<unsigned long long> h(4 * m);
    CSB_CUDA(cudaMemcpyAsync(h.data(), tr.get(), 4 * m * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaStreamSynchronize(st));
    double s3[3] = {0, 0, 0};
    int cnt = 0;
    for (int64_t k = 0; k + 1 < kstop; ++k, ++cnt) {
      s3[0] += double(h[4 * k + 2] - h[4 * k + 1]);        // exchange (slowest CTA + hop)
      s3[1] += double(h[4 * k + 3] - h[4 * k + 2]);        // update + next reflector
      s3[2] += double(h[4 * (k + 1) + 1] - h[4 * k + 3]);  // row sums + publish
    }
    std::fprintf(stderr, "eig grid m=%lld P=%d ns/step: exchange %.0f  update+reflector %.0f  row sums %.0f\n",
                 static_cast<long long>(m), P, s3[0] / cnt, s3[1] / cnt, s3[2] / cnt);
  }
  if (nt == kTriClusterMaxM) {
    if (!tri_cluster_reduce(ctx, st, tail.get(), nt, d.get() + kstop, e.get() + kstop))
      fail(CS_ERROR, "eigenvalues: cluster tail launch failed");
  } else if (nt > 2) {
    // (the attribute is per (function, device): set by the small path above on first use)
    static std::atomic<unsigned long long> tail_attr_dev{0};
    if (!(tail_attr_dev.load() >> ctx->device & 1ull)) {
      CSB_CUDA(cudaFuncSetAttribute(tridiag_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(tri_cta_smem(kTriCtaMaxM))));
      tail_attr_dev.fetch_or(1ull << ctx->device);
    }
    tridiag_cta_kernel<<<1, kTriCtaThreads, tri_cta_smem(nt), st>>>(tail.get(), nt, d.get() + kstop, e.get() + kstop);
    CSB_LAUNCH_CHECK();
  }
  return bisect_eigvals(st, d.get(), e.get(), m, w);
}

// eigenvalues (ascending) of the device tridiagonal (d, e) by bisection; the
// Gershgorin interval and LAPACK dstebz's pivmin are reduced on the device
// (no host round trip)
bool bisect_eigvals(cudaStream_t st, const double* dd, const double* de, int64_t m, double* w) {
  TmpBuf<double> prm(3);
  gershgorin_kernel<<<1, 1024, 0, st>>>(dd, de, static_cast<int>(m), prm.get());
  CSB_LAUNCH_CHECK();
  const size_t smem = static_cast<size_t>(2) * m * sizeof(double);
  tridiag_bisect_kernel<<<ceil_div(m, kBisectWarps), 128, smem, st>>>(dd, de, static_cast<int>(m), prm.get(), w);
  CSB_LAUNCH_CHECK();
  return true;  // stream-ordered: the temporaries are freed on st after the kernels
}

// ---------------------------------------------------------- eigensolver
// symmetric_eig (mset.cpp:57-70): precondition check, then cuSOLVER syevd
// (FP64, ascending eigenvalues, orthonormal eigenvectors) in place on V.
// `check` = false for the train's own Gram matrices (mirrored, symmetric by
// construction): skips the precondition's device reduction and host sync.
void eig_device(cs_ctx* ctx, const double* G, int64_t m, double* w, double* V, bool vectors = true,
                bool check = true) {
  cudaStream_t st = ctx->stream;
  if (m == 0) return;
  if (check) {
  TmpBuf<unsigned long long> stats(2);
  CSB_CUDA(cudaMemsetAsync(stats.get(), 0, 2 * sizeof(unsigned long long), st));
  symmetry_stats_kernel<<<grid_for(m * m), 256, 0, st>>>(G, m, stats.get());
  CSB_LAUNCH_CHECK();
  unsigned long long hs[2];
  CSB_CUDA(cudaMemcpyAsync(hs, stats.get(), sizeof hs, cudaMemcpyDeviceToHost, st));
  CSB_CUDA(cudaStreamSynchronize(st));
  double mag, asym;
  std::memcpy(&mag, &hs[0], 8);
  std::memcpy(&asym, &hs[1], 8);
  if (asym > 1e-9 * std::max(mag, 1.0)) fail(CS_SHAPE_ERROR, "symmetric_eig: matrix is not symmetric to 1e-9");
  }
  // eigenvalues only: own tridiagonalisation + bisection (m <= 2048)
  if (!vectors && tridiag_eigvals(ctx, G, m, w)) return;
  if (V != G) CSB_CUDA(cudaMemcpyAsync(V, G, m * m * sizeof(double), cudaMemcpyDeviceToDevice, st));
  const CusolverApi& api = cusolver_api();
  if (!ctx->solver) solver_check(api.create(&ctx->solver), "cusolverDnCreate");
  solver_check(api.set_stream(ctx->solver, st), "SetStream");
  int lwork = 0;
  const cusolverEigMode_t mode = vectors ? CUSOLVER_EIG_MODE_VECTOR : CUSOLVER_EIG_MODE_NOVECTOR;
  solver_check(api.syevd_buffer(ctx->solver, mode, CUBLAS_FILL_MODE_LOWER,
                                static_cast<int>(m), V, static_cast<int>(m), w, &lwork),
               "Dsyevd_bufferSize");
  TmpBuf<double> work(static_cast<size_t>(lwork) + 1);
  TmpBuf<int> info(1);
  solver_check(api.syevd(ctx->solver, mode, CUBLAS_FILL_MODE_LOWER,
                         static_cast<int>(m), V, static_cast<int>(m), w, work.get(), lwork, info.get()),
               "Dsyevd");
  int hinfo = 0;
  CSB_CUDA(cudaMemcpyAsync(&hinfo, info.get(), sizeof hinfo, cudaMemcpyDeviceToHost, st));
  CSB_CUDA(cudaStreamSynchronize(st));
  if (hinfo != 0) fail(CS_EIG_FAILURE, "symmetric_eig: eigensolver did not converge");
}

// the context's cuBLAS handle on its stream; false when cuBLAS is absent
bool cublas_handle(cs_ctx* ctx) {
  const CublasApi& bl = cublas_api();
  if (!bl.lib) return false;
  if (!ctx->blas && bl.create(&ctx->blas) != CUBLAS_STATUS_SUCCESS) {
    ctx->blas = nullptr;
    return false;
  }
  return bl.set_stream(ctx->blas, ctx->stream) == CUBLAS_STATUS_SUCCESS;
}

// G^-1 = L^-T L^-1 from the Cholesky factor L (lower, ld m) with DGEMMs on
// the FP64 tensor-core path instead of potrs(L, I)'s two m-RHS TRSMs (2 m^3
// flops at TRSM rates; 11.7 ms at m = 4000).  Both halves recurse on a 2 x 2
// block split at multiples of 128:
//   X = L^-1:  X11 = L11^-1, X22 = L22^-1, X21 = -X22 (L21 X11)
//   C = X^T X: C11 = X11^T X11 + X21^T X21, C21 = X22^T X21, C22 = X22^T X22
// ~2/3 m^3 flops each.  128-blocks: tri_inv_diag_kernel / one DGEMM.  Only
// C's lower triangle is meaningful (the caller symmetrises).  Returns false
// if cuBLAS is unavailable or a call fails (caller falls back to potrs).
bool tri_inverse_product(cs_ctx* ctx, const double* L, int64_t m, double* out) {
  if (!cublas_handle(ctx)) return false;
  cudaStream_t st = ctx->stream;
  const CublasApi& bl = cublas_api();
  const int ld = static_cast<int>(m);
  TmpBuf<double> X(static_cast<size_t>(m) * m);
  CSB_CUDA(cudaMemsetAsync(X.get(), 0, m * m * sizeof(double), st));
  CSB_CUDA(cudaMemsetAsync(out, 0, m * m * sizeof(double), st));
  const size_t smem = sizeof(double) * kTriInvB * (kTriInvB + 1);
  CSB_CUDA(cudaFuncSetAttribute(tri_inv_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
  tri_inv_diag_kernel<<<ceil_div(m, kTriInvB), kTriInvB, smem, st>>>(L, m, X.get());
  CSB_LAUNCH_CHECK();
  bool ok = true;
  const double one = 1.0, zero = 0.0, mone = -1.0;
  auto gemm = [&](cublasOperation_t ta, int r, int c, int k, const double* alpha, const double* A, int lda,
                  const double* B, int ldb, const double* beta, double* C, int ldc) {
    if (ok && bl.dgemm(ctx->blas, ta, CUBLAS_OP_N, r, c, k, alpha, A, lda, B, ldb, beta, C, ldc) !=
                  CUBLAS_STATUS_SUCCESS)
      ok = false;
  };
  // Split tree: node (r0, b) -> (r0, b1), (r0 + b1, b2), b1 = b/2 rounded up
  // to a multiple of 128.  Nodes of one depth are independent; both passes
  // run deepest level first (children complete before their parent reads X11
  // / X22, or adds into C11 over the children's beta = 0 writes), and each
  // level's nodes of equal (b1, b2) go to cuBLAS as one batched DGEMM.
  struct Node {
    int64_t r0, b1, b2;
  };
  std::vector<std::vector<Node>> levels;
  std::function<void(int64_t, int64_t, size_t)> build = [&](int64_t r0, int64_t b, size_t d) {
    if (b <= kTriInvB) return;
    const int64_t b1 = ((b / 2 + kTriInvB - 1) / kTriInvB) * kTriInvB, b2 = b - b1;
    if (levels.size() <= d) levels.resize(d + 1);
    levels[d].push_back({r0, b1, b2});
    build(r0, b1, d + 1);
    build(r0 + b1, b2, d + 1);
  };
  build(0, m, 0);
  size_t tmp_el = 0, max_batch = 1;
  for (const auto& lv : levels) {
    size_t el = 0;
    for (const Node& q : lv) el += static_cast<size_t>(q.b1 * q.b2);
    tmp_el = std::max(tmp_el, el);
    max_batch = std::max(max_batch, lv.size());
  }
  TmpBuf<double> T(tmp_el + 1);
  TmpBuf<const double*> ptrs(6 * max_batch);
  auto at = [&](const double* A, int64_t i, int64_t j) { return A + i + j * m; };
  // one batched DGEMM per (b1, b2) group of a level: C_i = alpha op(A_i) B_i + beta C_i
  auto batched = [&](cublasOperation_t ta, int r, int c, int k, const double* alpha,
                     const std::vector<const double*>& A, int lda, const std::vector<const double*>& B, int ldb,
                     const double* beta, const std::vector<const double*>& C, int ldc) {
    if (!ok) return;
    if (A.size() == 1) {
      gemm(ta, r, c, k, alpha, A[0], lda, B[0], ldb, beta, const_cast<double*>(C[0]), ldc);
      return;
    }
    const size_t nb = A.size();
    std::vector<const double*> h(3 * nb);
    std::copy(A.begin(), A.end(), h.begin());
    std::copy(B.begin(), B.end(), h.begin() + nb);
    std::copy(C.begin(), C.end(), h.begin() + 2 * nb);
    CSB_CUDA(cudaMemcpyAsync(ptrs.get(), h.data(), 3 * nb * sizeof(double*), cudaMemcpyHostToDevice, st));
    // the pointer table is reused by the next call: keep the copy ordered
    // before it (pageable H2D returns once staged; the stream orders the rest)
    if (bl.dgemm_batched(ctx->blas, ta, CUBLAS_OP_N, r, c, k, alpha, ptrs.get(), lda, ptrs.get() + nb, ldb, beta,
                         const_cast<double* const*>(ptrs.get() + 2 * nb), ldc,
                         static_cast<int>(nb)) != CUBLAS_STATUS_SUCCESS)
      ok = false;
  };
  auto groups = [](const std::vector<Node>& lv) {
    std::map<std::pair<int64_t, int64_t>, std::vector<Node>> g;
    for (const Node& q : lv) g[{q.b1, q.b2}].push_back(q);
    return g;
  };
  // X = L^-1: T_i = L21 X11, X21 = -X22 T_i
  for (size_t d = levels.size(); d-- > 0;) {
    size_t toff = 0;
    for (const auto& kv : groups(levels[d])) {
      const int64_t b1 = kv.first.first, b2 = kv.first.second;
      std::vector<const double*> A1, B1, C1, A2, C2;
      for (const Node& q : kv.second) {
        const int64_t r1 = q.r0 + b1;
        A1.push_back(at(L, r1, q.r0));
        B1.push_back(at(X.get(), q.r0, q.r0));
        C1.push_back(T.get() + toff);
        A2.push_back(at(X.get(), r1, r1));
        C2.push_back(at(X.get(), r1, q.r0));
        toff += static_cast<size_t>(b1 * b2);
      }
      batched(CUBLAS_OP_N, b2, b1, b1, &one, A1, ld, B1, ld, &zero, C1, static_cast<int>(b2));
      batched(CUBLAS_OP_N, b2, b1, b2, &mone, A2, ld, C1, static_cast<int>(b2), &zero, C2, ld);
    }
  }
  // C's 128-aligned diagonal blocks X_bb^T X_bb first (one strided-batched
  // DGEMM + the remainder block): the levels only add into them
  const int64_t full = m / kTriInvB, rem = m - full * kTriInvB;
  const long long stride = static_cast<long long>(kTriInvB) * (m + 1);
  if (full > 0 && ok &&
      bl.dgemm_strided(ctx->blas, CUBLAS_OP_T, CUBLAS_OP_N, kTriInvB, kTriInvB, kTriInvB, &one, X.get(), ld, stride,
                       X.get(), ld, stride, &zero, out, ld, stride, static_cast<int>(full)) != CUBLAS_STATUS_SUCCESS)
    ok = false;
  if (rem > 0) {
    const int64_t r0 = full * kTriInvB;
    gemm(CUBLAS_OP_T, rem, rem, rem, &one, at(X.get(), r0, r0), ld, at(X.get(), r0, r0), ld, &zero,
         out + r0 + r0 * m, ld);
  }
  // C = X^T X: C11 += X21^T X21, C21 = X22^T X21
  for (size_t d = levels.size(); d-- > 0;) {
    for (const auto& kv : groups(levels[d])) {
      const int64_t b1 = kv.first.first, b2 = kv.first.second;
      std::vector<const double*> X21, X22, C11, C21;
      for (const Node& q : kv.second) {
        const int64_t r1 = q.r0 + b1;
        X21.push_back(at(X.get(), r1, q.r0));
        X22.push_back(at(X.get(), r1, r1));
        C11.push_back(at(out, q.r0, q.r0));
        C21.push_back(at(out, r1, q.r0));
      }
      batched(CUBLAS_OP_T, b1, b1, b2, &one, X21, ld, X21, ld, &one, C11, ld);
      batched(CUBLAS_OP_T, b2, b1, b2, &one, X22, ld, X21, ld, &zero, C21, ld);
    }
  }
  return ok;
}

// Gram matrix of a model's normalised memory vectors (mset.cpp:151-152).
// FP64-precision models: `sim_exact`, the reference's loop order bit for bit.
// FP32-precision models (tolerance contract): the DMMA Gram of train_f64.cu
// -- D_norm^T D_norm on the FP64 tensor pipe (lower triangle, mirrored) with
// the kernel map of ||d_i||^2 + ||d_j||^2 - 2 S_ij, the exact unit diagonal
// and the direct-difference recompute of cancellation-prone entries fused in
// the epilogue (duplicate / near-duplicate memory vectors get the
// reference's values, so the rank decision matches the exact Gram).
// Deterministic, so the lazy eigen_spectrum re-forms the identical matrix.
// CSB_GRAM_EXACT=1 forces the exact kernel for every model.
void form_gram(cs_ctx* ctx, const cs_model* M, double* gram) {
  cudaStream_t st = ctx->stream;
  const int64_t n = M->n, m = M->m;
  const char* env = std::getenv("CSB_GRAM_EXACT");
  const bool exact = (env && env[0] == '1') || M->precision != CS_PRECISION_FP32;
  if (!exact) {
    dmma_gram(st, M->Dn.get(), n, m, M->kind, M->h, gram);
    return;
  }
  launch_sim_exact(st, M->Dn.get(), n, M->Dn.get(), n, n, m, m, M->kind, M->h, gram, m);
}

// Full-rank fast path of the pseudo-inverse: when every eigenvalue passes the
// reference cutoff (rank == m), G+ = V L^-1 V^T = G^-1 exactly, computed here
// by Cholesky factorisation + inverse (~m^3 flops instead of syevd's vector
// phase and the W W^T product).  Default: the own recursive blocked
// factorisation on the DMMA tensor pipe (train_f64.cu).  CSB_POTRI=1|2|3
// select the round-1 cuSOLVER routes (potri / potrs / potrf + cuBLAS
// recursion) for A/B runs.  Returns false when G is not numerically positive
// definite, in which case the caller takes the eigenvector path.
bool cholesky_inverse(cs_ctx* ctx, const double* G, int64_t m, double* out) {
  cudaStream_t st = ctx->stream;
  const int mi = static_cast<int>(m);
  const char* env = std::getenv("CSB_POTRI");
  if (!(env && (env[0] == '1' || env[0] == '2' || env[0] == '3'))) return dmma_chol_inverse(st, G, m, out);
  const CusolverApi& api = cusolver_api();
  if (!ctx->solver) solver_check(api.create(&ctx->solver), "cusolverDnCreate");
  solver_check(api.set_stream(ctx->solver, st), "SetStream");
  if (env[0] == '1') {
    // factor + potri (triangular inverse and L^-T L^-1 in place)
    CSB_CUDA(cudaMemcpyAsync(out, G, m * m * sizeof(double), cudaMemcpyDeviceToDevice, st));
    int l1 = 0, l2 = 0;
    solver_check(api.potrf_buffer(ctx->solver, CUBLAS_FILL_MODE_LOWER, mi, out, mi, &l1), "Dpotrf_bufferSize");
    solver_check(api.potri_buffer(ctx->solver, CUBLAS_FILL_MODE_LOWER, mi, out, mi, &l2), "Dpotri_bufferSize");
    TmpBuf<double> work(static_cast<size_t>(std::max(l1, l2)) + 1);
    TmpBuf<int> info(2);
    solver_check(api.potrf(ctx->solver, CUBLAS_FILL_MODE_LOWER, mi, out, mi, work.get(), l1, info.get()),
                 "Dpotrf");
    solver_check(api.potri(ctx->solver, CUBLAS_FILL_MODE_LOWER, mi, out, mi, work.get(), l2, info.get() + 1),
                 "Dpotri");
    int h[2] = {0, 0};
    CSB_CUDA(cudaMemcpyAsync(h, info.get(), sizeof h, cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaStreamSynchronize(st));
    if (h[0] != 0 || h[1] != 0) return false;
  } else if (env && (env[0] == '2' || env[0] == '3')) {
    // factor, then G^-1 = L^-T L^-1 by the blocked cuBLAS DGEMM recursion
    // (CSB_POTRI=3), or potrs(L, I) (CSB_POTRI=2) -- the round-1 routes, kept
    // for A/B runs
    TmpBuf<double> L(static_cast<size_t>(m) * m);
    CSB_CUDA(cudaMemcpyAsync(L.get(), G, m * m * sizeof(double), cudaMemcpyDeviceToDevice, st));
    int l1 = 0;
    solver_check(api.potrf_buffer(ctx->solver, CUBLAS_FILL_MODE_LOWER, mi, L.get(), mi, &l1), "Dpotrf_bufferSize");
    TmpBuf<double> work(static_cast<size_t>(l1) + 1);
    TmpBuf<int> info(2);
    CSB_CUDA(cudaMemsetAsync(info.get(), 0, 2 * sizeof(int), st));  // info[1] stays 0 on the blocked route
    solver_check(api.potrf(ctx->solver, CUBLAS_FILL_MODE_LOWER, mi, L.get(), mi, work.get(), l1, info.get()),
                 "Dpotrf");
    int hf = 0;
    CSB_CUDA(cudaMemcpyAsync(&hf, info.get(), sizeof hf, cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaStreamSynchronize(st));
    if (hf != 0) return false;  // not numerically positive definite
    const bool blocked = env[0] == '3' && tri_inverse_product(ctx, L.get(), m, out);
    if (!blocked) {
      set_identity_kernel<<<grid_for(m * m), 256, 0, st>>>(out, m);
      CSB_LAUNCH_CHECK();
      solver_check(api.potrs(ctx->solver, CUBLAS_FILL_MODE_LOWER, mi, mi, L.get(), mi, out, mi, info.get() + 1),
                   "Dpotrs");
    }
    int h[2] = {0, 0};
    CSB_CUDA(cudaMemcpyAsync(h, info.get(), sizeof h, cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaStreamSynchronize(st));
    if (h[0] != 0 || h[1] != 0) return false;
  }
  symmetrize_lower_kernel<<<grid_for(m * m), 256, 0, st>>>(out, m);
  CSB_LAUNCH_CHECK();
  return true;
}

// ------------------------------------------------------ FP32 operand packing
void choose_tc_shape(cs_model* M) {
  M->K1 = static_cast<int>((M->n + 2 + 15) / 16 * 16);  // + the ||d||^2, ||x||^2 columns; K = 16 per MMA
  // GEMM2's N: tcgen05 kind::f16 with M = 128 takes N in steps of 8, and
  // the MMA time is proportional to N (n = 100: 104 instead of 112 columns)
  // (measured: C2 0.140 -> 0.137 ms, n=100/m=4000 -3%)
#ifndef CSB_N2_ALIGN
#define CSB_N2_ALIGN 8
#endif
  M->N2 = static_cast<int>((M->n + CSB_N2_ALIGN - 1) / CSB_N2_ALIGN * CSB_N2_ALIGN);
  M->MT = 0;
  // (memory tile MT, TMEM buffers NB) in order of preference.  A TS-form
  // tcgen05.mma costs >= ~30 cycles whatever N (tools/mma_probe: N=16 and 32
  // both 29.6 cycles, N=64 hits the 32-cycle M*N/256 floor), so GEMM1 tiles
  // narrower than 64 waste the tensor pipe; double buffering (NB = 2)
  // decouples the epilogue.  Then the deepest operand ring (<= 4) that fits.
  // (MT, NB, SB) in order of preference.  NB = 2 decouples GEMM1 from the
  // similarity epilogue; measured (tools/estimate_sweep.py, timeline.py):
  // (64,2,1) beats (64,1,1) at n = 64, but at n = 100 the only double-ACC
  // shape that fits, (48,2,1), loses to (64,1,1) by 30% -- the narrower GEMM1
  // (N = 48 runs at the ~30-cycle MMA floor) and the serial S buffer cost more
  // than the GEMM1 wait it removes.
  int pref[10][3] = {{128, 2, 2}, {64, 2, 2}, {64, 2, 1}, {128, 1, 1}, {64, 1, 1},
                     {48, 2, 1},  {32, 2, 2}, {32, 2, 1}, {32, 1, 1}, {16, 2, 2}};
  int npref = 10;
  if (const char* e = std::getenv("CSB_TC_SHAPE")) {  // development override "MT,NB,SB"
    int a = 0, b = 0, c = 0;
    if (std::sscanf(e, "%d,%d,%d", &a, &b, &c) == 3) {
      pref[0][0] = a;
      pref[0][1] = b;
      pref[0][2] = c;
      npref = 1;
    }
  }
  for (int i = 0; i < npref; ++i) {
    const int MT = pref[i][0], NB = pref[i][1], SB = pref[i][2];
    const int cols = tc_tmem_cols(M->N2, M->K1, MT, NB, SB);
    const size_t stage = static_cast<size_t>(2) * MT * M->K1 * 2 + static_cast<size_t>(2) * M->N2 * MT * 2;
    const size_t budget = 227 * 1024 - tc_aux_bytes(M->K1);
    const int stages = static_cast<int>(std::min<size_t>(kMaxStages, budget / stage));
    if (cols <= kTmemCols && stages >= 2) {
      M->MT = MT;
      M->NB = NB;
      M->SB = SB;
      M->n_stages = stages;
      break;
    }
  }
  M->tc = M->MT > 0;
  if (M->tc) M->m_tiles = static_cast<int>((M->m + M->MT - 1) / M->MT);
}

void pack_fp32_operands(cs_ctx* ctx, cs_model* M) {
  cudaStream_t st = ctx->stream;
  choose_tc_shape(M);
  const int n = static_cast<int>(M->n), m = static_cast<int>(M->m);
  int m_pad = 0;
  if (M->tc) {
    m_pad = M->m_tiles * M->MT;
  } else {
    // two-GEMM path: GEMM-A N = memory vectors, GEMM-B N = signals
    M->gemm = true;
    M->bnA = m >= 256 ? 256 : 128;
    M->ntA = (m + M->bnA - 1) / M->bnA;
    m_pad = M->ntA * M->bnA;
    M->kcA = (n + 1 + kGemmBK - 1) / kGemmBK;
    M->bnB = n > 128 ? 256 : 128;
    M->ntB = (n + M->bnB - 1) / M->bnB;
    M->kcB = m_pad / kGemmBK;
  }
  // ||d||^2, FP32 D_norm, scales and max |D_norm| first: they fix the FP16
  // operand scales (pack_tc.cuh)
  M->dd.resize(m_pad);
  M->dn32.resize(static_cast<size_t>(n) * m);
  M->inv_scale.resize(n);
  M->scale_f.resize(n);
  TmpBuf<unsigned int> absmax(1);
  CSB_CUDA(cudaMemsetAsync(absmax.get(), 0, sizeof(unsigned int), st));
  TmpBuf<double> dd64(m_pad);
  dn_sqnorm_kernel<<<ceil_div(static_cast<int64_t>(m_pad) * 32, 256), 256, 0, st>>>(M->Dn.get(), n, m, m_pad,
                                                                                   dd64.get());
  CSB_LAUNCH_CHECK();
  pack_aux_kernel<<<grid_for(std::max<int64_t>(m_pad, static_cast<int64_t>(n) * m)), 256, 0, st>>>(
      M->Dn.get(), dd64.get(), M->scale.get(), n, m, m_pad, M->dd.get(), M->dn32.get(), M->inv_scale.get(),
      M->scale_f.get(), absmax.get());
  CSB_LAUNCH_CHECK();
  std::vector<float> dd_host(m_pad);
  unsigned int absmax_bits = 0;
  CSB_CUDA(cudaMemcpyAsync(dd_host.data(), M->dd.get(), m_pad * sizeof(float), cudaMemcpyDeviceToHost, st));
  CSB_CUDA(cudaMemcpyAsync(&absmax_bits, absmax.get(), sizeof absmax_bits, cudaMemcpyDeviceToHost, st));
  CSB_CUDA(cudaStreamSynchronize(st));
  M->dd_max = 0.f;
  for (float v : dd_host) M->dd_max = std::max(M->dd_max, v);
  float dn_absmax;
  std::memcpy(&dn_absmax, &absmax_bits, 4);
  if (!(2.f * dn_absmax < kF16Safe)) {
    // -2 d would leave the FP16 split's range (a memory vector beyond 16384
    // standard deviations): this model surveils on the exact FP64 path
    M->tc = false;
    M->gemm = false;
    return;
  }
  // ||d||^2 column: scale 2^-k_aug keeps it below 2^14; x carries 2^k_aug
  int k_aug = 0;
  if (M->dd_max > 16384.f) {
    int ex;
    std::frexp(static_cast<double>(M->dd_max), &ex);
    k_aug = ex - 14;
  }
  const double aug_scale = std::ldexp(1.0, -k_aug);
  M->aug_x = static_cast<float>(std::ldexp(1.0, k_aug));
  // P = D_norm * G+  (n x m), FP64, once per model, and its
  // per-signal power-of-two scales
  TmpBuf<double> P(static_cast<size_t>(n) * m);
  // P carries no reference association (the reference forms W = G+ S, then
  // D W): the DMMA GEMM of train_f64.cu on the FP64 tensor pipe
  dmma_gemm(st, 0, n, m, m, 1.0, M->Dn.get(), n, M->pinv.get(), m, 0.0, P.get(), n);
  M->p_shift.resize(n);
  M->scale_out_d.resize(n);
  M->scale_out_f.resize(n);
  p_row_scale_kernel<<<ceil_div(n, 32), 1024, 0, st>>>(P.get(), M->scale.get(), n, m, M->p_shift.get(),
                                                         M->scale_out_d.get(), M->scale_out_f.get());
  CSB_LAUNCH_CHECK();
  // Similarity centring (two-GEMM path): GEMM-B accumulates P (S - s_c)
  // and the epilogue adds s_c P 1 back.  tcgen05's FP32 accumulation
  // truncates, and with P's cancellation (sum |P s| ~ 600 |P s| at C3) the
  // partial sums, not the products, set the error; centring S shrinks them.
  // s_c = the kernel at the typical squared distance of two memory vectors
  // (2 mean ||d||^2), rounded to 8 bits so that S - s_c is exact.
  {
    double mean_dd = 0.0;
    for (int i = 0; i < m; ++i) mean_dd += dd_host[i];
    mean_dd /= static_cast<double>(m);
    const double d2 = 2.0 * mean_dd;
    const double sk = M->kind == CS_KERNEL_GAUSSIAN ? std::exp(-d2 / (2.0 * M->h * M->h))
                                                    : 1.0 / (1.0 + std::sqrt(d2) / M->h);
    M->s_center = static_cast<float>(std::round(sk * 256.0) / 256.0);
    // the fused kernel (m <= a few thousand, K = m short) does not centre:
    // its error is ~1e-5 without, and the extra subtraction per pair cost 3%
    if (M->tc || std::getenv("CSB_NO_CENTER")) M->s_center = 0.f;
    M->add_d.resize(n);
    M->add_f.resize(n);
    p_center_add_kernel<<<ceil_div(static_cast<int64_t>(n) * 32, 256), 256, 0, st>>>(
        P.get(), M->scale.get(), n, m, static_cast<double>(M->s_center), M->add_d.get(), M->add_f.get());
    CSB_LAUNCH_CHECK();
  }
  if (M->tc) {
    M->dn_tiles.resize(static_cast<size_t>(M->m_tiles) * 2 * M->MT * M->K1);
    M->p_tiles.resize(static_cast<size_t>(M->m_tiles) * 2 * M->N2 * M->MT);
    pack_dn_tiles_kernel<<<grid_for(static_cast<int64_t>(M->m_tiles) * M->MT * M->K1), 256, 0, st>>>(
        M->Dn.get(), dd64.get(), n, m, M->MT, M->K1, M->m_tiles, aug_scale, M->dn_tiles.get());
    CSB_LAUNCH_CHECK();
    pack_p_tiles_kernel<<<grid_for(static_cast<int64_t>(M->m_tiles) * M->MT * M->N2), 256, 0, st>>>(
        P.get(), M->p_shift.get(), n, m, M->MT, M->N2, M->m_tiles, M->p_tiles.get());
    CSB_LAUNCH_CHECK();
  } else {
    const size_t a_el = static_cast<size_t>(M->ntA) * M->kcA * gemm_block_halves(M->bnA);
    const size_t b_el = static_cast<size_t>(M->ntB) * M->kcB * gemm_block_halves(M->bnB);
    M->dn_gemm.resize(a_el);
    M->p_gemm.resize(b_el);
    pack_dn_gemm_kernel<<<grid_for(static_cast<int64_t>(a_el / 2)), 256, 0, st>>>(
        M->Dn.get(), dd64.get(), n, m, M->bnA, M->ntA, M->kcA, aug_scale, M->dn_gemm.get());
    CSB_LAUNCH_CHECK();
    pack_p_gemm_kernel<<<grid_for(static_cast<int64_t>(b_el / 2)), 256, 0, st>>>(
        P.get(), M->p_shift.get(), n, m, M->bnB, M->ntB, M->kcB, M->p_gemm.get());
    CSB_LAUNCH_CHECK();
  }
}

// ----------------------------------------------------------------- train
// CSB_TRACE=1: synchronise and report the wall time of each train phase on
// stderr (diagnostics; off by default).
struct PhaseTrace {
  bool on = false;
  cudaStream_t st;
  std::chrono::steady_clock::time_point t0;
  explicit PhaseTrace(cudaStream_t s) : st(s) {
    const char* e = std::getenv("CSB_TRACE");
    on = e && e[0] == '1';
    t0 = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[csb] %-24s %9.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  }
};

cs_model* train_device(cs_ctx* ctx, const double* X, int64_t N, int64_t n, int64_t m, int kind,
                       double bandwidth, int precision) {
  PhaseTrace trace(ctx->stream);
  check_kind(kind);
  if (precision != CS_PRECISION_FP64 && precision != CS_PRECISION_FP32)
    fail(CS_CONFIG_ERROR, "unknown precision");
  cudaStream_t st = ctx->stream;
  std::unique_ptr<cs_model> M(new cs_model);
  M->device = ctx->device;
  M->n = n;
  M->m = m;
  M->kind = kind;
  M->precision = precision;
  TmpBuf<int64_t> picked;
  trace.mark("enter");
  select_device(ctx, X, N, n, m, picked, nullptr);  // mset.cpp:142 (indices land in ctx->pin)
  trace.mark("select_memory_vectors");
  M->h = resolve_h(bandwidth, n);                            // mset.cpp:143-144
  M->D.resize(n * m);
  gather_memory_kernel<<<grid_for(n * m), 256, 0, st>>>(X, N, n, picked.get(), m, M->D.get());
  CSB_LAUNCH_CHECK();
  M->scale.resize(n);                                        // mset.cpp:145
  scale_seq_kernel<<<ceil_div(n, 4), 128, 0, st>>>(X, N, n, M->scale.get());
  CSB_LAUNCH_CHECK();
  M->Dn.resize(n * m);                                       // mset.cpp:147-149
  div_rows_kernel<<<grid_for(n * m), 256, 0, st>>>(M->D.get(), M->scale.get(), n, m, M->Dn.get());
  CSB_LAUNCH_CHECK();
  TmpBuf<double> gram(m * m);                                // mset.cpp:151-152
  trace.mark("scale + normalise");
  form_gram(ctx, M.get(), gram.get());
  trace.mark("gram");
  // Pseudo-inverse (mset.cpp:153-170).  Fast path: Cholesky inverse of G,
  // certified full rank -- every eigenvalue of the SPD matrix G satisfies
  // lambda_min / lambda_max >= 1 / (||G||_1 ||G^-1||_1), so a 1-norm
  // condition number below kCertifiedCond (half the reference's 1e10
  // cutoff ratio, margin for rounding) proves rank == m, and then
  // G+ = V L^-1 V^T = G^-1.  Otherwise the reference's eigen route.
  const char* force = std::getenv("CSB_TRAIN_EIGVEC");
  const bool vec_path = force && force[0] == '1';
  const char* eager_env = std::getenv("CSB_EAGER_SPECTRUM");
  const bool eager = eager_env && eager_env[0] == '1';
  M->spectrum.resize(m);
  M->spectrum_host.resize(m);
  M->pinv.resize(m * m);
  bool done = false;
  int64_t rank = 0;
  // Eager spectrum with the own eigenvalue solver (m <= kTriMaxM, no host
  // round trip inside): it runs on a side stream concurrently with the
  // certified Cholesky inverse, which decides rank == m on its own; the
  // spectrum is joined before train returns (the reference's contract,
  // mset.cpp:153-154).  If the certification fails, the eigenvalues decide
  // the rank as below.
  const bool eig_async = eager && !vec_path && m <= kTriMaxM;
  TmpBuf<double> V;  // syevd works in place on a copy of G
  cudaEvent_t eig_done = nullptr;
  if (eig_async) {
    V.resize(m * m);  // only touched if the own solver falls back to syevd
    cudaStream_t side = ctx->aux[0];
    cudaEvent_t gram_ready;
    CSB_CUDA(cudaEventCreateWithFlags(&gram_ready, cudaEventDisableTiming));
    CSB_CUDA(cudaEventCreateWithFlags(&eig_done, cudaEventDisableTiming));
    CSB_CUDA(cudaEventRecord(gram_ready, st));
    CSB_CUDA(cudaStreamWaitEvent(side, gram_ready, 0));
    cudaEventDestroy(gram_ready);
    {
      struct Swap {  // ctx->stream is the side stream for this call only
        cs_ctx* c;
        cudaStream_t keep;
        ~Swap() { c->stream = keep; }
      } swap{ctx, st};
      ctx->stream = side;
      StreamScope scope(side);
      eig_device(ctx, gram.get(), m, M->spectrum.get(), V.get(), false, false);
    }
    CSB_CUDA(cudaEventRecord(eig_done, side));
  }
  if (!vec_path && (!eager || eig_async) && cholesky_inverse(ctx, gram.get(), m, M->pinv.get())) {
    TmpBuf<unsigned long long> nrm(2);
    CSB_CUDA(cudaMemsetAsync(nrm.get(), 0, 2 * sizeof(unsigned long long), st));
    const int nb = static_cast<int>(std::min<int64_t>(m, 4 * 148));
    norm1_kernel<<<nb, 256, 0, st>>>(gram.get(), m, nrm.get());
    norm1_kernel<<<nb, 256, 0, st>>>(M->pinv.get(), m, nrm.get() + 1);
    CSB_LAUNCH_CHECK();
    unsigned long long hb[2];
    CSB_CUDA(cudaMemcpyAsync(hb, nrm.get(), sizeof hb, cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaStreamSynchronize(st));
    double g1, gi1;
    std::memcpy(&g1, &hb[0], 8);
    std::memcpy(&gi1, &hb[1], 8);
    constexpr double kCertifiedCond = 5e9;
    if (std::isfinite(g1 * gi1) && g1 * gi1 < kCertifiedCond) {
      rank = m;
      done = true;
      M->spectrum_ready = eig_async;  // eager: computed beside, joined below
    }
    trace.mark("pinv (certified Cholesky)");
  }
  if (eig_async && !done) {  // the eigenvalues decide the rank: join now
    CSB_CUDA(cudaStreamWaitEvent(st, eig_done, 0));
    cudaEventDestroy(eig_done);
    eig_done = nullptr;
  }
  if (!done) {
    // eigenvalues first: they decide the rank exactly as the reference does
    V.resize(m * m);
    if (!eig_async) eig_device(ctx, gram.get(), m, M->spectrum.get(), V.get(), vec_path, false);
    trace.mark(vec_path ? "symmetric_eig (syevd)" : "eigenvalues (own solver up to m = 2048, syevd N above)");
    CSB_CUDA(cudaMemcpyAsync(M->spectrum_host.data(), M->spectrum.get(), m * sizeof(double),
                             cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaStreamSynchronize(st));
    const double cutoff = 1e-10 * M->spectrum_host[m - 1];  // mset.cpp:156-163
    for (int64_t i = 0; i < m; ++i)
      if (M->spectrum_host[i] > cutoff) ++rank;
    if (rank == 0) fail(CS_DEGENERATE_MODEL, "train: all Gram eigenvalues below cutoff");
    if (rank == m && !vec_path) {
      done = cholesky_inverse(ctx, gram.get(), m, M->pinv.get());
      trace.mark("pinv (Cholesky inverse)");
    }
  }
  M->rank = rank;
  if (!done) {
    if (!vec_path) {
      eig_device(ctx, gram.get(), m, M->spectrum.get(), V.get(), true, false);
      trace.mark("symmetric_eig (syevd V)");
      CSB_CUDA(cudaMemcpyAsync(M->spectrum_host.data(), M->spectrum.get(), m * sizeof(double),
                               cudaMemcpyDeviceToHost, st));
      CSB_CUDA(cudaStreamSynchronize(st));
      const double c2 = 1e-10 * M->spectrum_host[m - 1];
      rank = 0;
      for (int64_t i = 0; i < m; ++i)
        if (M->spectrum_host[i] > c2) ++rank;
      if (rank == 0) fail(CS_DEGENERATE_MODEL, "train: all Gram eigenvalues below cutoff");
      M->rank = rank;
    }
    TmpBuf<double> W(m * rank);                              // mset.cpp:165-170
    whiten_kernel<<<grid_for(m * rank), 256, 0, st>>>(V.get(), M->spectrum.get(), m, rank, W.get());
    CSB_LAUNCH_CHECK();
    launch_gemm_exact<false, true>(st, W.get(), m, W.get(), m, m, rank, m, M->pinv.get(), m);
    trace.mark("pinv (W W^T)");
  }
  if (precision == CS_PRECISION_FP32) pack_fp32_operands(ctx, M.get());
  if (eig_done) {  // certified while the spectrum was computed beside: join it last
    CSB_CUDA(cudaStreamWaitEvent(st, eig_done, 0));
    cudaEventDestroy(eig_done);
    CSB_CUDA(cudaMemcpyAsync(M->spectrum_host.data(), M->spectrum.get(), m * sizeof(double),
                             cudaMemcpyDeviceToHost, st));
  }
  CSB_CUDA(cudaStreamSynchronize(st));
  trace.mark("fp32 operand packing");
  M->source_indices.resize(m);  // copied into ctx->pin by select_device, complete now
  std::memcpy(M->source_indices.data(), ctx->pin, m * sizeof(int64_t));
  return M.release();
}

// ------------------------------------------------------------- estimate
void check_model_shape(const cs_model* M, int64_t n) {
  if (n != M->n) {
    char buf[200];
    std::snprintf(buf, sizeof buf,
                  "estimate: observation signal count %lld does not match model signal count %lld",
                  static_cast<long long>(n), static_cast<long long>(M->n));
    fail(CS_SHAPE_ERROR, buf);
  }
  if (M->rank < 1) fail(CS_DEGENERATE_MODEL, "estimate: model rank is 0");
}

// FP64, reference association, exact order (mset.cpp:186-197).  Device
// buffers; processes observations in chunks of the S/W workspace.
void estimate_fp64_device(cs_ctx* ctx, cudaStream_t st, const cs_model* M, const double* obs,
                          int64_t N, int64_t ld, double* est, double* resid) {
  const int64_t n = M->n, m = M->m;
  // Chunk of Nc observations: four workspaces of (2n + 2m) x Nc doubles,
  // at most 2^28 doubles per m x Nc buffer and half the free device memory;
  // halved on an allocation failure.  Every kernel of this path is exact per
  // observation, so the chunking never changes a bit of the result.
  const int64_t budget = (int64_t{1} << 28);
  int64_t Nc = std::max<int64_t>(1, std::min<int64_t>(N, budget / std::max<int64_t>(m, 1)));
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
    const int64_t have = static_cast<int64_t>(std::min(ctx->wsB.count, ctx->wsC.count) / std::max<int64_t>(m, 1));
    const int64_t cap = static_cast<int64_t>(free_b / 2 / (8 * static_cast<size_t>(2 * n + 2 * m)));
    Nc = std::max<int64_t>(1, std::min(Nc, std::max(cap, have)));
  } else {
    cudaGetLastError();
  }
  for (;;) {
    try {
      ctx->wsA.resize(n * Nc);
      ctx->wsB.resize(m * Nc);
      ctx->wsC.resize(m * Nc);
      ctx->wsD.resize(n * Nc);
      break;
    } catch (const Failure&) {
      cudaGetLastError();
      if (Nc == 1) throw;
      Nc = (Nc + 1) / 2;
    }
  }
  for (int64_t t0 = 0; t0 < N; t0 += Nc) {
    const int64_t nc = std::min(Nc, N - t0);
    dim3 tg(ceil_div(nc, 32), ceil_div(n, 32)), tb(32, 8);
    transpose_div_kernel<<<tg, tb, 0, st>>>(obs, ld, t0, nc, n, M->scale.get(), ctx->wsA.get());
    CSB_LAUNCH_CHECK();
    launch_sim_exact(st, M->Dn.get(), n, ctx->wsA.get(), n, n, m, nc, M->kind, M->h, ctx->wsB.get(), m);
    launch_gemm_exact<false, false>(st, M->pinv.get(), m, ctx->wsB.get(), m, m, m, nc, ctx->wsC.get(), m);
    launch_gemm_exact<false, false>(st, M->Dn.get(), n, ctx->wsC.get(), m, n, m, nc, ctx->wsD.get(), n);
    finish_estimate_kernel<<<tg, tb, 0, st>>>(ctx->wsD.get(), nc, n, M->scale.get(), obs, ld, t0,
                                              est, resid);
    CSB_LAUNCH_CHECK();
  }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// libcuda link dependency)
PFN_cuTensorMapEncodeTiled_v12000 out_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

// N x n column-major FP32 output (leading dimension ld) as a 2D tensor map
// whose box is one 128-observation tile of all n signals
bool encode_out_map(CUtensorMap* m, const void* ptr, int64_t N, int n, int64_t ld) {
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(N), static_cast<cuuint64_t>(n)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kObsTile), static_cast<cuuint32_t>(n)};
  const cuuint32_t es[2] = {1, 1};
  return out_map_encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename IO>
void launch_tc(cs_ctx* ctx, cudaStream_t st, const cs_model* M, const IO* obs, int64_t N,
               int64_t ld, IO* est, IO* resid) {
  if (N == 0) return;
  TcParams p{};
  p.obs = obs;
  p.N = N;
  p.ld = ld;
  p.n = static_cast<int>(M->n);
  p.K1 = M->K1;
  p.N2 = M->N2;
  p.m = static_cast<int>(M->m);
  p.m_tiles = M->m_tiles;
  p.dn_tiles = M->dn_tiles.get();
  p.p_tiles = M->p_tiles.get();
  p.dd = M->dd.get();
  p.dn32 = M->dn32.get();
  p.inv_scale = M->inv_scale.get();
  p.scale_f = M->scale_out_f.get();
  p.scale_d = M->scale_out_d.get();
  p.norm_d = M->scale.get();
  p.aug_x = M->aug_x;
  p.kind = M->kind;
  p.inv_h = static_cast<float>(1.0 / M->h);
  p.g_coef = static_cast<float>(1.4426950408889634 / (2.0 * M->h * M->h));
  p.tau = 1.0f / 128.0f;
  p.dd_max = M->dd_max;
  p.est = est;
  p.resid = resid;
  p.dn_stage_bytes = static_cast<uint32_t>(2 * M->MT * M->K1 * 2);  // FP16 hi | lo
  p.p_stage_bytes = static_cast<uint32_t>(2 * M->N2 * M->MT * 2);
  p.n_stages = M->n_stages;
  size_t smem = M->n_stages * (static_cast<size_t>(p.dn_stage_bytes) + p.p_stage_bytes) + tc_aux_bytes(p.K1);
  // staged tile edge: FP32 I/O, TMA-compatible input and outputs (16-byte
  // aligned, leading dimension a multiple of 4) and room for [2][n][128]
  // FP32 next to an operand ring of >= 2 stages
  p.staged = 0;
  if constexpr (sizeof(IO) == 4) {
    const size_t stage = static_cast<size_t>(p.dn_stage_bytes) + p.p_stage_bytes;
    const size_t out_bytes = static_cast<size_t>(2) * M->n * kObsTile * 4;
    const size_t budget = 227 * 1024;
    const bool aligned = (ld % 4 == 0) && (reinterpret_cast<uintptr_t>(est) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(resid) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(obs) % 16 == 0) && (est || resid);
    const char* env = std::getenv("CSB_STAGED_READOUT");
    const bool allow = !(env && env[0] == '0');
    if (allow && aligned && M->n <= 256 && tc_aux_bytes(p.K1) + out_bytes + 128 + 2 * stage <= budget &&
        out_map_encoder() != nullptr) {
      const int ns = static_cast<int>(std::min<size_t>(
          M->n_stages, (budget - tc_aux_bytes(p.K1) - out_bytes - 128) / stage));
      p.n_stages = ns;
      p.stage_out_off = static_cast<uint32_t>((ns * stage + tc_aux_bytes(p.K1) + 127) / 128 * 128);
      smem = p.stage_out_off + out_bytes;
      bool ok = encode_out_map(&p.tmap_obs, obs, N, static_cast<int>(M->n), ld);
      if (est) ok = ok && encode_out_map(&p.tmap_est, est, N, static_cast<int>(M->n), ld);
      if (resid) ok = ok && encode_out_map(&p.tmap_res, resid, N, static_cast<int>(M->n), ld);
      if (ok) {
        p.staged = 1;
        // split tile edge: measured 3-8% faster for short memory loops
        // (n=20: T=2, n=64: T=8) and 1% slower at C2 (T=16)
        p.split_edge = M->m_tiles <= 12 ? 1 : 0;
        if (const char* e = std::getenv("CSB_SPLIT_EDGE")) p.split_edge = e[0] == '1';
      } else {
        p.n_stages = M->n_stages;
        smem = M->n_stages * stage + tc_aux_bytes(p.K1);
      }
    }
  }
  const int tiles = static_cast<int>((N + kObsTile - 1) / kObsTile);
  const int grid = std::min(tiles, ctx->sm_count);
#ifdef CSB_TIMELINE
  TmpBuf<unsigned long long> tl(static_cast<size_t>(5) * kTlCap * 2);
  CSB_CUDA(cudaMemsetAsync(tl.get(), 0, 5 * kTlCap * 2 * 8, st));
  p.timeline = tl.get();
#endif
  auto go = [&](auto kernel) {
    CSB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    // CSB_CLUSTER=2|4: clusters of CTAs share the operand stream by multicast
    // (estimate_tc.cuh); the persistent grid is sized to the clusters that
    // fit at once.  Off by default: measured no faster at C2 (the operand
    // stream from L2 is not what bounds the step).
    int cl = 1;
    if (const char* e = std::getenv("CSB_CLUSTER")) cl = std::max(1, std::atoi(e));
    int g = grid;
    if (cl > 1) {
      static std::mutex mu;
      static std::map<std::tuple<const void*, size_t, int>, int> fit;  // max active clusters
      std::lock_guard<std::mutex> lock(mu);
      const auto key = std::make_tuple(reinterpret_cast<const void*>(kernel), smem, cl);
      auto it = fit.find(key);
      if (it == fit.end()) {
        cudaLaunchConfig_t q{};
        q.gridDim = dim3(static_cast<unsigned>(ctx->sm_count / cl * cl));
        q.blockDim = dim3(tc_threads(M->NB, M->SB));
        q.dynamicSmemBytes = smem;
        cudaLaunchAttribute a{};
        a.id = cudaLaunchAttributeClusterDimension;
        a.val.clusterDim.x = cl;
        a.val.clusterDim.y = 1;
        a.val.clusterDim.z = 1;
        q.attrs = &a;
        q.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, kernel, &q) != cudaSuccess) {
          cudaGetLastError();
          n = 0;
        }
        it = fit.emplace(key, n).first;
      }
      const int max_ctas = it->second * cl;
      g = (grid + cl - 1) / cl * cl;
      if (max_ctas < cl) {
        cl = 1;
        g = grid;
      } else if (g > max_ctas) {
        g = max_ctas;
      }
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(g));
    cfg.blockDim = dim3(tc_threads(M->NB, M->SB));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = cl;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = cl > 1 ? 1 : 0;
    CSB_CUDA(cudaLaunchKernelEx(&cfg, kernel, p));
    CSB_LAUNCH_CHECK();
#ifdef CSB_TIMELINE
    std::vector<unsigned long long> h(static_cast<size_t>(5) * kTlCap * 2);
    CSB_CUDA(cudaMemcpyAsync(h.data(), tl.get(), h.size() * 8, cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaStreamSynchronize(st));
    if (const char* out = std::getenv("CSB_TIMELINE_OUT")) {
      if (FILE* f = std::fopen(out, "wb")) {
        std::fwrite(h.data(), 8, h.size(), f);
        std::fclose(f);
      }
    }
#endif
  };
  // staged tile edge (FP32 I/O) and plain variants of each TMEM plan
  auto pick = [&](auto staged_tag) {
    constexpr bool S = decltype(staged_tag)::value;
    switch (M->MT * 100 + M->NB * 10 + M->SB) {
      case 12822: go(mset_estimate_tc_kernel<128, 2, 2, IO, S>); return true;
      case 6422: go(mset_estimate_tc_kernel<64, 2, 2, IO, S>); return true;
      case 6421: go(mset_estimate_tc_kernel<64, 2, 1, IO, S>); return true;
      case 4821: go(mset_estimate_tc_kernel<48, 2, 1, IO, S>); return true;
      case 12811: go(mset_estimate_tc_kernel<128, 1, 1, IO, S>); return true;
      case 6411: go(mset_estimate_tc_kernel<64, 1, 1, IO, S>); return true;
      case 3222: go(mset_estimate_tc_kernel<32, 2, 2, IO, S>); return true;
      case 3221: go(mset_estimate_tc_kernel<32, 2, 1, IO, S>); return true;
      case 3211: go(mset_estimate_tc_kernel<32, 1, 1, IO, S>); return true;
      case 1622: go(mset_estimate_tc_kernel<16, 2, 2, IO, S>); return true;
    }
    return false;
  };
  bool launched;
  if constexpr (sizeof(IO) == 4) {
    launched = p.staged ? pick(std::true_type{}) : pick(std::false_type{});
  } else {
    launched = pick(std::false_type{});
  }
  if (!launched) fail(CS_ERROR, "internal: bad tensor-core tile shape");
}

// Large-n surveillance: per observation block, pack x -> GEMM-A (similarity
// epilogue writes S operand blocks) -> GEMM-B (estimate / residual epilogue).
template <int BN, class Epi>
void launch_gemm3x(cs_ctx* ctx, cudaStream_t st, const GemmShape& g, const Epi& epi) {
  const int tiles = g.m_tiles * g.n_tiles;
  if (tiles == 0) return;
  const size_t smem = gemm3x_smem_bytes<BN>();
  auto kernel = gemm3x_f16_kernel<BN, Epi>;
  CSB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  kernel<<<std::min(tiles, ctx->sm_count), kGemmThreads, smem, st>>>(g, epi);
  CSB_LAUNCH_CHECK();
}

template <typename IO>
void estimate_gemm(cs_ctx* ctx, cudaStream_t st, const cs_model* M, const IO* obs, int64_t N, int64_t ld,
                   IO* est, IO* resid, int slot = 0) {
  if (N == 0) return;
  const int n = static_cast<int>(M->n), m = static_cast<int>(M->m);
  const int64_t m_pad = static_cast<int64_t>(M->ntA) * M->bnA;
  // block size: S operand (FP16 hi + lo: 4 bytes per observation x memory vector) <= 1 GiB
  int64_t Nb = std::max<int64_t>(kGemmBM, ((int64_t{1} << 30) / (m_pad * 4)) / kGemmBM * kGemmBM);
  Nb = std::min<int64_t>(Nb, (N + kGemmBM - 1) / kGemmBM * kGemmBM);
  ctx->wsX[slot].resize(static_cast<size_t>(Nb) * M->kcA * kGemmBK * 2);
  ctx->wsS[slot].resize(static_cast<size_t>(Nb) * m_pad * 2);  // FP16 hi | lo
  ctx->wsXX[slot].resize(Nb);
  for (int64_t t0 = 0; t0 < N; t0 += Nb) {
    const int64_t nc = std::min(Nb, N - t0);
    const int mt = static_cast<int>((nc + kGemmBM - 1) / kGemmBM);
    pack_obs_kernel<IO><<<grid_for(static_cast<int64_t>(mt) * kGemmBM * M->kcA * kGemmBK / 8), 256, 0, st>>>(
        obs + t0, nc, ld, n, M->scale.get(), M->inv_scale.get(), M->aug_x, M->kcA, ctx->wsX[slot].get());
    CSB_LAUNCH_CHECK();
    obs_sqnorm_kernel<IO><<<grid_for(nc), 256, 0, st>>>(obs + t0, nc, ld, n, M->scale.get(),
                                                         M->inv_scale.get(), ctx->wsXX[slot].get());
    CSB_LAUNCH_CHECK();
    EpiSim es{};
    es.s_tiles = ctx->wsS[slot].get();
    es.s_k_chunks = M->kcB;
    es.xx = ctx->wsXX[slot].get();
    es.dd = M->dd.get();
    es.dn32 = M->dn32.get();
    es.obs = obs + t0;
    es.inv_scale_f = M->inv_scale.get();
    es.scale_d = M->scale.get();
    es.io_f64 = sizeof(IO) == 8;
    es.N = nc;
    es.ld = ld;
    es.n = n;
    es.m = m;
    es.kind = M->kind;
    es.inv_h = static_cast<float>(1.0 / M->h);
    es.g_coef = static_cast<float>(1.4426950408889634 / (2.0 * M->h * M->h));
    es.tau = 1.0f / 128.0f;
    es.dd_max = M->dd_max;
    es.s_center = M->s_center;
    const GemmShape ga{ctx->wsX[slot].get(), M->dn_gemm.get(), mt, M->ntA, M->kcA};
    if (M->bnA == 256) launch_gemm3x<256>(ctx, st, ga, es);
    else launch_gemm3x<128>(ctx, st, ga, es);
    EpiOut<IO> eo{obs + t0, est ? est + t0 : nullptr, resid ? resid + t0 : nullptr, M->scale_out_f.get(),
                  M->scale_out_d.get(), nc, ld, n, M->add_f.get(), M->add_d.get()};
    const GemmShape gb{ctx->wsS[slot].get(), M->p_gemm.get(), mt, M->ntB, M->kcB};
    if (M->bnB == 256) launch_gemm3x<256>(ctx, st, gb, eo);
    else launch_gemm3x<128>(ctx, st, gb, eo);
  }
}

void estimate_device_any(cs_ctx* ctx, cudaStream_t st, const cs_model* M, const void* obs,
                         int dtype, int64_t N, int64_t ld, void* est, void* resid) {
  if (M->precision == CS_PRECISION_FP32 && M->gemm) {
    if (dtype == CS_DTYPE_F32)
      estimate_gemm<float>(ctx, st, M, static_cast<const float*>(obs), N, ld, static_cast<float*>(est),
                           static_cast<float*>(resid));
    else
      estimate_gemm<double>(ctx, st, M, static_cast<const double*>(obs), N, ld, static_cast<double*>(est),
                            static_cast<double*>(resid));
    return;
  }
  if (M->precision == CS_PRECISION_FP32 && M->tc) {
    if (dtype == CS_DTYPE_F32)
      launch_tc<float>(ctx, st, M, static_cast<const float*>(obs), N, ld, static_cast<float*>(est),
                       static_cast<float*>(resid));
    else
      launch_tc<double>(ctx, st, M, static_cast<const double*>(obs), N, ld,
                        static_cast<double*>(est), static_cast<double*>(resid));
    return;
  }
  // FP64 path (also serves FP32 models whose n exceeds the fused kernel's
  // TMEM budget -- see DESIGN.md "large-n surveillance").
  if (dtype != CS_DTYPE_F64) fail(CS_CONFIG_ERROR, "FP64 surveillance requires FP64 device I/O");
  estimate_fp64_device(ctx, st, M, static_cast<const double*>(obs), N, ld,
                       static_cast<double*>(est), static_cast<double*>(resid));
}

}  // namespace

// SPRT over device residuals (sprt.cuh); state / counts are host arrays.
template <typename IO>
void sprt_device(cs_ctx* ctx, const IO* resid, int64_t N, int64_t n, int64_t ld, const double* c,
                 const double* h, double A, double B, double* state, uint8_t* d_flags, int64_t* counts) {
  cudaStream_t st = ctx->stream;
  for (int64_t s = 0; s < n; ++s)
    if (!(c[s] > 0.0) || !std::isfinite(c[s]) || !std::isfinite(h[s]))
      fail(CS_CONFIG_ERROR, "sprt: per-signal coefficients must be finite and c > 0");
  if (!(A < 0.0 && B > 0.0)) fail(CS_CONFIG_ERROR, "sprt: thresholds must satisfy A < 0 < B");
  if (N == 0 || n == 0) return;
  if (n > 65535) fail(CS_CONFIG_ERROR, "sprt: at most 65535 signals per call");
  const int chunks = static_cast<int>((N + kSprtChunk - 1) / kSprtChunk);
  // one device block [c | h | state | counts] and one pinned host block:
  // a single H2D before and a single D2H after the two kernels
  TmpBuf<double> dblk(6 * n);
  double* const dc_p = dblk.get();
  double* const dh_p = dc_p + n;
  double* const dstate_p = dh_p + n;
  unsigned long long* const dcount_p = reinterpret_cast<unsigned long long*>(dstate_p + 2 * n);
  TmpBuf<SprtChunk> rec(static_cast<size_t>(n) * chunks);
  double* hp = static_cast<double*>(ctx->pinned(6 * n * sizeof(double)));
  std::memcpy(hp, c, n * 8);
  std::memcpy(hp + n, h, n * 8);
  std::memcpy(hp + 2 * n, state, 2 * n * 8);
  CSB_CUDA(cudaMemcpyAsync(dc_p, hp, 4 * n * 8, cudaMemcpyHostToDevice, st));
  const bool vec = (reinterpret_cast<uintptr_t>(resid) % 16 == 0) && ((ld * sizeof(IO)) % 16 == 0);
  const dim3 grid(ceil_div(chunks, kSprtCta), static_cast<unsigned>(n));
  if (vec)
    sprt_speculate_kernel<IO, true><<<grid, kSprtCta, 0, st>>>(resid, N, ld, dc_p, dh_p, A, B,
                                                               dstate_p, chunks, d_flags, rec.get());
  else
    sprt_speculate_kernel<IO, false><<<grid, kSprtCta, 0, st>>>(resid, N, ld, dc_p, dh_p, A, B,
                                                                dstate_p, chunks, d_flags, rec.get());
  CSB_LAUNCH_CHECK();
  sprt_fixup_kernel<IO><<<ceil_div(n, 4), 128, 0, st>>>(resid, N, static_cast<int>(n), ld, dc_p, dh_p,
                                                         A, B, dstate_p, chunks, d_flags, rec.get(),
                                                         dcount_p);
  CSB_LAUNCH_CHECK();
  // state and counts are adjacent: one D2H into the pinned block (the host
  // copies of c / h there are no longer needed)
  CSB_CUDA(cudaMemcpyAsync(hp, dstate_p, 4 * n * 8, cudaMemcpyDeviceToHost, st));
  CSB_CUDA(cudaStreamSynchronize(st));
  std::memcpy(state, hp, 2 * n * 8);
  if (counts) {
    const unsigned long long* hc = reinterpret_cast<const unsigned long long*>(hp + 2 * n);
    for (int64_t i = 0; i < 2 * n; ++i) counts[i] = static_cast<int64_t>(hc[i]);
  }
}

// eigen_spectrum of a model trained on the certified-Cholesky path: re-form
// the Gram matrix (bitwise the one train factorised) and take its
// eigenvalues on a private context.
void materialize_spectrum(const cs_model* M) {
  std::lock_guard<std::mutex> lock(M->spectrum_mu);
  if (M->spectrum_ready) return;
  cs_ctx* ctx = nullptr;
  if (cs_ctx_create(M->device, &ctx) != CS_OK) fail(CS_ERROR, "eigen_spectrum: " + g_last_error);
  std::unique_ptr<cs_ctx, cs_status (*)(cs_ctx*)> guard(ctx, cs_ctx_destroy);
  StreamScope scope(ctx->stream);
  const int64_t m = M->m;
  TmpBuf<double> gram(m * m), V(m * m);
  form_gram(ctx, M, gram.get());
  M->spectrum.resize(m);
  eig_device(ctx, gram.get(), m, M->spectrum.get(), V.get(), false, false);
  CSB_CUDA(cudaMemcpyAsync(M->spectrum_host.data(), M->spectrum.get(), m * sizeof(double),
                           cudaMemcpyDeviceToHost, ctx->stream));
  CSB_CUDA(cudaStreamSynchronize(ctx->stream));
  M->spectrum_ready = true;
}

// ======================================================================= ABI
extern "C" {

const char* cs_last_error(void) { return g_last_error.c_str(); }

// error channel for the host-side data feed (synth.cpp)
cs_status cs__set_error(cs_status code, const char* msg) {
  g_last_error = msg ? msg : "";
  return code;
}
const char* cs_version(void) { return "cstress-b200 0.1.0 (sm_100a)"; }

cs_status cs_ctx_create(int device, cs_ctx** out) {
  return guarded([&] {
    if (!out) fail(CS_CONFIG_ERROR, "cs_ctx_create: null output");
    int count = 0;
    CSB_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) fail(CS_CONFIG_ERROR, "cs_ctx_create: no such device");
    set_device(device);
    std::unique_ptr<cs_ctx> c(new cs_ctx);
    c->device = device;
    cudaDeviceProp prop{};
    CSB_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) fail(CS_ERROR, std::string("cs_ctx_create: sm_100a device required, found ") + prop.name);
    c->sm_count = prop.multiProcessorCount;
    c->name = prop.name;
    configure_pool(device);
    CSB_CUDA(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
    for (auto& a : c->aux) CSB_CUDA(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
    c->stream = c->own;
    *out = c.release();  // cuSOLVER handle created on the first eigendecomposition
  });
}

cs_status cs_ctx_destroy(cs_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    set_device(ctx->device);
    cudaDeviceSynchronize();  // workspaces are returned to the pool below
    if (ctx->solver) cusolver_api().destroy(ctx->solver);
    if (ctx->blas) cublas_api().destroy(ctx->blas);
    if (ctx->own) cudaStreamDestroy(ctx->own);
    for (auto s : ctx->aux)
      if (s) cudaStreamDestroy(s);
    if (ctx->pin) cudaFreeHost(ctx->pin);
    delete ctx;
  });
}

cs_status cs_ctx_set_stream(cs_ctx* ctx, void* stream) {
  return guarded([&] {
    if (!ctx) fail(CS_CONFIG_ERROR, "null context");
    ctx->stream = static_cast<cudaStream_t>(stream);
  });
}

cs_status cs_ctx_reset_stream(cs_ctx* ctx) {
  return guarded([&] {
    if (!ctx) fail(CS_CONFIG_ERROR, "null context");
    ctx->stream = ctx->own;
  });
}

cs_status cs_ctx_synchronize(cs_ctx* ctx) {
  return guarded([&] {
    set_device(ctx->device);
    CSB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

cs_status cs_ctx_describe(cs_ctx* ctx, char* buf, size_t buflen) {
  return guarded([&] {
    std::snprintf(buf, buflen,
                  "%s, %d SMs; FP64 exact-order SIMT (train, reference-association "
                  "surveillance); tcgen05 3xTF32 fused surveillance; cuSOLVER syevd",
                  ctx->name.c_str(), ctx->sm_count);
  });
}

cs_status cs_sim_matrix(cs_ctx* ctx, const double* A, const double* B, int64_t n, int64_t p,
                        int64_t q, int kind, double bandwidth, double* out) {
  return guarded([&] {
    check_kind(kind);
    set_device(ctx->device);
    const double h = resolve_h(bandwidth, n);
    if (p == 0 || q == 0) return;
    StreamScope scope(ctx->stream);
    TmpBuf<double> dA(n * p + 1), dB(n * q + 1), dO(p * q);
    cudaStream_t st = ctx->stream;
    CSB_CUDA(cudaMemcpyAsync(dA.get(), A, n * p * sizeof(double), cudaMemcpyHostToDevice, st));
    CSB_CUDA(cudaMemcpyAsync(dB.get(), B, n * q * sizeof(double), cudaMemcpyHostToDevice, st));
    launch_sim_exact(st, dA.get(), n, dB.get(), n, n, p, q, kind, h, dO.get(), p);
    CSB_CUDA(cudaMemcpyAsync(out, dO.get(), p * q * sizeof(double), cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaStreamSynchronize(st));
  });
}

cs_status cs_matmul(cs_ctx* ctx, const double* A, const double* B, int64_t p, int64_t k, int64_t q,
                    double* out) {
  return guarded([&] {
    set_device(ctx->device);
    if (p == 0 || q == 0) return;
    cudaStream_t st = ctx->stream;
    StreamScope scope(ctx->stream);
    TmpBuf<double> dA(p * k + 1), dB(k * q + 1), dO(p * q);
    CSB_CUDA(cudaMemcpyAsync(dA.get(), A, p * k * sizeof(double), cudaMemcpyHostToDevice, st));
    CSB_CUDA(cudaMemcpyAsync(dB.get(), B, k * q * sizeof(double), cudaMemcpyHostToDevice, st));
    launch_gemm_exact<false, false>(st, dA.get(), p, dB.get(), k, p, k, q, dO.get(), p);
    CSB_CUDA(cudaMemcpyAsync(out, dO.get(), p * q * sizeof(double), cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaStreamSynchronize(st));
  });
}

cs_status cs_batched_solve(cs_ctx* ctx, const double* G, const double* S, int64_t m, int64_t q,
                           double* out) {
  // backends.cpp:288-293: batched_solve(G+, S) == matmul(G+, S)
  return cs_matmul(ctx, G, S, m, m, q, out);
}

cs_status cs_symmetric_eig(cs_ctx* ctx, const double* G, int64_t m, double* w, double* V) {
  return guarded([&] {
    set_device(ctx->device);
    if (m == 0) return;
    cudaStream_t st = ctx->stream;
    StreamScope scope(ctx->stream);
    TmpBuf<double> dG(m * m), dV(m * m), dw(m);
    CSB_CUDA(cudaMemcpyAsync(dG.get(), G, m * m * sizeof(double), cudaMemcpyHostToDevice, st));
    eig_device(ctx, dG.get(), m, dw.get(), dV.get());
    CSB_CUDA(cudaMemcpyAsync(w, dw.get(), m * sizeof(double), cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaMemcpyAsync(V, dV.get(), m * m * sizeof(double), cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaStreamSynchronize(st));
  });
}

cs_status cs_symmetric_eigvals(cs_ctx* ctx, const double* G, int64_t m, double* w) {
  return guarded([&] {
    if (!ctx || (!G && m > 0) || (!w && m > 0)) fail(CS_CONFIG_ERROR, "symmetric_eigvals: null argument");
    if (m == 0) return;
    set_device(ctx->device);
    StreamScope scope(ctx->stream);
    TmpBuf<double> dG(static_cast<size_t>(m) * m), dV(static_cast<size_t>(m) * m), dw(m);
    CSB_CUDA(cudaMemcpyAsync(dG.get(), G, m * m * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    eig_device(ctx, dG.get(), m, dw.get(), dV.get(), false);
    CSB_CUDA(cudaMemcpyAsync(w, dw.get(), m * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CSB_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

cs_status cs_select_memory_vectors(cs_ctx* ctx, const double* X, int64_t N, int64_t n, int64_t m,
                                   int64_t* idx, double* D) {
  return guarded([&] {
    set_device(ctx->device);
    cudaStream_t st = ctx->stream;
    StreamScope scope(st);
    TmpBuf<double> dX(N * n + 1);
    CSB_CUDA(cudaMemcpyAsync(dX.get(), X, N * n * sizeof(double), cudaMemcpyHostToDevice, st));
    TmpBuf<int64_t> picked;
    std::vector<int64_t> host;
    select_device(ctx, dX.get(), N, n, m, picked, &host);
    std::memcpy(idx, host.data(), m * sizeof(int64_t));
    if (D) {
      TmpBuf<double> dD(n * m);
      gather_memory_kernel<<<grid_for(n * m), 256, 0, st>>>(dX.get(), N, n, picked.get(), m, dD.get());
      CSB_LAUNCH_CHECK();
      CSB_CUDA(cudaMemcpyAsync(D, dD.get(), n * m * sizeof(double), cudaMemcpyDeviceToHost, st));
      CSB_CUDA(cudaStreamSynchronize(st));
    }
  });
}

cs_status cs_mset_train_device(cs_ctx* ctx, const double* dX, int64_t N, int64_t n, int64_t m,
                               int kind, double bandwidth, int precision, cs_model** out) {
  return guarded([&] {
    if (!out) fail(CS_CONFIG_ERROR, "cs_mset_train: null output");
    set_device(ctx->device);
    StreamScope scope(ctx->stream);
    *out = train_device(ctx, dX, N, n, m, kind, bandwidth, precision);
  });
}

cs_status cs_mset_train(cs_ctx* ctx, const double* X, int64_t N, int64_t n, int64_t m, int kind,
                        double bandwidth, int precision, cs_model** out) {
  return guarded([&] {
    if (!out) fail(CS_CONFIG_ERROR, "cs_mset_train: null output");
    set_device(ctx->device);
    StreamScope scope(ctx->stream);
    TmpBuf<double> dX(N * n + 1);
    CSB_CUDA(cudaMemcpyAsync(dX.get(), X, N * n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    *out = train_device(ctx, dX.get(), N, n, m, kind, bandwidth, precision);
  });
}

cs_status cs_mset_estimate_device(cs_ctx* ctx, const cs_model* M, const void* obs, int dtype,
                                  int64_t N, int64_t n, int64_t ld, void* est, void* resid) {
  return guarded([&] {
    if (!M) fail(CS_CONFIG_ERROR, "model was not trained by algorithm mset2");
    set_device(ctx->device);
    check_model_shape(M, n);
    if (ld < N) fail(CS_SHAPE_ERROR, "estimate: leading dimension smaller than observation count");
    estimate_device_any(ctx, ctx->stream, M, obs, dtype, N, ld, est, resid);
  });
}

// Host FP64 in/out: chunks alternate over two streams, each running
// H2D -> kernel -> D2H, so copies in both directions overlap compute.
cs_status cs_mset_estimate(cs_ctx* ctx, const cs_model* M, const double* obs, int64_t N,
                           int64_t n, double* est, double* resid) {
  return guarded([&] {
    if (!M) fail(CS_CONFIG_ERROR, "model was not trained by algorithm mset2");
    set_device(ctx->device);
    check_model_shape(M, n);
    if (N == 0) return;
    const bool tc = M->precision == CS_PRECISION_FP32 && M->tc;
    const bool gm = M->precision == CS_PRECISION_FP32 && M->gemm;
    // chunk: a multiple of the 128-observation tile.  The fused path is
    // PCIe-bound here, so chunks are small (~8 MB in, 16 MB out) and three
    // streams keep both copy directions busy; the two-GEMM path needs larger
    // launches (~256 MB of input) and uses two of the slots.
    int64_t chunk_doubles = gm ? (int64_t{1} << 25) : (int64_t{1} << 19);
    if (const char* e = std::getenv("CSB_E2E_CHUNK_DOUBLES")) chunk_doubles = std::atoll(e);
    int64_t Nc = std::max<int64_t>(kObsTile, chunk_doubles / std::max<int64_t>(n, 1));
    Nc = (Nc + kObsTile - 1) / kObsTile * kObsTile;
    if (!tc && !gm) Nc = std::max<int64_t>(1, std::min<int64_t>(Nc, (int64_t{1} << 27) / std::max<int64_t>(M->m, 1)));
    Nc = std::min(Nc, N);
    const int slots = gm ? 2 : cs_ctx::kSlots;
    cudaEvent_t start;
    CSB_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    CSB_CUDA(cudaEventRecord(start, ctx->stream));
    for (int b = 0; b < slots; ++b) {
      ctx->io_in[b].resize(Nc * n);
      ctx->io_est[b].resize(Nc * n);
      ctx->io_res[b].resize(Nc * n);
      CSB_CUDA(cudaStreamWaitEvent(ctx->aux[b], start, 0));
    }
    int64_t chunk = 0;
    for (int64_t t0 = 0; t0 < N; t0 += Nc, ++chunk) {
      const int b = static_cast<int>(chunk % slots);
      cudaStream_t st = ctx->aux[b];
      const int64_t nc = std::min(Nc, N - t0);
      CSB_CUDA(cudaMemcpy2DAsync(ctx->io_in[b].get(), nc * sizeof(double), obs + t0, N * sizeof(double),
                                 nc * sizeof(double), n, cudaMemcpyHostToDevice, st));
      double* de = est ? ctx->io_est[b].get() : nullptr;
      double* dr = resid ? ctx->io_res[b].get() : nullptr;
      if (tc) {
        launch_tc<double>(ctx, st, M, ctx->io_in[b].get(), nc, nc, de, dr);
      } else if (gm) {
        estimate_gemm<double>(ctx, st, M, ctx->io_in[b].get(), nc, nc, de, dr, b);
      } else {
        estimate_fp64_device(ctx, st, M, ctx->io_in[b].get(), nc, nc, de, dr);
      }
      if (est)
        CSB_CUDA(cudaMemcpy2DAsync(est + t0, N * sizeof(double), de, nc * sizeof(double),
                                   nc * sizeof(double), n, cudaMemcpyDeviceToHost, st));
      if (resid)
        CSB_CUDA(cudaMemcpy2DAsync(resid + t0, N * sizeof(double), dr, nc * sizeof(double),
                                   nc * sizeof(double), n, cudaMemcpyDeviceToHost, st));
      if (!tc && !gm) CSB_CUDA(cudaStreamSynchronize(st));  // FP64 path shares one workspace
    }
    for (int b = 0; b < slots; ++b) CSB_CUDA(cudaStreamSynchronize(ctx->aux[b]));
    cudaEventDestroy(start);
  });
}

cs_status cs_sprt_device(cs_ctx* ctx, const void* d_resid, int dtype, int64_t N, int64_t n, int64_t ld,
                         const double* c, const double* h, double A, double B, double* state,
                         uint8_t* d_flags, int64_t* counts) {
  return guarded([&] {
    if (!ctx || !c || !h || !state || (!d_flags && N * n > 0)) fail(CS_CONFIG_ERROR, "sprt: null argument");
    if (ld < N) fail(CS_SHAPE_ERROR, "sprt: leading dimension smaller than observation count");
    set_device(ctx->device);
    StreamScope scope(ctx->stream);
    if (dtype == CS_DTYPE_F64)
      sprt_device<double>(ctx, static_cast<const double*>(d_resid), N, n, ld, c, h, A, B, state, d_flags, counts);
    else if (dtype == CS_DTYPE_F32)
      sprt_device<float>(ctx, static_cast<const float*>(d_resid), N, n, ld, c, h, A, B, state, d_flags, counts);
    else
      fail(CS_CONFIG_ERROR, "sprt: unknown dtype");
  });
}

cs_status cs_sprt(cs_ctx* ctx, const double* resid, int64_t N, int64_t n, const double* c, const double* h,
                  double A, double B, double* state, uint8_t* flags, int64_t* counts) {
  return guarded([&] {
    if (!ctx || !c || !h || !state || (!resid && N * n > 0)) fail(CS_CONFIG_ERROR, "sprt: null argument");
    set_device(ctx->device);
    StreamScope scope(ctx->stream);
    TmpBuf<double> dr(static_cast<size_t>(N) * n + 1);
    TmpBuf<uint8_t> df(static_cast<size_t>(N) * n + 1);
    if (N * n > 0)
      CSB_CUDA(cudaMemcpyAsync(dr.get(), resid, N * n * 8, cudaMemcpyHostToDevice, ctx->stream));
    sprt_device<double>(ctx, dr.get(), N, n, N, c, h, A, B, state, df.get(), counts);
    if (flags && N * n > 0) {
      CSB_CUDA(cudaMemcpyAsync(flags, df.get(), N * n, cudaMemcpyDeviceToHost, ctx->stream));
      CSB_CUDA(cudaStreamSynchronize(ctx->stream));
    }
  });
}

cs_status cs_model_info(const cs_model* M, int64_t* n, int64_t* m, int64_t* rank, int* kind,
                        double* h, int* precision) {
  return guarded([&] {
    if (!M) fail(CS_CONFIG_ERROR, "null model");
    if (n) *n = M->n;
    if (m) *m = M->m;
    if (rank) *rank = M->rank;
    if (kind) *kind = M->kind;
    if (h) *h = M->h;
    if (precision) *precision = M->precision;
  });
}

cs_status cs_model_export(const cs_model* M, int64_t* idx, double* D, double* pinv, double* spectrum,
                          double* scale) {
  return guarded([&] {
    if (!M) fail(CS_CONFIG_ERROR, "null model");
    set_device(M->device);
    const int64_t n = M->n, m = M->m;
    if (idx) std::memcpy(idx, M->source_indices.data(), m * sizeof(int64_t));
    if (D) CSB_CUDA(cudaMemcpy(D, M->D.get(), n * m * sizeof(double), cudaMemcpyDeviceToHost));
    if (pinv) CSB_CUDA(cudaMemcpy(pinv, M->pinv.get(), m * m * sizeof(double), cudaMemcpyDeviceToHost));
    if (spectrum) {
      materialize_spectrum(M);
      std::memcpy(spectrum, M->spectrum_host.data(), m * sizeof(double));
    }
    if (scale) CSB_CUDA(cudaMemcpy(scale, M->scale.get(), n * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

cs_status cs_model_import(cs_ctx* ctx, int64_t n, int64_t m, int kind, double bandwidth, int64_t rank,
                          const int64_t* idx, const double* D, const double* pinv,
                          const double* spectrum, const double* scale, int precision,
                          cs_model** out) {
  return guarded([&] {
    check_kind(kind);
    if (!out || !D || !pinv || !scale) fail(CS_CONFIG_ERROR, "cs_model_import: null argument");
    set_device(ctx->device);
    cudaStream_t st = ctx->stream;
    StreamScope scope(st);
    std::unique_ptr<cs_model> M(new cs_model);
    M->device = ctx->device;
    M->n = n;
    M->m = m;
    M->rank = rank;
    M->kind = kind;
    M->h = resolve_h(bandwidth, n);
    M->precision = precision;
    M->source_indices.assign(idx ? idx : nullptr, idx ? idx + m : nullptr);
    if (!idx) M->source_indices.assign(m, -1);
    M->spectrum_host.assign(spectrum ? spectrum : nullptr, spectrum ? spectrum + m : nullptr);
    if (!spectrum) M->spectrum_host.assign(m, 0.0);
    M->D.resize(n * m);
    M->Dn.resize(n * m);
    M->scale.resize(n);
    M->pinv.resize(m * m);
    M->spectrum.resize(m);
    CSB_CUDA(cudaMemcpyAsync(M->D.get(), D, n * m * sizeof(double), cudaMemcpyHostToDevice, st));
    CSB_CUDA(cudaMemcpyAsync(M->scale.get(), scale, n * sizeof(double), cudaMemcpyHostToDevice, st));
    CSB_CUDA(cudaMemcpyAsync(M->pinv.get(), pinv, m * m * sizeof(double), cudaMemcpyHostToDevice, st));
    CSB_CUDA(cudaMemcpyAsync(M->spectrum.get(), M->spectrum_host.data(), m * sizeof(double),
                             cudaMemcpyHostToDevice, st));
    // load_model rebuilds memory_normalized (mset.cpp:306-308)
    div_rows_kernel<<<grid_for(n * m), 256, 0, st>>>(M->D.get(), M->scale.get(), n, m, M->Dn.get());
    CSB_LAUNCH_CHECK();
    if (precision == CS_PRECISION_FP32) pack_fp32_operands(ctx, M.get());
    CSB_CUDA(cudaStreamSynchronize(st));
    *out = M.release();
  });
}

cs_status csb_prepare_uniform(int64_t n, int64_t N, double phi, double rho, double variance,
                              double skewness, double kurtosis, double fc[4]);
}  // extern "C"
bool csb_uniform_cholesky(int64_t n, double rho, std::vector<double>& diag, std::vector<double>& below);
extern "C" {

}  // extern "C"
namespace {
cs_status synthesize_uniform_device(cs_ctx* ctx, int64_t n, int64_t N, double phi, double rho, double variance,
                                    double skewness, double kurtosis, uint64_t seed, double* d_out,
                                    float* d_out32);
}
extern "C" {

cs_status cs_synthesize_uniform_device(cs_ctx* ctx, int64_t n, int64_t N, double phi, double rho,
                                       double variance, double skewness, double kurtosis,
                                       uint64_t seed, double* d_out) {
  return synthesize_uniform_device(ctx, n, N, phi, rho, variance, skewness, kurtosis, seed, d_out, nullptr);
}

cs_status cs_synthesize_uniform_device_f32(cs_ctx* ctx, int64_t n, int64_t N, double phi, double rho,
                                           double variance, double skewness, double kurtosis, uint64_t seed,
                                           double* d_work, float* d_out32) {
  if (!d_out32) return guarded([] { fail(CS_CONFIG_ERROR, "synthesize: null FP32 output"); });
  return synthesize_uniform_device(ctx, n, N, phi, rho, variance, skewness, kurtosis, seed, d_work, d_out32);
}

}  // extern "C"

namespace {
cs_status synthesize_uniform_device(cs_ctx* ctx, int64_t n, int64_t N, double phi, double rho, double variance,
                                    double skewness, double kurtosis, uint64_t seed, double* d_out,
                                    float* d_out32) {
  double fc[4];
  const cs_status st0 = csb_prepare_uniform(n, N, phi, rho, variance, skewness, kurtosis, fc);
  if (st0 != CS_OK) return st0;
  return guarded([&] {
    set_device(ctx->device);
    cudaStream_t st = ctx->stream;
    std::vector<double> diag, below;
    const bool mix = n > 1;
    if (mix && !csb_uniform_cholesky(n, rho, diag, below))
      fail(CS_BAD_CORRELATION, "correlation matrix not positive semidefinite within jitter cap 1e-06");
    // chunk length ct = 2^ct_log2 in [32, kChunkT]: the longest that still
    // gives ~2 resident warps' worth of chunk walkers per SM, but no shorter
    // than ~sqrt(N / 10), which balances a walker's ct sequential steps
    // against the carry scan's N / (32 ct) dependent iterations per channel
    // (both latency chains when n x N is small)
    int occ_log2 = 10, lat_log2 = 5;
    while (occ_log2 > 5 && n * ((N + (int64_t{1} << occ_log2) - 1) >> occ_log2) < int64_t{148} * 256 * 2)
      --occ_log2;
    while (lat_log2 < 10 && (int64_t{1} << (2 * (lat_log2 + 1))) * 10 <= N) ++lat_log2;
    const int ct_log2 = std::max(occ_log2, lat_log2);
    const int ct = 1 << ct_log2;
    const int64_t chunks = (N + ct - 1) / ct;
    StreamScope scope(st);
    TmpBuf<unsigned long long> seeds(n);
    TmpBuf<double> state0(n), ends(n * chunks), carry(n * chunks), mean(n), sd(n), dg(n + 1), bl(n + 1),
        phipow(kChunkT), fscale(n), isd(n);
    TmpBuf<double> sums(3 * n * chunks);
    const int nb = ceil_div(N, kApplyT);
    synth_seeds_kernel<<<ceil_div(n, 128), 128, 0, st>>>(seed, static_cast<int>(n), seeds.get());
    synth_burnin_kernel<<<ceil_div(n * 32, 128), 128, 0, st>>>(seeds.get(), static_cast<int>(n), phi, state0.get());
    synth_phi_pow_kernel<<<ceil_div(kChunkT, 256), 256, 0, st>>>(phi, phipow.get());
    synth_ar_local_kernel<<<ceil_div(n * chunks, kArThreads), kArThreads, 0, st>>>(
        seeds.get(), static_cast<int>(n), N, ct, phi, phipow.get(), d_out, ends.get(), sums.get());
    synth_ar_carry_kernel<<<ceil_div(n, kCarryThreads / 32), kCarryThreads, 0, st>>>(
        state0.get(), ends.get(), sums.get(), phipow.get(), static_cast<int>(n), N, ct, phi, carry.get(), mean.get(),
        isd.get());
    CSB_LAUNCH_CHECK();
    if (mix) {
      CSB_CUDA(cudaMemcpyAsync(dg.get(), diag.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
      CSB_CUDA(cudaMemcpyAsync(bl.get(), below.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
    }
    synth_std_mix_kernel<<<ceil_div(N, 256), 256, 0, st>>>(d_out, static_cast<int>(n), N, ct_log2, carry.get(),
                                                           phipow.get(), mean.get(), isd.get(), dg.get(),
                                                           bl.get(), mix ? 1 : 0, fc[0], fc[1], fc[2], fc[3]);
    col_moments_kernel<<<static_cast<unsigned>(n), 256, 0, st>>>(d_out, N, mean.get(), sd.get());
    synth_scale_factor_kernel<<<ceil_div(n, 128), 128, 0, st>>>(sd.get(), static_cast<int>(n), variance,
                                                                fscale.get());
    if (d_out32)
      synth_scale_f32_kernel<<<dim3(nb, static_cast<unsigned>(n)), 256, 0, st>>>(d_out, N, fscale.get(), d_out32);
    else
      synth_scale_kernel<<<dim3(nb, static_cast<unsigned>(n)), 256, 0, st>>>(d_out, N, fscale.get());
    CSB_LAUNCH_CHECK();
    CSB_CUDA(cudaStreamSynchronize(st));
  });
}
}  // namespace

extern "C" {

cs_status cs_model_destroy(cs_model* M) {
  return guarded([&] {
    if (!M) return;
    cudaSetDevice(M->device);
    cudaDeviceSynchronize();  // no call may still read the model's buffers
    delete M;
  });
}

}  // extern "C"

// ================================================================ model wire
// One contiguous device buffer per model (include/cstress_b200.h, "Model
// wire format"): [header 1 KiB][source indices m x i64][spectrum m x f64]
// [device buffers, each 256-byte aligned, in visit order].  The receiving
// rank reads only the header back to the host; the payload stays on the
// device (D2D copies), so a broadcast of the buffer is the whole transfer.
namespace {

constexpr char kWireMagic[8] = {'C', 'S', 'B', 'W', 'I', 'R', 'E', '2'};
constexpr int kWireBuffers = 18;
constexpr int64_t kWireHeader = 1024;

struct WireHeader {
  char magic[8];
  int64_t total_bytes;
  int64_t n, m, rank;
  int32_t kind, precision;
  double h;
  int32_t spectrum_ready, tc, MT, NB, SB, K1, N2, m_tiles, n_stages, gemm;
  int32_t bnA, ntA, kcA, bnB, ntB, kcB;
  float dd_max, aug_x, s_center;
  int64_t count[kWireBuffers];  // elements per device buffer
  int64_t elem[kWireBuffers];   // element size per device buffer
};
static_assert(sizeof(WireHeader) <= kWireHeader, "wire header exceeds its slot");

// every device buffer of a model, in wire order (the one place that lists them)
template <class M, class F>
void visit_model_buffers(M* model, F&& f) {
  f(model->D); f(model->Dn); f(model->scale); f(model->pinv); f(model->spectrum);
  f(model->dn_tiles); f(model->p_tiles); f(model->dd); f(model->dn32); f(model->inv_scale);
  f(model->scale_f); f(model->scale_out_f); f(model->p_shift); f(model->scale_out_d);
  f(model->dn_gemm); f(model->p_gemm); f(model->add_f); f(model->add_d);
}

int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }

WireHeader wire_header(const cs_model* M) {
  WireHeader w;
  std::memset(&w, 0, sizeof w);
  std::memcpy(w.magic, kWireMagic, 8);
  w.n = M->n; w.m = M->m; w.rank = M->rank; w.kind = M->kind; w.precision = M->precision; w.h = M->h;
  w.spectrum_ready = M->spectrum_ready ? 1 : 0;
  w.tc = M->tc; w.MT = M->MT; w.NB = M->NB; w.SB = M->SB; w.K1 = M->K1; w.N2 = M->N2;
  w.m_tiles = M->m_tiles; w.n_stages = M->n_stages; w.gemm = M->gemm;
  w.bnA = M->bnA; w.ntA = M->ntA; w.kcA = M->kcA; w.bnB = M->bnB; w.ntB = M->ntB; w.kcB = M->kcB;
  w.dd_max = M->dd_max; w.aug_x = M->aug_x; w.s_center = M->s_center;
  int i = 0;
  visit_model_buffers(M, [&](const auto& b) {
    w.count[i] = static_cast<int64_t>(b.count);
    w.elem[i] = static_cast<int64_t>(sizeof(*b.ptr));
    ++i;
  });
  int64_t off = kWireHeader + align256(16 * w.m);
  for (int k = 0; k < kWireBuffers; ++k) off += align256(w.count[k] * w.elem[k]);
  w.total_bytes = off;
  return w;
}

}  // namespace

extern "C" {

cs_status cs_model_wire_size(const cs_model* M, int64_t* bytes) {
  return guarded([&] {
    if (!M || !bytes) fail(CS_CONFIG_ERROR, "cs_model_wire_size: null argument");
    *bytes = wire_header(M).total_bytes;
  });
}

cs_status cs_model_pack_device(cs_ctx* ctx, const cs_model* M, void* d_wire, int64_t bytes) {
  return guarded([&] {
    if (!ctx || !M || !d_wire) fail(CS_CONFIG_ERROR, "cs_model_pack_device: null argument");
    if (M->device != ctx->device) fail(CS_CONFIG_ERROR, "cs_model_pack_device: model lives on another device");
    set_device(ctx->device);
    std::lock_guard<std::mutex> lock(M->spectrum_mu);  // not mid-materialisation
    const WireHeader w = wire_header(M);
    if (bytes < w.total_bytes) fail(CS_CONFIG_ERROR, "cs_model_pack_device: wire buffer too small");
    cudaStream_t st = ctx->stream;
    auto* base = static_cast<unsigned char*>(d_wire);
    const int64_t m = M->m;
    std::vector<unsigned char> host(kWireHeader + 16 * m, 0);
    std::memcpy(host.data(), &w, sizeof w);
    std::memcpy(host.data() + kWireHeader, M->source_indices.data(), 8 * m);
    std::memcpy(host.data() + kWireHeader + 8 * m, M->spectrum_host.data(), 8 * m);
    CSB_CUDA(cudaMemcpyAsync(base, host.data(), host.size(), cudaMemcpyHostToDevice, st));
    int64_t off = kWireHeader + align256(16 * m);
    visit_model_buffers(M, [&](const auto& b) {
      const int64_t nb = static_cast<int64_t>(b.count * sizeof(*b.ptr));
      if (nb) CSB_CUDA(cudaMemcpyAsync(base + off, b.ptr, nb, cudaMemcpyDeviceToDevice, st));
      off += align256(nb);
    });
    CSB_CUDA(cudaStreamSynchronize(st));  // `host` is pageable: complete before it goes
  });
}

cs_status cs_model_unpack_device(cs_ctx* ctx, const void* d_wire, int64_t bytes, cs_model** out) {
  return guarded([&] {
    if (!ctx || !d_wire || !out) fail(CS_CONFIG_ERROR, "cs_model_unpack_device: null argument");
    if (bytes < kWireHeader) fail(CS_CONFIG_ERROR, "cs_model_unpack_device: buffer shorter than the header");
    set_device(ctx->device);
    cudaStream_t st = ctx->stream;
    StreamScope scope(st);
    const auto* base = static_cast<const unsigned char*>(d_wire);
    WireHeader w;
    CSB_CUDA(cudaMemcpyAsync(&w, base, sizeof w, cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaStreamSynchronize(st));
    if (std::memcmp(w.magic, kWireMagic, 8) != 0)
      fail(CS_IO_ERROR, "cs_model_unpack_device: not a model wire buffer (bad magic)");
    if (w.total_bytes > bytes)
      fail(CS_CONFIG_ERROR, "cs_model_unpack_device: buffer shorter than the wire it holds");
    if (w.n < 1 || w.m < 1) fail(CS_IO_ERROR, "cs_model_unpack_device: corrupt header");
    check_kind(w.kind);
    std::unique_ptr<cs_model> M(new cs_model);
    M->device = ctx->device;
    M->n = w.n; M->m = w.m; M->rank = w.rank; M->kind = w.kind; M->precision = w.precision; M->h = w.h;
    M->spectrum_ready = w.spectrum_ready != 0;
    M->tc = w.tc; M->MT = w.MT; M->NB = w.NB; M->SB = w.SB; M->K1 = w.K1; M->N2 = w.N2;
    M->m_tiles = w.m_tiles; M->n_stages = w.n_stages; M->gemm = w.gemm;
    M->bnA = w.bnA; M->ntA = w.ntA; M->kcA = w.kcA; M->bnB = w.bnB; M->ntB = w.ntB; M->kcB = w.kcB;
    M->dd_max = w.dd_max; M->aug_x = w.aug_x; M->s_center = w.s_center;
    const int64_t m = w.m;
    M->source_indices.resize(m);
    M->spectrum_host.resize(m);
    CSB_CUDA(cudaMemcpyAsync(M->source_indices.data(), base + kWireHeader, 8 * m, cudaMemcpyDeviceToHost, st));
    CSB_CUDA(cudaMemcpyAsync(M->spectrum_host.data(), base + kWireHeader + 8 * m, 8 * m,
                             cudaMemcpyDeviceToHost, st));
    int64_t off = kWireHeader + align256(16 * m);
    int i = 0;
    visit_model_buffers(M.get(), [&](auto& b) {
      if (w.elem[i] != static_cast<int64_t>(sizeof(*b.ptr)))
        fail(CS_IO_ERROR, "cs_model_unpack_device: wire layout from another library version");
      const int64_t nb = w.count[i] * w.elem[i];
      if (w.count[i]) {
        b.resize(static_cast<size_t>(w.count[i]));
        CSB_CUDA(cudaMemcpyAsync(b.ptr, base + off, nb, cudaMemcpyDeviceToDevice, st));
      }
      off += align256(nb);
      ++i;
    });
    CSB_CUDA(cudaStreamSynchronize(st));
    *out = M.release();
  });
}

}  // extern "C"
