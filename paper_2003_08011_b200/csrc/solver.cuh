// solver.cuh -- lazily bound cuSOLVER entry points for the FP64 symmetric
// eigendecomposition (symmetric_eig, mset.cpp:57-70).
//
// cuSOLVER and its dependencies (cuBLAS / cuBLASLt / cuSPARSE / nvJitLink,
// ~1.5 GB) are not linked at load time: on a cold box, mapping them costs
// minutes.  They are dlopen'ed on the first eigendecomposition, preferring
// the copies PyTorch itself maps (the venv's nvidia/* packages), so a process
// that already imported torch shares their pages.
#pragma once

#include <cublas_v2.h>
#include <cusolverDn.h>
#include <dlfcn.h>

#include <cstdlib>
#include <mutex>
#include <string>

#include "common.cuh"

namespace csb {

struct CusolverApi {
  void* lib = nullptr;
  std::string path;
  cusolverStatus_t (*create)(cusolverDnHandle_t*) = nullptr;
  cusolverStatus_t (*destroy)(cusolverDnHandle_t) = nullptr;
  cusolverStatus_t (*set_stream)(cusolverDnHandle_t, cudaStream_t) = nullptr;
  cusolverStatus_t (*syevd_buffer)(cusolverDnHandle_t, cusolverEigMode_t, cublasFillMode_t, int,
                                   const double*, int, const double*, int*) = nullptr;
  cusolverStatus_t (*syevd)(cusolverDnHandle_t, cusolverEigMode_t, cublasFillMode_t, int, double*,
                            int, double*, double*, int, int*) = nullptr;
  // Cholesky factor / inverse (full-rank fast path of the pseudo-inverse)
  cusolverStatus_t (*potrf_buffer)(cusolverDnHandle_t, cublasFillMode_t, int, double*, int, int*) = nullptr;
  cusolverStatus_t (*potrf)(cusolverDnHandle_t, cublasFillMode_t, int, double*, int, double*, int,
                            int*) = nullptr;
  cusolverStatus_t (*potri_buffer)(cusolverDnHandle_t, cublasFillMode_t, int, double*, int, int*) = nullptr;
  cusolverStatus_t (*potri)(cusolverDnHandle_t, cublasFillMode_t, int, double*, int, double*, int,
                            int*) = nullptr;
  cusolverStatus_t (*potrs)(cusolverDnHandle_t, cublasFillMode_t, int, int, const double*, int, double*, int,
                            int*) = nullptr;
};

// cuBLAS DGEMM (FP64 tensor-core path) for the train pipeline's one plain
// library product, P = D_norm G+.  Bound lazily like cuSOLVER; null api.lib when absent.
struct CublasApi {
  void* lib = nullptr;
  cublasStatus_t (*create)(cublasHandle_t*) = nullptr;
  cublasStatus_t (*destroy)(cublasHandle_t) = nullptr;
  cublasStatus_t (*set_stream)(cublasHandle_t, cudaStream_t) = nullptr;
  cublasStatus_t (*dgemm)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int, const double*,
                          const double*, int, const double*, int, const double*, double*, int) = nullptr;
  cublasStatus_t (*dgemm_batched)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int,
                                  const double*, const double* const*, int, const double* const*, int,
                                  const double*, double* const*, int, int) = nullptr;
  cublasStatus_t (*dgemm_strided)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int,
                                  const double*, const double*, int, long long, const double*, int, long long,
                                  const double*, double*, int, long long, int) = nullptr;
};

inline const CublasApi& cublas_api() {
  static CublasApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* candidates[] = {
        std::getenv("CSB_CUBLAS"),
        "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/cublas/lib/libcublas.so.12",
        "libcublas.so.12",
        "/usr/local/cuda/lib64/libcublas.so.12",
    };
    for (const char* c : candidates) {
      if (!c) continue;
      if (void* h = dlopen(c, RTLD_NOW | RTLD_LOCAL)) {
        api.lib = h;
        break;
      }
    }
    if (!api.lib) return;
    api.create = reinterpret_cast<decltype(api.create)>(dlsym(api.lib, "cublasCreate_v2"));
    api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(api.lib, "cublasDestroy_v2"));
    api.set_stream = reinterpret_cast<decltype(api.set_stream)>(dlsym(api.lib, "cublasSetStream_v2"));
    api.dgemm = reinterpret_cast<decltype(api.dgemm)>(dlsym(api.lib, "cublasDgemm_v2"));
    api.dgemm_batched = reinterpret_cast<decltype(api.dgemm_batched)>(dlsym(api.lib, "cublasDgemmBatched"));
    api.dgemm_strided =
        reinterpret_cast<decltype(api.dgemm_strided)>(dlsym(api.lib, "cublasDgemmStridedBatched"));
    if (!api.create || !api.destroy || !api.set_stream || !api.dgemm || !api.dgemm_strided || !api.dgemm_batched) api.lib = nullptr;
  });
  return api;
}

inline const CusolverApi& cusolver_api() {
  static CusolverApi api;
  static std::once_flag once;
  static std::string error;
  std::call_once(once, [] {
    const char* env = std::getenv("CSB_CUSOLVER");
    const char* candidates[] = {
        env,
        "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/cusolver/lib/libcusolver.so.11",
        "libcusolver.so.11",
        "/usr/local/cuda/lib64/libcusolver.so.11",
    };
    for (const char* c : candidates) {
      if (!c) continue;
      void* h = dlopen(c, RTLD_NOW | RTLD_LOCAL);
      if (!h) {
        error += std::string(dlerror()) + "; ";
        continue;
      }
      api.lib = h;
      api.path = c;
      break;
    }
    if (!api.lib) return;
    api.create = reinterpret_cast<decltype(api.create)>(dlsym(api.lib, "cusolverDnCreate"));
    api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(api.lib, "cusolverDnDestroy"));
    api.set_stream = reinterpret_cast<decltype(api.set_stream)>(dlsym(api.lib, "cusolverDnSetStream"));
    api.syevd_buffer =
        reinterpret_cast<decltype(api.syevd_buffer)>(dlsym(api.lib, "cusolverDnDsyevd_bufferSize"));
    api.syevd = reinterpret_cast<decltype(api.syevd)>(dlsym(api.lib, "cusolverDnDsyevd"));
    api.potrf_buffer =
        reinterpret_cast<decltype(api.potrf_buffer)>(dlsym(api.lib, "cusolverDnDpotrf_bufferSize"));
    api.potrf = reinterpret_cast<decltype(api.potrf)>(dlsym(api.lib, "cusolverDnDpotrf"));
    api.potri_buffer =
        reinterpret_cast<decltype(api.potri_buffer)>(dlsym(api.lib, "cusolverDnDpotri_bufferSize"));
    api.potri = reinterpret_cast<decltype(api.potri)>(dlsym(api.lib, "cusolverDnDpotri"));
    api.potrs = reinterpret_cast<decltype(api.potrs)>(dlsym(api.lib, "cusolverDnDpotrs"));
    if (!api.create || !api.destroy || !api.set_stream || !api.syevd_buffer || !api.syevd ||
        !api.potrf_buffer || !api.potrf || !api.potri_buffer || !api.potri || !api.potrs) {
      error += "missing cuSOLVER symbols in " + api.path;
      api.lib = nullptr;
    }
  });
  if (!api.lib) fail(CS_ERROR, "symmetric_eig: cannot load cuSOLVER (" + error + ")");
  return api;
}

}  // namespace csb
