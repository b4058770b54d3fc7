// common.cuh -- error plumbing and device-memory helpers shared by the
// B200 MSET2 kernels.  Internal C++ only; the public surface is the C-ABI in
// include/cstress_b200.h.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>

#include "cstress_b200.h"

namespace csb {

// Internal failure carrying a cs_status (1:1 with the reference's exception
// classes, errors.hpp:9-74) and the reference's message text.
struct Failure {
  cs_status code;
  std::string msg;
};

[[noreturn]] inline void fail(cs_status code, std::string msg) {
  throw Failure{code, std::move(msg)};
}

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    char buf[512];
    std::snprintf(buf, sizeof buf, "CUDA error in %s (%s:%d): %s", what, file, line,
                  cudaGetErrorString(e));
    fail(CS_ERROR, buf);
  }
}
#define CSB_CUDA(x) ::csb::cuda_check((x), #x, __FILE__, __LINE__)
#define CSB_LAUNCH_CHECK() ::csb::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// Owning device buffer (grow-only when reused as workspace).
template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  size_t count = 0;
  DevBuf() = default;
  explicit DevBuf(size_t n) { resize(n); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), count(o.count) { o.ptr = nullptr; o.count = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      ptr = o.ptr;
      count = o.count;
      o.ptr = nullptr;
      o.count = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    count = 0;
  }
  void resize(size_t n) {  // discards contents
    if (n <= count && ptr) return;
    release();
    if (n == 0) return;
    CSB_CUDA(cudaMalloc(&ptr, n * sizeof(T)));
    count = n;
  }
  T* get() const { return ptr; }
};

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace csb
