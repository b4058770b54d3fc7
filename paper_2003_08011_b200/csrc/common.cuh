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

// Stream the C-ABI call in progress runs on (set by the entry points); device
// buffers are allocated / freed stream-ordered on it from the device's
// default memory pool, whose release threshold is raised so freed blocks are
// cached instead of returned to the driver (no device-wide sync per free).
inline cudaStream_t& alloc_stream() {
  static thread_local cudaStream_t s = nullptr;
  return s;
}

inline void configure_pool(int device) {
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t threshold = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
  }
}

struct StreamScope {  // RAII: route DevBuf traffic to `s` for one call
  cudaStream_t prev;
  explicit StreamScope(cudaStream_t s) : prev(alloc_stream()) { alloc_stream() = s; }
  ~StreamScope() { alloc_stream() = prev; }
};

// Owning device buffer (grow-only when reused as workspace).
template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  size_t count = 0;
  DevBuf() = default;
  explicit DevBuf(size_t n) { resize(n); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), count(o.count), stream(o.stream) {
    o.ptr = nullptr;
    o.count = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      ptr = o.ptr;
      count = o.count;
      stream = o.stream;
      o.ptr = nullptr;
      o.count = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (ptr) {
      cudaFreeAsync(ptr, stream);
    }
    ptr = nullptr;
    count = 0;
  }
  void resize(size_t n) {  // discards contents
    if (n <= count && ptr) return;
    release();
    if (n == 0) return;
    // every buffer comes from the device's caching pool: a plain cudaMalloc /
    // cudaFree pair per model buffer cost 2-30 ms of page mapping and an
    // implicit device sync per train call.  Temporaries are freed on their
    // call's stream; long-lived (model / context) buffers on the legacy
    // stream after their owner synchronised the device.
    CSB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ptr), n * sizeof(T), alloc_stream()));
    // a long-lived buffer may next be used on another stream: complete the
    // allocation before returning it (cheap when the pool has the block)
    if (!async) CSB_CUDA(cudaStreamSynchronize(alloc_stream()));
    stream = async ? alloc_stream() : nullptr;
    count = n;
  }
  cudaStream_t stream = nullptr;
  bool async = false;  // call-local temporary (freed stream-ordered on its call's stream)
  T* get() const { return ptr; }
};

// Call-local temporary: allocated and freed stream-ordered on alloc_stream()
// from the (caching) device memory pool.  Must not outlive the call's stream.
template <typename T>
struct TmpBuf : DevBuf<T> {
  TmpBuf() { this->async = true; }
  explicit TmpBuf(size_t n) {
    this->async = true;
    this->resize(n);
  }
};

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace csb
