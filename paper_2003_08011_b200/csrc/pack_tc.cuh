// pack_tc.cuh -- one-time (train) pre-tiling of the FP32 tensor-core operands.
#pragma once

#include "sm100_ptx.cuh"

namespace csb {

// Operand pre-tiling (once per model, at train time).  Canonical K-major,
// no-swizzle layout: element (r, k) of an R x K block sits at byte
//   (r%8)*16 + (r/8)*128 + (k%4)*4 + (k/4)*LBO,  LBO = (R/8)*128.
__device__ __forceinline__ size_t canon_off(int r, int k, int R) {
  return static_cast<size_t>((r & 7) * 4 + (r >> 3) * 32 + (k & 3) + (k >> 2) * (R / 8) * 32);
}

// D_norm^T tiles: block j holds memory vectors j*MT.. as rows, signals as K,
// pre-scaled for the GEMM-form distance: column k < n holds -2 d_k (exact),
// column n holds ||d||^2 (FP64, split) -- with x augmented by a constant 1 in
// column n, GEMM1 yields ||d||^2 - 2 x.d directly (one FADD of ||x||^2 left).
__global__ void pack_dn_tiles_kernel(const double* __restrict__ Dn, int n, int m, int MT, int K1,
                                     int m_tiles, float* __restrict__ out) {
  const int64_t per = static_cast<int64_t>(MT) * K1;
  const int64_t total = per * m_tiles;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(e / per);
    const int rem = static_cast<int>(e % per);
    const int r = rem % MT, k = rem / MT;
    const int mem = j * MT + r;
    double v = 0.0;
    if (mem < m) {
      if (k < n) {
        v = -2.0 * Dn[k + static_cast<int64_t>(mem) * n];
      } else if (k == n) {
        for (int s = 0; s < n; ++s) {
          const double d = Dn[s + static_cast<int64_t>(mem) * n];
          v = fma(d, d, v);
        }
      }
    }
    const float f = static_cast<float>(v);
    const float hi = __uint_as_float(ptx::to_tf32(f));
    const float lo = static_cast<float>(v - static_cast<double>(hi));
    float* blk = out + static_cast<size_t>(j) * 2 * per;
    blk[canon_off(r, k, MT)] = hi;
    blk[per + canon_off(r, k, MT)] = lo;
  }
}

// P^T tiles: block j holds signals as rows (N2), memory vectors j*MT.. as K.
__global__ void pack_p_tiles_kernel(const double* __restrict__ P, int n, int m, int MT, int N2,
                                    int m_tiles, float* __restrict__ out) {
  const int64_t per = static_cast<int64_t>(N2) * MT;
  const int64_t total = per * m_tiles;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(e / per);
    const int rem = static_cast<int>(e % per);
    const int r = rem % N2, k = rem / N2;
    const int mem = j * MT + k;
    const double v = (r < n && mem < m) ? P[r + static_cast<int64_t>(mem) * n] : 0.0;
    const float f = static_cast<float>(v);
    const float hi = __uint_as_float(ptx::to_tf32(f));
    const float lo = static_cast<float>(v - static_cast<double>(hi));
    float* blk = out + static_cast<size_t>(j) * 2 * per;
    blk[canon_off(r, k, N2)] = hi;
    blk[per + canon_off(r, k, N2)] = lo;
  }
}

// ||D_norm(:, c)||^2 (FP64 -> FP32, zero padded), D_norm in FP32, 1/scale.
__global__ void pack_aux_kernel(const double* __restrict__ Dn, const double* __restrict__ scale,
                                int n, int m, int m_pad, float* __restrict__ dd,
                                float* __restrict__ dn32, float* __restrict__ inv_scale,
                                float* __restrict__ scale_f) {
  const int64_t tid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t c = tid; c < m_pad; c += stride) {
    double a = 0.0;
    if (c < m)
      for (int s = 0; s < n; ++s) {
        const double v = Dn[s + c * n];
        a = fma(v, v, a);
      }
    dd[c] = static_cast<float>(a);
  }
  for (int64_t e = tid; e < static_cast<int64_t>(n) * m; e += stride) dn32[e] = static_cast<float>(Dn[e]);
  for (int64_t s = tid; s < n; s += stride) {
    inv_scale[s] = static_cast<float>(1.0 / scale[s]);
    scale_f[s] = static_cast<float>(scale[s]);
  }
}


}  // namespace csb
