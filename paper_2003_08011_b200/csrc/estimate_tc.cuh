// estimate_tc.cuh -- fused MSET2 surveillance on 5th-gen tensor cores.
//
// Per observation x (n signals) and memory matrix D_norm (n x m):
//   s_i   = k( ||x||^2 + ||d_i||^2 - 2 x.d_i )          (similarity, kernels.hpp:54-57)
//   x_hat = scale .* (P s),   P = D_norm G+  (n x m)     (reassociated mset.cpp:189-193)
//   r     = x - x_hat                                     (mset.cpp:197)
// This is attention-shaped (Q = X, K = D_norm, V = P^T, elementwise kernel map
// instead of softmax, no normaliser) and is computed flash-style: the m x N
// similarity matrix never touches HBM (the reference materialises it,
// mset.cpp:189-191).
//
// One CTA (persistent, grid = #SMs) owns a 128-observation tile at a time and
// streams the memory matrix in MT-wide tiles.  Warp roles:
//   warp 0      producer: 1D bulk copies (TMA engine) of pre-tiled D_norm^T and
//               P^T operand tiles into a 2-deep shared-memory ring each
//   warp 1      MMA issuer (one thread): tcgen05.mma kind::tf32
//   warps 2..5  epilogue: x prologue, TMEM->reg kernel map, reg->TMEM S,
//               final estimate / residual stores
// TMEM (512 columns x 128 lanes, lane = observation):
//   [0, N2)             O   = S P^T accumulator          (GEMM2 D)
//   [N2, N2+2K1)        X   = x_norm hi | lo              (GEMM1 A, "TS" form)
//   [.., +MT)           ACC = X D_norm accumulator         (GEMM1 D)
//   [.., +2MT)          S   = similarity hi | lo           (GEMM2 A, "TS" form)
// FP32-accurate products on TF32 hardware: every operand v is split into
// hi = rna_tf32(v), lo = v - hi and each GEMM issues hi*hi + hi*lo + lo*hi
// (3xTF32).  Single-pass TF32 misses the 1e-3 tolerance.
// d2 in GEMM form cancels near zero; entries with d2 < tau (|x|^2+|d|^2) are
// recomputed by direct difference, which keeps memory vectors
// reproducing themselves.
#pragma once

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace csb {

constexpr int kTcThreads = 192;
constexpr int kObsTile = 128;
constexpr int kTmemCols = 512;

struct TcParams {
  const void* obs;  // N x n, leading dim ld, IO type
  int64_t N, ld;
  int n, K1, N2, m, m_tiles;
  const float* dn_tiles;  // m_tiles x [hi | lo] (MT x K1 canonical K-major)
  const float* p_tiles;   // m_tiles x [hi | lo] (N2 x MT canonical K-major)
  const float* dd;        // m_tiles*MT squared norms of D_norm columns (0 padded)
  const float* dn32;      // n x m D_norm in FP32 (direct-difference recompute)
  const float* inv_scale; // n
  const float* scale_f;   // n
  const double* scale_d;  // n
  int kind;
  float inv_h;   // 1/h            (inverse distance)
  float g_coef;  // log2(e)/(2h^2) (gaussian)
  float tau;     // near-zero recompute threshold
  void* est;
  void* resid;
  uint32_t dn_stage_bytes, p_stage_bytes;
};

template <typename IO>
__device__ __forceinline__ float load_norm(const IO* obs, int64_t idx, int s,
                                           const TcParams& p) {
  if constexpr (sizeof(IO) == 8) {
    return static_cast<float>(static_cast<double>(obs[idx]) / p.scale_d[s]);
  } else {
    return static_cast<float>(obs[idx]) * p.inv_scale[s];
  }
}

template <int MT, typename IO>
__global__ void __launch_bounds__(kTcThreads, 1) mset_estimate_tc_kernel(const TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint8_t* dn_ring = smem;
  uint8_t* p_ring = smem + 2 * p.dn_stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(p_ring + 2 * p.p_stage_bytes);
  uint64_t* dn_full = bars + 0;
  uint64_t* dn_empty = bars + 2;
  uint64_t* p_full = bars + 4;
  uint64_t* p_empty = bars + 6;
  uint64_t* x_ready = bars + 8;
  uint64_t* x_free = bars + 9;
  uint64_t* acc_full = bars + 10;
  uint64_t* acc_free = bars + 11;
  uint64_t* s_ready = bars + 12;
  uint64_t* s_free = bars + 13;
  uint64_t* o_full = bars + 14;
  uint64_t* o_free = bars + 15;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 16);

  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) ptx::mbar_init(&bars[i], 1);
    ptx::mbar_init(x_ready, 4);
    ptx::mbar_init(x_free, 1);
    ptx::mbar_init(acc_full, 1);
    ptx::mbar_init(acc_free, 4);
    ptx::mbar_init(s_ready, 4);
    ptx::mbar_init(s_free, 1);
    ptx::mbar_init(o_full, 1);
    ptx::mbar_init(o_free, 4);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc(tmem_holder, kTmemCols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  const int K1 = p.K1, N2 = p.N2;
  const uint32_t colO = 0;
  const uint32_t colXh = N2, colXl = N2 + K1;
  const uint32_t colS = N2 + 2 * K1;
  const uint32_t colSh = colS + MT, colSl = colS + 2 * MT;
  const int n_tiles = static_cast<int>((p.N + kObsTile - 1) / kObsTile);

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      uint32_t g = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        for (int j = 0; j < p.m_tiles; ++j, ++g) {
          const uint32_t st = g & 1, u = g >> 1;
          ptx::mbar_wait(&dn_empty[st], (u & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&dn_full[st], p.dn_stage_bytes);
          ptx::bulk_g2s(dn_ring + st * p.dn_stage_bytes,
                        p.dn_tiles + static_cast<size_t>(j) * (p.dn_stage_bytes / 4),
                        p.dn_stage_bytes, &dn_full[st]);
          ptx::mbar_wait(&p_empty[st], (u & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&p_full[st], p.p_stage_bytes);
          ptx::bulk_g2s(p_ring + st * p.p_stage_bytes,
                        p.p_tiles + static_cast<size_t>(j) * (p.p_stage_bytes / 4),
                        p.p_stage_bytes, &p_full[st]);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc1 = ptx::idesc_tf32(128, MT);
      const uint32_t idesc2 = ptx::idesc_tf32(128, N2);
      const uint32_t SBO = 128;
      const uint32_t LBO1 = (MT / 8) * 128;  // D_norm^T tile: MT rows x K1
      const uint32_t LBO2 = (N2 / 8) * 128;  // P^T tile: N2 rows x MT
      uint32_t g1 = 0, g2 = 0, tcount = 0;
      auto issue_g2 = [&](int jj) {
        const uint32_t st = g2 & 1, u = g2 >> 1;
        ptx::mbar_wait(s_ready, g2 & 1);
        ptx::mbar_wait(&p_full[st], u & 1);
        if (jj == 0) ptx::mbar_wait(o_free, (tcount & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t hi = ptx::smem_u32(p_ring + st * p.p_stage_bytes);
        const uint32_t lo = hi + N2 * MT * 4;
#pragma unroll
        for (int kk = 0; kk < MT / 8; ++kk) {
          const uint64_t bh = ptx::smem_desc(hi + kk * 2 * LBO2, LBO2, SBO);
          const uint64_t bl = ptx::smem_desc(lo + kk * 2 * LBO2, LBO2, SBO);
          const uint32_t ah = tmem + colSh + kk * 8, al = tmem + colSl + kk * 8;
          const uint32_t first = (jj == 0 && kk == 0);
          ptx::mma_tf32_ts(tmem + colO, al, bh, idesc2, first ? 0u : 1u);
          ptx::mma_tf32_ts(tmem + colO, ah, bl, idesc2, 1u);
          ptx::mma_tf32_ts(tmem + colO, ah, bh, idesc2, 1u);
        }
        ptx::tc_commit(s_free);
        ptx::tc_commit(&p_empty[st]);
        ++g2;
      };
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++tcount) {
        ptx::mbar_wait(x_ready, tcount & 1);
        for (int j = 0; j < p.m_tiles; ++j) {
          const uint32_t st = g1 & 1, u = g1 >> 1;
          ptx::mbar_wait(&dn_full[st], u & 1);
          ptx::mbar_wait(acc_free, (g1 & 1) ^ 1);
          ptx::tc_fence_after();
          const uint32_t hi = ptx::smem_u32(dn_ring + st * p.dn_stage_bytes);
          const uint32_t lo = hi + MT * K1 * 4;
          for (int kk = 0; kk < K1 / 8; ++kk) {
            const uint64_t bh = ptx::smem_desc(hi + kk * 2 * LBO1, LBO1, SBO);
            const uint64_t bl = ptx::smem_desc(lo + kk * 2 * LBO1, LBO1, SBO);
            const uint32_t ah = tmem + colXh + kk * 8, al = tmem + colXl + kk * 8;
            ptx::mma_tf32_ts(tmem + colS, al, bh, idesc1, kk > 0 ? 1u : 0u);
            ptx::mma_tf32_ts(tmem + colS, ah, bl, idesc1, 1u);
            ptx::mma_tf32_ts(tmem + colS, ah, bh, idesc1, 1u);
          }
          ptx::tc_commit(acc_full);
          ptx::tc_commit(&dn_empty[st]);
          if (j == p.m_tiles - 1) ptx::tc_commit(x_free);
          ++g1;
          if (j >= 1) issue_g2(j - 1);
        }
        issue_g2(p.m_tiles - 1);
        ptx::tc_commit(o_full);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = 32 * q + lane;
    const uint32_t lane_off = static_cast<uint32_t>(32 * q) << 16;
    const IO* obs = static_cast<const IO*>(p.obs);
    IO* est = static_cast<IO*>(p.est);
    IO* resid = static_cast<IO*>(p.resid);

    uint32_t prologue_count = 0;
    auto prologue = [&](int tile, float& xx) {
      ptx::mbar_wait(x_free, (prologue_count & 1) ^ 1);
      ++prologue_count;
      ptx::tc_fence_after();
      const int64_t t = static_cast<int64_t>(tile) * kObsTile + row;
      const bool valid = t < p.N;
      float acc = 0.f;
      for (int k8 = 0; k8 < K1 / 8; ++k8) {
        uint32_t hi[8], lo[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int s = k8 * 8 + e;
          float xv = 0.f;
          if (valid && s < p.n) xv = load_norm<IO>(obs, t + static_cast<int64_t>(s) * p.ld, s, p);
          acc = fmaf(xv, xv, acc);
          const uint32_t h = ptx::to_tf32(xv);
          hi[e] = h;
          lo[e] = __float_as_uint(xv - __uint_as_float(h));
        }
        ptx::tmem_st8(tmem + lane_off + colXh + k8 * 8, hi);
        ptx::tmem_st8(tmem + lane_off + colXl + k8 * 8, lo);
      }
      xx = acc;
      ptx::tc_wait_st();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(x_ready);
    };

    uint32_t g = 0, tcount = 0;
    float xx_cur = 0.f, xx_next = 0.f;
    if (static_cast<int>(blockIdx.x) < n_tiles) prologue(blockIdx.x, xx_cur);
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++tcount) {
      const int64_t t = static_cast<int64_t>(tile) * kObsTile + row;
      const bool valid = t < p.N;
      for (int j = 0; j < p.m_tiles; ++j, ++g) {
        float v[MT];
        ptx::mbar_wait(acc_full, g & 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int c = 0; c < MT / 16; ++c) ptx::tmem_ld16(tmem + lane_off + colS + c * 16, &v[c * 16]);
        ptx::tc_wait_ld();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(acc_free);

        const float* dd = p.dd + static_cast<size_t>(j) * MT;
#pragma unroll
        for (int c = 0; c < MT; ++c) {
          const int mem = j * MT + c;
          const float ddc = __ldg(dd + c);
          const float base = xx_cur + ddc;
          float d2 = fmaf(-2.f, v[c], base);
          if (d2 < p.tau * base && valid && mem < p.m) {
            // direct difference (rare): cancellation-free d2
            float a = 0.f;
            for (int s = 0; s < p.n; ++s) {
              const float xv = load_norm<IO>(obs, t + static_cast<int64_t>(s) * p.ld, s, p);
              const float dv = __ldg(p.dn32 + static_cast<size_t>(mem) * p.n + s);
              const float d = xv - dv;
              a = fmaf(d, d, a);
            }
            d2 = a;
          }
          d2 = fmaxf(d2, 0.f);
          float sv;
          if (p.kind == CS_KERNEL_GAUSSIAN) {
            sv = exp2f(-d2 * p.g_coef);
          } else {
            const float r = d2 > 0.f ? d2 * rsqrtf(d2) : 0.f;
            sv = __fdividef(1.f, fmaf(r, p.inv_h, 1.f));
          }
          v[c] = mem < p.m ? sv : 0.f;
        }
        ptx::mbar_wait(s_free, (g & 1) ^ 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int c = 0; c < MT / 16; ++c) {
          uint32_t hi[16], lo[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float sv = v[c * 16 + e];
            const uint32_t h = ptx::to_tf32(sv);
            hi[e] = h;
            lo[e] = __float_as_uint(sv - __uint_as_float(h));
          }
          ptx::tmem_st16(tmem + lane_off + colSh + c * 16, hi);
          ptx::tmem_st16(tmem + lane_off + colSl + c * 16, lo);
        }
        ptx::tc_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(s_ready);
      }
      // next tile's x prologue overlaps this tile's last GEMM2
      const int next = tile + gridDim.x;
      if (next < n_tiles) prologue(next, xx_next);

      // readout: estimate = scale .* O, residual = x - estimate
      ptx::mbar_wait(o_full, tcount & 1);
      ptx::tc_fence_after();
      for (int c = 0; c < N2 / 16; ++c) {
        float o[16];
        ptx::tmem_ld16(tmem + lane_off + colO + c * 16, o);
        ptx::tc_wait_ld();
        if (valid) {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const int s = c * 16 + e;
            if (s < p.n) {
              const int64_t idx = t + static_cast<int64_t>(s) * p.ld;
              if constexpr (sizeof(IO) == 8) {
                const double ev = static_cast<double>(o[e]) * p.scale_d[s];
                if (est) est[idx] = ev;
                if (resid) resid[idx] = static_cast<double>(obs[idx]) - ev;
              } else {
                const float ev = o[e] * p.scale_f[s];
                if (est) est[idx] = ev;
                if (resid) resid[idx] = static_cast<float>(obs[idx]) - ev;
              }
            }
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(o_free);
      xx_cur = xx_next;
    }
  }
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kTmemCols);
  }
}

// ---------------------------------------------------------------------------
// Operand pre-tiling (once per model, at train time).  Canonical K-major,
// no-swizzle layout: element (r, k) of an R x K block sits at byte
//   (r%8)*16 + (r/8)*128 + (k%4)*4 + (k/4)*LBO,  LBO = (R/8)*128.
__device__ __forceinline__ size_t canon_off(int r, int k, int R) {
  return static_cast<size_t>((r & 7) * 4 + (r >> 3) * 32 + (k & 3) + (k >> 2) * (R / 8) * 32);
}

// D_norm^T tiles: block j holds memory vectors j*MT.. as rows, signals as K.
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
    const double v = (k < n && mem < m) ? Dn[k + static_cast<int64_t>(mem) * n] : 0.0;
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
