// sprt.cuh -- Wald SPRT alarm flags on residual streams.
//
// Not in the reference (SPEC.md:14 and :190 exclude anomaly decision logic);
// the definition is the project's own and oracle/cstress_oracle.c:or_sprt is
// its checker (parity against the reference: unpinned).  Per signal s, two
// one-sided mean tests with reset on either decision:
//   positive  lambda += c_s * (r - h_s)      negative  lambda += c_s * ((-r) - h_s)
//   lambda >= B: alarm (flag bit 0 / 1), lambda = 0;  lambda <= A: lambda = 0
// in FP64 with explicit round-to-nearest operations in exactly that order (no
// FMA contraction), so the flags are bit-identical to the sequential oracle.
//
// The recurrence is sequential in time; the GPU runs it in three passes:
//   1. speculative: every (signal, chunk of kSprtChunk steps) runs from
//      lambda = 0 (chunk 0 from the carried-in state, so it is exact) and
//      writes its flags and final state;
//   2. fix-up: one thread per signal walks the chunks in order; a chunk whose
//      true incoming state is (0, 0) was computed exactly, otherwise it is
//      re-run from the true state in lock-step with the speculative (from 0)
//      trajectory until the two coincide bit for bit -- after a common reset
//      they are identical -- which is typically a few reset cycles;
//   3. alarm counts per signal: word-wide reads of the flag bytes, popcounts
//      and a warp-shuffle reduction.
#pragma once

#include "common.cuh"

namespace csb {

constexpr int kSprtChunk = 256;

struct SprtStep {
  double c, h, A, B;
  // one step of both tests; returns the flag bits
  __device__ __forceinline__ uint8_t operator()(double r, double& lp, double& ln) const {
    uint8_t f = 0;
    lp = __dadd_rn(lp, __dmul_rn(c, __dsub_rn(r, h)));
    if (lp >= B) {
      f |= 1;
      lp = 0.0;
    } else if (lp <= A) {
      lp = 0.0;
    }
    ln = __dadd_rn(ln, __dmul_rn(c, __dsub_rn(-r, h)));
    if (ln >= B) {
      f |= 2;
      ln = 0.0;
    } else if (ln <= A) {
      ln = 0.0;
    }
    return f;
  }
};

template <typename IO>
__global__ void sprt_speculate_kernel(const IO* __restrict__ resid, int64_t N, int n, int64_t ld,
                                      const double* __restrict__ c, const double* __restrict__ h, double A,
                                      double B, const double* __restrict__ state, int chunks,
                                      uint8_t* __restrict__ flags, double* __restrict__ spec_final) {
  const int64_t total = static_cast<int64_t>(n) * chunks;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(e % chunks);
    const int s = static_cast<int>(e / chunks);
    const SprtStep step{c[s], h[s], A, B};
    double lp = k == 0 ? state[2 * s] : 0.0, ln = k == 0 ? state[2 * s + 1] : 0.0;
    const int64_t t0 = static_cast<int64_t>(k) * kSprtChunk;
    const int64_t t1 = min(N, t0 + kSprtChunk);
    const IO* r = resid + static_cast<int64_t>(s) * ld;
    uint8_t* f = flags + static_cast<int64_t>(s) * N;
    for (int64_t t = t0; t < t1; ++t) f[t] = step(static_cast<double>(__ldg(r + t)), lp, ln);
    spec_final[2 * e] = lp;
    spec_final[2 * e + 1] = ln;
  }
}

template <typename IO>
__global__ void sprt_fixup_kernel(const IO* __restrict__ resid, int64_t N, int n, int64_t ld,
                                  const double* __restrict__ c, const double* __restrict__ h, double A, double B,
                                  double* __restrict__ state, int chunks, uint8_t* __restrict__ flags,
                                  const double* __restrict__ spec_final) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const SprtStep step{c[s], h[s], A, B};
  const IO* r = resid + static_cast<int64_t>(s) * ld;
  uint8_t* f = flags + static_cast<int64_t>(s) * N;
  const double* spec = spec_final + static_cast<int64_t>(s) * chunks * 2;
  double tp = spec[0], tn = spec[1];  // chunk 0 ran from the true state
  for (int k = 1; k < chunks; ++k) {
    if (tp == 0.0 && tn == 0.0) {  // speculation was exact
      tp = spec[2 * k];
      tn = spec[2 * k + 1];
      continue;
    }
    double sp = 0.0, sn = 0.0;  // the speculative trajectory, recomputed
    const int64_t t0 = static_cast<int64_t>(k) * kSprtChunk;
    const int64_t t1 = min(N, t0 + kSprtChunk);
    bool merged = false;
    for (int64_t t = t0; t < t1; ++t) {
      const double x = static_cast<double>(r[t]);
      f[t] = step(x, tp, tn);
      step(x, sp, sn);
      if (tp == sp && tn == sn) {
        merged = true;
        break;
      }
    }
    if (merged) {
      tp = spec[2 * k];
      tn = spec[2 * k + 1];
    }
  }
  state[2 * s] = tp;
  state[2 * s + 1] = tn;
}

// alarm counts per signal: block per signal, warp-shuffle reduction
__global__ void sprt_count_kernel(const uint8_t* __restrict__ flags, int64_t N, int n,
                                  unsigned long long* __restrict__ counts) {
  __shared__ unsigned long long part[2][32];
  const int s = blockIdx.x;
  const uint8_t* f = flags + static_cast<int64_t>(s) * N;
  unsigned long long cp = 0, cn = 0;
  for (int64_t t = threadIdx.x; t < N; t += blockDim.x) {
    const uint8_t v = f[t];
    cp += v & 1;
    cn += (v >> 1) & 1;
  }
  for (int o = 16; o > 0; o >>= 1) {
    cp += __shfl_xor_sync(0xffffffffu, cp, o);
    cn += __shfl_xor_sync(0xffffffffu, cn, o);
  }
  if ((threadIdx.x & 31) == 0) {
    part[0][threadIdx.x >> 5] = cp;
    part[1][threadIdx.x >> 5] = cn;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int w = blockDim.x / 32;
    cp = threadIdx.x < w ? part[0][threadIdx.x] : 0;
    cn = threadIdx.x < w ? part[1][threadIdx.x] : 0;
    for (int o = 16; o > 0; o >>= 1) {
      cp += __shfl_xor_sync(0xffffffffu, cp, o);
      cn += __shfl_xor_sync(0xffffffffu, cn, o);
    }
    if (threadIdx.x == 0) {
      counts[2 * s] = cp;
      counts[2 * s + 1] = cn;
    }
  }
}

}  // namespace csb
