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
// The recurrence is sequential in time; the GPU runs it in two passes over
// the N x n column-major residuals (each signal contiguous in time):
//   1. speculate (HBM-bound): a CTA owns one signal and kSprtCta consecutive
//      chunks of kSprtChunk steps, one chunk per thread, every chunk started
//      from lambda = 0 (chunk 0 from the carried-in state, so it is exact).
//      The CTA stages kSprtSeg steps of all its chunks per round in shared
//      memory: the loads are lane-consecutive observations of one chunk
//      (128-byte lines, float4 / double2 vectors when the leading dimension
//      allows), the next round's tile is prefetched into registers while the
//      current one is evaluated, and the flag bytes go back through a
//      transposed shared tile as lane-consecutive (coalesced) 4-byte stores.
//      Then every chunk but the CTA's first ASSUMES that its predecessor's
//      speculative final state is its true incoming state (it is, whenever
//      the predecessor's own re-run merged -- nearly always) and re-runs
//      from it in lock-step with the from-0 trajectory until the two
//      coincide bit for bit (after a common reset they are identical;
//      typically a few steps), fixing its flags and counts.  It records the
//      merge step and its final state under that assumption.
//   2. walk (one warp per signal): chunk by chunk, the true incoming state
//      is compared with the one pass 1 assumed; where they agree (every
//      chunk up to the first that failed to merge, and every CTA-first chunk
//      whose true input is (0, 0)) pass 1's result stands; elsewhere the
//      chunk is re-run from the true state against both the assumed and the
//      from-0 trajectories, so the flags pass 1 wrote are replaced and the
//      counts corrected exactly.  Residuals arrive 32 at a time as one
//      coalesced warp load; per-chunk counts plus corrections reduce by warp
//      shuffles into the per-signal alarm counts -- flags are never re-read.
#pragma once

#include "common.cuh"

namespace csb {

#ifndef CSB_SPRT_MINB
#define CSB_SPRT_MINB 6  // resident speculate CTAs per SM (FP32 residuals)
#endif
constexpr int kSprtChunk = 2048;  // steps per speculative chunk
constexpr int kSprtSeg = 32;      // steps per staged round
constexpr int kSprtCta = 128;     // chunks (threads) per CTA

struct SprtStep {
  double c, h, A, B;
  // one step of both tests; returns the flag bits
  __device__ __forceinline__ uint32_t operator()(double r, double& lp, double& ln) const {
    lp = __dadd_rn(lp, __dmul_rn(c, __dsub_rn(r, h)));
    ln = __dadd_rn(ln, __dmul_rn(c, __dsub_rn(-r, h)));
    return decide(lp) | (decide(ln) << 1);
  }
  // the same step with the flag bits OR-ed straight into a packed word
  // (bit SHIFT: positive alarm, SHIFT + 1: negative) by predicated ORs --
  // the speculate pass's inner loop (no 0/1 select, shift and combine)
  template <int SHIFT>
  __device__ __forceinline__ void into(double r, double& lp, double& ln, uint32_t& word) const {
    lp = __dadd_rn(lp, __dmul_rn(c, __dsub_rn(r, h)));
    ln = __dadd_rn(ln, __dmul_rn(c, __dsub_rn(-r, h)));
    asm("{\n\t.reg .pred pa, pz;\n\t"
        "setp.ge.f64 pa, %0, %2;\n\t"
        "setp.le.or.f64 pz, %0, %3, pa;\n\t"
        "selp.f64 %0, 0d0000000000000000, %0, pz;\n\t"
        "@pa or.b32 %1, %1, %4;\n\t}"
        : "+d"(lp), "+r"(word)
        : "d"(B), "d"(A), "n"(1u << SHIFT));
    asm("{\n\t.reg .pred pa, pz;\n\t"
        "setp.ge.f64 pa, %0, %2;\n\t"
        "setp.le.or.f64 pz, %0, %3, pa;\n\t"
        "selp.f64 %0, 0d0000000000000000, %0, pz;\n\t"
        "@pa or.b32 %1, %1, %4;\n\t}"
        : "+d"(ln), "+r"(word)
        : "d"(B), "d"(A), "n"(1u << (SHIFT + 1)));
  }
  // lambda >= B: alarm and reset; lambda <= A: reset -- branch-free, the
  // reset predicate folded into the second compare (setp .or), so a
  // decision is two compares and one 64-bit select (NaN never decides,
  // exactly like the oracle's comparisons)
  __device__ __forceinline__ uint32_t decide(double& l) const {
    uint32_t f;
    asm("{\n\t.reg .pred pa, pz;\n\t"
        "setp.ge.f64 pa, %0, %2;\n\t"
        "setp.le.or.f64 pz, %0, %3, pa;\n\t"
        "selp.f64 %0, 0d0000000000000000, %0, pz;\n\t"
        "selp.u32 %1, 1, 0, pa;\n\t}"
        : "+d"(l), "=r"(f)
        : "d"(B), "d"(A));
    return f;
  }
};

template <typename IO>
struct SprtVec;  // the widest aligned vector of IO (16 bytes)
template <>
struct SprtVec<float> {
  using T = float4;
  static constexpr int k = 4;
};
template <>
struct SprtVec<double> {
  using T = double2;
  static constexpr int k = 2;
};

// Per-chunk record of pass 1 (one per (signal, chunk)).
struct SprtChunk {
  double spec_p, spec_n;    // final state of the from-0 (speculative) trajectory
  double fin_p, fin_n;      // final state under the assumed incoming state
  uint32_t counts;          // alarms under the assumption: positive | negative << 16
  uint32_t info;            // bit 0: re-run under an assumption; bit 1: merged; bits 2..: merge step
};

// Flag byte of step `t` (within a round-aligned word of 4) into a packed word.
__device__ __forceinline__ uint32_t sprt_pos_count(uint32_t w) { return __popc(w & 0x01010101u); }
__device__ __forceinline__ uint32_t sprt_neg_count(uint32_t w) { return __popc(w & 0x02020202u); }

// Re-run steps [t0, t1) of a residual column from the true state (tp, tn) in
// lock-step with trajectory (sp, sn) until they coincide bit for bit; writes
// the true flags and accumulates (true - other) alarm counts.  Returns the
// number of steps taken (t1 - t0 if they never met).  Scalar loads (a few
// steps per chunk, typically).
template <typename IO>
__device__ __forceinline__ int64_t sprt_rerun(const SprtStep& step, const IO* __restrict__ r, uint8_t* f,
                                              int64_t t0, int64_t t1, double& tp, double& tn, double& sp,
                                              double& sn, int& dp, int& dn) {
  for (int64_t t = t0; t < t1; ++t) {
    const double x = static_cast<double>(__ldg(r + t));
    const uint32_t fn = step(x, tp, tn);
    const uint32_t fo = step(x, sp, sn);
    f[t] = static_cast<uint8_t>(fn);
    dp += static_cast<int>(fn & 1) - static_cast<int>(fo & 1);
    dn += static_cast<int>(fn >> 1) - static_cast<int>(fo >> 1);
    if (tp == sp && tn == sn) return t + 1 - t0;
  }
  return t1 - t0;
}

// Pass 1.  grid (ceil(chunks / kSprtCta), n), block kSprtCta.  VEC: the
// residual column and its leading dimension are 16-byte aligned.
template <typename IO, bool VEC>
__global__ void __launch_bounds__(kSprtCta, sizeof(IO) == 4 ? CSB_SPRT_MINB : 4) sprt_speculate_kernel(
    const IO* __restrict__ resid, int64_t N, int64_t ld, const double* __restrict__ c,
    const double* __restrict__ h, double A, double B, const double* __restrict__ state, int chunks,
    uint8_t* __restrict__ flags, SprtChunk* __restrict__ rec) {
  using V = typename SprtVec<IO>::T;
  constexpr int kV = SprtVec<IO>::k;
  // rows padded to a 16-byte multiple (36 floats / 34 doubles): the staging
  // writes and the per-thread row reads are both 128-bit and conflict-free
  // (per 8-lane phase the rows start 4 banks apart)
  constexpr int kRow = kSprtSeg + 16 / static_cast<int>(sizeof(IO));
  __shared__ __align__(16) IO rs[kSprtCta][kRow];
  __shared__ uint32_t fw[kSprtCta][kSprtSeg / 4 + 1];
  __shared__ double sfin[kSprtCta][2];
  const int s = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int chunk0 = blockIdx.x * kSprtCta;
  const int k = chunk0 + tid;
  const int n_here = min(kSprtCta, chunks - chunk0);  // chunks in this CTA
  const SprtStep step{c[s], h[s], A, B};
  const IO* r = resid + static_cast<int64_t>(s) * ld;
  uint8_t* f = flags + static_cast<int64_t>(s) * N;
  double lp = k == 0 ? state[2 * s] : 0.0, ln = k == 0 ? state[2 * s + 1] : 0.0;
  uint32_t cp = 0, cn = 0;
  // this CTA's region of the column: <= kSprtCta * kSprtChunk steps, so all
  // offsets below are 32-bit
  const int64_t cta_start = static_cast<int64_t>(chunk0) * kSprtChunk;
  const IO* rc = r + cta_start;
  uint8_t* fc = f + cta_start;
  const int rem = static_cast<int>(min(N - cta_start, static_cast<int64_t>(kSprtCta) * kSprtChunk));
  const int my0 = tid * kSprtChunk;
  const int my_end = min(rem, my0 + kSprtChunk);

  // Staged tile of a round: kSprtCta segments (one per chunk) of kSprtSeg
  // consecutive steps.  VEC: thread `tid` loads vector tid % kLanesPerSeg of
  // segments tid / kLanesPerSeg + j * kSegsPerPass; otherwise element `lane`
  // of segments warp + j * kWarps.  Either way a warp instruction reads whole
  // 128-byte lines of lane-consecutive observations.
  constexpr int kLanesPerSeg = kSprtSeg / kV;             // vectors per segment
  constexpr int kSegsPerPass = kSprtCta / kLanesPerSeg;   // segments one pass of the CTA covers
  constexpr int kVecLoads = kSprtCta / kSegsPerPass;      // passes per round (VEC)
  constexpr int kWarps = kSprtCta / 32;
  constexpr int kScalarLoads = kSprtCta / kWarps;         // segments per warp per round (scalar)
  V prev[VEC ? kVecLoads : 1];
  IO pres[VEC ? 1 : kScalarLoads];

  auto load_round = [&](int round) {
    const int off = round * kSprtSeg;
    if constexpr (VEC) {
#pragma unroll
      for (int j = 0; j < kVecLoads; ++j) {
        const int o = (tid / kLanesPerSeg + j * kSegsPerPass) * kSprtChunk + off + (tid % kLanesPerSeg) * kV;
        if (o + kV <= rem) {
          prev[j] = __ldg(reinterpret_cast<const V*>(rc + o));
        } else {
          IO* e = reinterpret_cast<IO*>(&prev[j]);
#pragma unroll
          for (int q = 0; q < kV; ++q) e[q] = o + q < rem ? __ldg(rc + o + q) : IO(0);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < kScalarLoads; ++j) {
        const int o = (warp + j * kWarps) * kSprtChunk + off + lane;
        pres[j] = o < rem ? __ldg(rc + o) : IO(0);
      }
    }
  };
  auto stage_round = [&]() {
    if constexpr (VEC) {
#pragma unroll
      for (int j = 0; j < kVecLoads; ++j)
        *reinterpret_cast<V*>(&rs[tid / kLanesPerSeg + j * kSegsPerPass][(tid % kLanesPerSeg) * kV]) = prev[j];
    } else {
#pragma unroll
      for (int j = 0; j < kScalarLoads; ++j) rs[warp + j * kWarps][lane] = pres[j];
    }
  };
  // four steps of this thread's row -> one packed flag word
  auto four = [&](int w, int valid) -> uint32_t {
    IO x[4];
    if constexpr (sizeof(IO) == 4) {
      const float4 v = *reinterpret_cast<const float4*>(&rs[tid][4 * w]);
      x[0] = v.x, x[1] = v.y, x[2] = v.z, x[3] = v.w;
    } else {
      const double2 v0 = *reinterpret_cast<const double2*>(&rs[tid][4 * w]);
      const double2 v1 = *reinterpret_cast<const double2*>(&rs[tid][4 * w + 2]);
      x[0] = v0.x, x[1] = v0.y, x[2] = v1.x, x[3] = v1.y;
    }
    uint32_t word = 0;
    if (valid == 4) {
      step.into<0>(static_cast<double>(x[0]), lp, ln, word);
      step.into<8>(static_cast<double>(x[1]), lp, ln, word);
      step.into<16>(static_cast<double>(x[2]), lp, ln, word);
      step.into<24>(static_cast<double>(x[3]), lp, ln, word);
    } else {
      if (valid > 0) step.into<0>(static_cast<double>(x[0]), lp, ln, word);
      if (valid > 1) step.into<8>(static_cast<double>(x[1]), lp, ln, word);
      if (valid > 2) step.into<16>(static_cast<double>(x[2]), lp, ln, word);
    }
    return word;
  };

  const int rounds = (min(rem, kSprtChunk) + kSprtSeg - 1) / kSprtSeg;
  const bool words_ok = (reinterpret_cast<uintptr_t>(f) & 3) == 0;
  load_round(0);
  for (int round = 0; round < rounds; ++round) {
    stage_round();
    __syncthreads();
    if (round + 1 < rounds) load_round(round + 1);  // in flight while this round is evaluated
    const int off = round * kSprtSeg;
    if (tid < n_here) {
      const int t0 = my0 + off;
      if (t0 + kSprtSeg <= my_end) {  // full round: no bounds checks
#pragma unroll
        for (int w = 0; w < kSprtSeg / 4; ++w) {
          const uint32_t word = four(w, 4);
          fw[tid][w] = word;
          cp += sprt_pos_count(word);
          cn += sprt_neg_count(word);
        }
      } else {
        for (int w = 0; w < kSprtSeg / 4; ++w) {
          const uint32_t word = four(w, max(0, min(4, my_end - (t0 + 4 * w))));
          fw[tid][w] = word;
          cp += sprt_pos_count(word);
          cn += sprt_neg_count(word);
        }
      }
    }
    __syncthreads();
    // flags back out, lane-consecutive: a warp writes 4 segments (8 words
    // each) per instruction; byte stores where the column is not 4-aligned
#pragma unroll
    for (int it = 0; it < kSprtCta / (4 * kWarps); ++it) {
      const int seg = (it * kWarps + warp) * 4 + (lane >> 3), w = lane & 7;
      if (seg >= n_here) break;
      const int o = seg * kSprtChunk + off + 4 * w;
      const uint32_t word = fw[seg][w];
      if (words_ok && o + 4 <= rem) {
        *reinterpret_cast<uint32_t*>(fc + o) = word;
      } else {
        for (int q = 0; q < 4; ++q)
          if (o + q < rem) fc[o + q] = static_cast<uint8_t>(word >> (8 * q));
      }
    }
  }
  const int64_t start = cta_start + my0;
  const int64_t chunk_end = cta_start + my_end;
  // ---- assumed-input re-run (chunks 1.. of the CTA): the predecessor's
  // speculative final state is taken as this chunk's incoming state
  sfin[tid][0] = lp;
  sfin[tid][1] = ln;
  __syncthreads();
  if (tid >= n_here) return;
  const double sp_fin = lp, sn_fin = ln;
  uint32_t info = 0;
  int dp = 0, dn = 0;
  if (tid > 0) {
    double tp = sfin[tid - 1][0], tn = sfin[tid - 1][1];
    if (!(tp == 0.0 && tn == 0.0)) {
      double sp = 0.0, sn = 0.0;
      const int64_t steps = sprt_rerun(step, r, f, start, chunk_end, tp, tn, sp, sn, dp, dn);
      const bool merged = tp == sp && tn == sn;
      info = 1u | (merged ? 2u : 0u) | (static_cast<uint32_t>(steps) << 2);
      if (!merged) {  // the assumed trajectory's own final state
        lp = tp;
        ln = tn;
      }
    }
  }
  SprtChunk& out = rec[static_cast<int64_t>(s) * chunks + k];
  out.spec_p = sp_fin;
  out.spec_n = sn_fin;
  out.fin_p = lp;
  out.fin_n = ln;
  out.counts = static_cast<uint32_t>(static_cast<int>(cp) + dp) | (static_cast<uint32_t>(static_cast<int>(cn) + dn) << 16);
  out.info = info;
}

// Pass 2.  One warp per signal (block 128 = 4 signals).
template <typename IO>
__global__ void __launch_bounds__(128) sprt_fixup_kernel(
    const IO* __restrict__ resid, int64_t N, int n, int64_t ld, const double* __restrict__ c,
    const double* __restrict__ h, double A, double B, double* __restrict__ state, int chunks,
    uint8_t* __restrict__ flags, const SprtChunk* __restrict__ rec, unsigned long long* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int s = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (s >= n) return;
  const SprtStep step{c[s], h[s], A, B};
  const IO* r = resid + static_cast<int64_t>(s) * ld;
  uint8_t* f = flags + static_cast<int64_t>(s) * N;
  const SprtChunk* cr = rec + static_cast<int64_t>(s) * chunks;
  long long cp = 0, cn = 0;  // pass-1 counts of every chunk, corrected below where a chunk is re-run
  for (int k = lane; k < chunks; k += 32) {
    cp += cr[k].counts & 0xffffu;
    cn += cr[k].counts >> 16;
  }
  double tp = cr[0].fin_p, tn = cr[0].fin_n;  // chunk 0 ran from the true state
  for (int kb = 1; kb < chunks; kb += 32) {
    // lane j holds chunk kb + j's record and its predecessor's speculative final
    const int kl = kb + lane;
    SprtChunk mine{};
    double prev_p = 0.0, prev_n = 0.0;
    if (kl < chunks) {
      mine = cr[kl];
      prev_p = cr[kl - 1].spec_p;
      prev_n = cr[kl - 1].spec_n;
    }
    const int nb = min(32, chunks - kb);
    for (int j = 0; j < nb; ++j) {
      const int k = kb + j;
      const uint32_t info = __shfl_sync(0xffffffffu, mine.info, j);
      // the incoming state pass 1 assumed: the predecessor's speculative
      // final (re-run chunks) or (0, 0) (CTA-first chunks and chunks whose
      // assumed input was (0, 0) -- the from-0 run is then exact for it)
      double ap = 0.0, an = 0.0;
      if (k % kSprtCta != 0) {
        ap = __shfl_sync(0xffffffffu, prev_p, j);
        an = __shfl_sync(0xffffffffu, prev_n, j);
      }
      if (tp == ap && tn == an) {  // pass 1 ran this chunk from its true state
        tp = __shfl_sync(0xffffffffu, mine.fin_p, j);
        tn = __shfl_sync(0xffffffffu, mine.fin_n, j);
        continue;
      }
      // Re-run from the true state beside the assumed (what pass 1 wrote up
      // to its merge step) and the from-0 trajectory (what stands after it).
      const int64_t t0 = static_cast<int64_t>(k) * kSprtChunk;
      const int64_t t1 = min(N, t0 + kSprtChunk);
      const int64_t p_end = (info & 1u) ? t0 + (info >> 2) : t0;  // steps pass 1 rewrote
      double sp = 0.0, sn = 0.0;
      bool merged = false;
      for (int64_t base = t0; base < t1 && !(merged && base >= p_end); base += 32) {
        const IO x_lane = (base + lane < t1) ? __ldg(r + base + lane) : IO(0);
        const int steps = t1 - base < 32 ? static_cast<int>(t1 - base) : 32;
        uint32_t mine_new = 0, mine_old = 0;
        int done = steps;
        for (int q = 0; q < steps; ++q) {
          const double x = static_cast<double>(__shfl_sync(0xffffffffu, x_lane, q));
          const uint32_t fn = step(x, tp, tn);
          const uint32_t fs = step(x, sp, sn);
          const uint32_t fa = step(x, ap, an);
          const uint32_t fold = (base + q < p_end) ? fa : fs;  // the byte pass 1 left
          if (lane == q) {
            mine_new = fn;
            mine_old = fold;
          }
          merged = merged || (tp == sp && tn == sn);
          if (merged && base + q + 1 >= p_end) {
            done = q + 1;
            break;
          }
        }
        if (lane < done) {
          f[base + lane] = static_cast<uint8_t>(mine_new);
          cp += static_cast<long long>(mine_new & 1) - static_cast<long long>(mine_old & 1);
          cn += static_cast<long long>(mine_new >> 1) - static_cast<long long>(mine_old >> 1);
        }
      }
      if (merged) {
        tp = __shfl_sync(0xffffffffu, mine.spec_p, j);
        tn = __shfl_sync(0xffffffffu, mine.spec_n, j);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    cp += __shfl_xor_sync(0xffffffffu, cp, o);
    cn += __shfl_xor_sync(0xffffffffu, cn, o);
  }
  if (lane == 0) {
    state[2 * s] = tp;
    state[2 * s + 1] = tn;
    counts[2 * s] = static_cast<unsigned long long>(cp);
    counts[2 * s + 1] = static_cast<unsigned long long>(cn);
  }
}

}  // namespace csb
