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
// streams the memory matrix in MT-wide tiles ("steps").  Warp roles:
//   warps 0, 1   producers: 1D bulk copies (TMA engine) of the pre-tiled
//                D_norm^T (warp 0) and P^T (warp 1) operand tiles into
//                n_stages-deep shared-memory rings
//   warps 2, 3   MMA issuers (one thread each): tcgen05.mma kind::f16, GEMM1
//                (warp 2) one or two steps ahead of GEMM2 (warp 3).
//   warps 4..    epilogue (16, or 8, see tc_epi_warps): two sets; set e owns the steps with
//                j % 2 == e (and TMEM buffer e), each warp a 32-lane quarter
//                and half of the MT columns.  All 16 warps share the x
//                prologue and the final estimate / residual readout.
// TMEM (512 columns x 128 lanes, lane = observation):
//   O   [N2]            S P^T accumulator                 (GEMM2 D)
//   X   [K1]            x_norm hi | lo, f16x2 pairs       (GEMM1 A, "TS" form)
//   ACC [NB x MT]       X D_norm accumulators             (GEMM1 D)
//   S   [SB x MT]       2^14 S hi | lo, f16x2 pairs       (GEMM2 A, "TS" form)
// FP32-accurate products on FP16 tensor cores: every operand v is split into
// hi = rn_f16(v), lo = rn_f16(v - hi) and each GEMM issues hi*hi + hi*lo +
// lo*hi (3xFP16, exact power-of-two operand scales, pack_tc.cuh).  A single
// 10-bit-mantissa pass misses the 1e-3 tolerance.  Rows holding a
// value outside the split's safe range (|x_norm| >= 2^15) are flagged in the
// prologue and recomputed by direct difference.
// d2 in GEMM form cancels near zero; entries with d2 < tau (|x|^2+|d|^2) are
// recomputed by direct difference, which keeps memory vectors
// reproducing themselves.
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "pack_tc.cuh"
#include "sm100_ptx.cuh"

namespace csb {

// Epilogue warps per TMEM plan: 16 (two sets of 8 with NB = 2), or 8 for
// double-ACC single-S plans (sets of 4, each warp a whole step's columns for
// its lane quarter).  8 leave 168 registers per thread instead of 96 (the
// register file is split over the four SMSPs, and 20 warps put five on one
// of them); measured: 12% faster with (64,2,1) at n = 128, 9% slower with
// (64,2,2) at C2 (fewer warps to hide the kernel map's latency).
// CSB_EPI_WARPS=8|16 forces one count for every plan (A/B builds).
__host__ __device__ constexpr int tc_epi_warps(int NB, int SB) {
#ifdef CSB_EPI_WARPS
  return CSB_EPI_WARPS + 0 * (NB + SB);
#else
  return (NB == 2 && SB == 1) ? 8 : 16;
#endif
}
__host__ __device__ constexpr int tc_threads(int NB, int SB) {
  return 128 + 32 * tc_epi_warps(NB, SB);  // 2 producers, 2 MMA issuers, epilogue
}
constexpr int kObsTile = 128;
constexpr int kTmemCols = 512;
constexpr int kMaxStages = 4;

struct TcParams {
  const void* obs;  // N x n, leading dim ld, IO type
  int64_t N, ld;
  int n, K1, N2, m, m_tiles;
  int n_stages;
  const __half* dn_tiles; // m_tiles x [hi | lo] (MT x K1 canonical K-major, FP16)
  const __half* p_tiles;  // m_tiles x [hi | lo] (N2 x MT canonical K-major, FP16)
  const float* dd;        // m_tiles*MT squared norms of D_norm columns (0 padded)
  const float* dn32;      // n x m D_norm in FP32 (direct-difference recompute)
  const float* inv_scale; // n
  const float* scale_f;   // n  estimate multipliers scale_s * 2^(k_s - 14)
  const double* scale_d;  // n  (FP64 copy of the same)
  const double* norm_d;   // n  signal scales (x / scale normalisation, FP64 I/O)
  float aug_x;            // value of x's ||d||^2 column (1 / the column's scale)
  int kind;
  float inv_h;   // 1/h            (inverse distance)
  float g_coef;  // log2(e)/(2h^2) (gaussian)
  float tau;     // near-zero recompute threshold
  float dd_max;  // max ||d_i||^2: per-row prefilter bound for the guard
  void* est;
  void* resid;
  uint32_t dn_stage_bytes, p_stage_bytes;
  unsigned long long* timeline;  // CSB_TIMELINE builds only: per-warp event records
  // staged tile edge (FP32 I/O when shared memory allows): a [2][n][128]
  // FP32 staging area, halves A and B.  During tile k TMA loads x(k + 1)
  // into A (for the next prologue) and x(k) into B (for this readout); at
  // the edge the prologue reads A, the readout reads B, writes the residuals
  // over B and the estimates over A, and two TMA tensor stores write them
  // back asynchronously.  No global loads or stores at the tile edge: with
  // per-thread loads the x prologue and readout each waited ~6k cycles on
  // spilled load batches.
  int staged;
  int split_edge;          // staged, NB = 2: split the tile edge between the step sets
  uint32_t stage_out_off;  // byte offset of the staging area
  CUtensorMap tmap_obs, tmap_est, tmap_res;
};

// Development instrumentation (tools/timeline.py): with -DCSB_TIMELINE the
// producer, MMA and two epilogue warps of CTA 0 record (event, step, clock64)
// triples; compiled out otherwise.
#ifdef CSB_TIMELINE
constexpr int kTlCap = 8192;
// one recording thread per slot keeps its record count in a register (tl_n):
// a counter in global memory cost a dependent L2 round trip per event and
// distorted the short phases being measured
#define CSB_TL(slot, ev, j)                                                                   \
  do {                                                                                      \
    if (blockIdx.x == 0 && lane == 0 && p.timeline && tl_n + 1 < kTlCap) {                  \
      unsigned long long* tl_ = p.timeline + (slot) * kTlCap * 2;                             \
      tl_[2 + 2 * tl_n] = (static_cast<unsigned long long>(ev) << 32) | static_cast<unsigned>(j); \
      tl_[3 + 2 * tl_n] = clock64();                                                        \
      tl_[0] = ++tl_n;                                                                      \
    }                                                                                       \
  } while (0)
#else
#define CSB_TL(slot, ev, j) \
  do {                      \
  } while (0)
#endif

// TMEM columns used for a given shape, ACC buffer count NB and S buffer
// count SB (each 1 or 2, SB <= NB).
__host__ __device__ constexpr int tc_tmem_cols(int N2, int K1, int MT, int NB, int SB) {
  return (N2 + 15) / 16 * 16 + K1 + NB * MT + SB * MT;  // X and S as f16x2 hi | lo pairs
}

// Shared-memory footprint of everything but the operand rings: barriers,
// staged scales and the per-row ||x||^2 partials.
__host__ __device__ constexpr size_t tc_aux_bytes(int K1) {
  return 512 + static_cast<size_t>(K1) * (4 + 4 + 8 + 8) + 2 * 4 * kObsTile * 4 + 2 * 4 * kObsTile +
         2 * kObsTile * 4 + 2 * kObsTile;
}

// Development switches (A/B builds): how many of every four reciprocals of the
// inverse-distance map go to MUFU (the rest run as FMA-pipe Newton
// iterations), and which roles suspend in their mbarrier waits (0 none,
// 1 epilogue, 2 every role; measured: 0 is as fast at C2 and 9% faster at
// n = 20).
#ifndef CSB_RCP_MUFU
#define CSB_RCP_MUFU 4  // measured (C2, n=100/m=4000): 4 beats 2 by 3-8%, n=64 within 1.5%
#endif
// staged readout: 8-column O chunks read per TMEM load wait
#ifndef CSB_G1_2X
#define CSB_G1_2X 0  // 1: GEMM1 without the x_hi * D_lo product (D_norm at FP16 precision; A/B only)
#endif
#ifndef CSB_MAP2
#define CSB_MAP2 0  // 1: kernel map and S split on packed FP32 pairs (FFMA2 / FADD2)
#endif
#ifndef CSB_RD_BATCH
#define CSB_RD_BATCH 2
#endif
#ifndef CSB_WAIT_SLEEP
#define CSB_WAIT_SLEEP 0
#endif

// ring position: (index, phase) advanced in issue order
struct Ring {
  uint32_t idx = 0, phase = 0, n = 1;
  __device__ explicit Ring(uint32_t n_) : n(n_) {}
  __device__ void next() {
    if (++idx == n) {
      idx = 0;
      phase ^= 1;
    }
  }
};

// NB = 2: double-buffered ACC, two epilogue sets alternate steps, GEMM1 two
//         steps ahead; SB = 2 also double-buffers S, SB = 1 shares one S
//         buffer between the sets (GEMM1 still never waits for the
//         similarity epilogue).  NB = 1: single buffers, all 16 epilogue
//         warps work on every step (4 column groups), GEMM1 one step ahead.
template <int MT, int NB, int SB, typename IO, bool STAGED>
__global__ void __launch_bounds__(tc_threads(NB, SB), 1) mset_estimate_tc_kernel(const __grid_constant__ TcParams p) {
  static_assert(NB == 1 || NB == 2, "one or two TMEM buffers");
  static_assert(SB >= 1 && SB <= NB, "S buffers");
  static_assert(!STAGED || sizeof(IO) == 4, "staged tile edge: FP32 I/O");
  // Staged, two step sets, p.split_edge: the tile edge is split between the
  // sets -- the set that does not own the last step stages the next tile's x
  // (it is done with the tile first), the other reads O out; see the epilogue.
  const bool kSplitEdge = STAGED && NB == 2 && p.split_edge;
  constexpr int kEpiWarps = tc_epi_warps(NB, SB);
  static_assert(kEpiWarps == 8 || kEpiWarps == 16, "8 or 16 epilogue warps");
  constexpr int kSetWarps = kEpiWarps / NB;      // warps per step set
  constexpr int COLS = MT * 4 / kSetWarps;       // columns per epilogue warp
  constexpr int CH = COLS % 16 == 0 ? 16 : 8;    // TMEM access chunk
  static_assert(COLS % 8 == 0, "epilogue column slice must be a multiple of 8");
  extern __shared__ __align__(1024) uint8_t smem[];
  // warp index via shfl: the compiler then knows every role branch is
  // warp-uniform and keeps the MMA issue loop on the uniform datapath
  const int warp = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x) / 32, 0);
  const int lane = threadIdx.x % 32;
  const int NS = p.n_stages;
#ifdef CSB_TIMELINE
  int tl_n = 0;  // timeline records written by this thread
#endif
  constexpr int io_bytes = sizeof(IO);
  uint8_t* dn_ring = smem;
  uint8_t* p_ring = smem + NS * p.dn_stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(p_ring + NS * p.p_stage_bytes);
  uint64_t* dn_full = bars + 0;    // [4]
  uint64_t* dn_empty = bars + 4;   // [4]
  uint64_t* p_full = bars + 8;     // [4]
  uint64_t* p_empty = bars + 12;   // [4]
  uint64_t* acc_full = bars + 16;  // [2]
  uint64_t* acc_free = bars + 18;  // [2]
  uint64_t* s_ready = bars + 20;   // [2]
  uint64_t* s_free = bars + 22;    // [2]
  uint64_t* x_ready = bars + 24;
  uint64_t* x_free = bars + 25;
  uint64_t* o_full = bars + 26;
  uint64_t* o_free = bars + 27;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 28);
  uint64_t* xa_full = bars + 29;  // staged: x of the next tile in staging half A
  uint64_t* xb_full = bars + 30;  // staged: x of this tile in staging half B
  uint64_t* a_done = bars + 31;   // split edge: prologue done with half A, ||x||^2 posted
  uint64_t* g2_last = bars + 32;  // GEMM2 of a tile's last step has been issued
  double* s_inv_d = reinterpret_cast<double*>(bars + 64);
  double* s_scale_d = s_inv_d + p.K1;
  float* s_inv_f = reinterpret_cast<float*>(s_scale_d + p.K1);
  float* s_scale_f = s_inv_f + p.K1;
  float* s_xx = s_scale_f + p.K1;  // [2][4][kObsTile] ||x||^2 partials (by tile parity)
  uint8_t* s_bad = reinterpret_cast<uint8_t*>(s_xx + 2 * 4 * kObsTile);  // [2][4][kObsTile] out-of-range flags
  float* s_xx_tot = reinterpret_cast<float*>(s_bad + 2 * 4 * kObsTile);  // [2][kObsTile] split edge: ||x||^2 per row
  uint8_t* s_bad_tot = reinterpret_cast<uint8_t*>(s_xx_tot + 2 * kObsTile);  // [2][kObsTile]

  // Thread-block cluster of CL CTAs (CL = 1 without a cluster launch): the
  // operand tiles are identical for every CTA, so each CTA's producer copies
  // a 1/CL slice of each stage and multicasts it into every CTA of the
  // cluster (L2 -> SM operand traffic / CL: with one copy per CTA the 148
  // SMs streaming the same tiles out of L2 bounded the step time); a ring
  // slot is refilled once the MMAs of every CTA have released it.
  const uint32_t CL = ptx::cluster_nctarank();
  const uint32_t cl_rank = CL > 1 ? ptx::cluster_ctarank() : 0;
  const uint16_t cl_mask = static_cast<uint16_t>((1u << CL) - 1);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) ptx::mbar_init(&bars[i], (i & 4) ? CL : 1);  // [4..7], [12..15]: empty
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&acc_full[b], 1);
      ptx::mbar_init(&acc_free[b], kSetWarps);
      ptx::mbar_init(&s_ready[b], kSetWarps);
      ptx::mbar_init(&s_free[b], 1);
    }
    ptx::mbar_init(x_ready, kSplitEdge ? kSetWarps : kEpiWarps);
    ptx::mbar_init(x_free, 1);
    ptx::mbar_init(o_full, 1);
    ptx::mbar_init(xa_full, 1);
    ptx::mbar_init(xb_full, 1);
    ptx::mbar_init(o_free, kSplitEdge ? kSetWarps : kEpiWarps);
    ptx::mbar_init(a_done, 4);
    ptx::mbar_init(g2_last, 1);
    ptx::fence_mbar_init();
  }
  for (int s = threadIdx.x; s < p.K1; s += blockDim.x) {
    const bool ok = s < p.n;
    s_inv_d[s] = ok ? 1.0 / p.norm_d[s] : 0.0;
    s_scale_d[s] = ok ? p.scale_d[s] : 0.0;
    s_inv_f[s] = ok ? p.inv_scale[s] : 0.f;
    s_scale_f[s] = ok ? p.scale_f[s] : 0.f;
  }
  if (warp == 0) ptx::tmem_alloc(tmem_holder, kTmemCols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  // The CTA owns all 512 TMEM columns (1 CTA/SM), so the allocation always
  // starts at lane 0, column 0.  Using the constant (checked) keeps every
  // TMEM operand of the MMA issue loop in uniform registers; an address
  // loaded from shared memory is per-thread to the compiler and turns each
  // tcgen05.mma into an R2UR/VOTEU waterfall.
  if (*tmem_holder != 0u) __trap();
  constexpr uint32_t tmem = 0;
  if (CL > 1) ptx::cluster_sync();  // peers' barriers initialised before any multicast

  auto rwait = [](uint64_t* bar, uint32_t parity) {  // producer / MMA waits
    if constexpr (CSB_WAIT_SLEEP >= 2) {
      ptx::mbar_wait_sleep(bar, parity);
    } else {
      ptx::mbar_wait(bar, parity);
    }
  };
  const int K1 = p.K1, N2 = p.N2;
  const uint32_t colO = 0;
  // O's TMEM columns are kept at a multiple of 16 (GEMM2's N = N2 may be a
  // multiple of 8 only: tcgen05 N steps by 8 for M = 128)
  const uint32_t colXh = (N2 + 15) / 16 * 16, colXl = colXh + K1 / 2;
  const uint32_t colAcc = colXh + K1;      // + b*MT
  const uint32_t colS = colAcc + NB * MT;  // + b*MT (hi), + MT/2 (lo)
  const int n_tiles = static_cast<int>((p.N + kObsTile - 1) / kObsTile);
  const int T = p.m_tiles;
  // tile slots: every CTA of a cluster runs as many as the cluster's first
  // CTA (the operand rings are shared); slots past the last tile are dummies
  // with no valid rows.  Slot k of this CTA is tile blockIdx.x + k * grid.
  const int cl_base = static_cast<int>(blockIdx.x - cl_rank);
  const int n_iter = cl_base < n_tiles ? (n_tiles - cl_base + static_cast<int>(gridDim.x) - 1) / gridDim.x : 0;
  const int tile_end = static_cast<int>(blockIdx.x) + n_iter * static_cast<int>(gridDim.x);  // loop bound

  if (warp <= 1) {
    // ----------------------------------------------------------- producers
    // (whole warp, converged; one elected lane issues).  Warp 0 streams the
    // D_norm^T ring, warp 1 the P^T ring: with one producer for both, the
    // D tile for GEMM1(j + 1) queued behind the wait for a free P slot, i.e.
    // behind GEMM2(j - 1) and hence the similarity epilogue, and GEMM1
    // starved (tools/timeline.py).
    {
      const bool dn = warp == 0;
      uint64_t* full = dn ? dn_full : p_full;
      uint64_t* empty = dn ? dn_empty : p_empty;
      uint8_t* ring = dn ? dn_ring : p_ring;
      const uint8_t* src = reinterpret_cast<const uint8_t*>(dn ? static_cast<const void*>(p.dn_tiles)
                                                               : static_cast<const void*>(p.p_tiles));
      const uint32_t bytes = dn ? p.dn_stage_bytes : p.p_stage_bytes;
      Ring r(NS);
      for (int tile = blockIdx.x; tile < tile_end; tile += gridDim.x) {
        // warm L2 with the next tile's observations (one 128-row segment per
        // signal column): the x prologue then reads L2, not a DRAM burst
        // that every CTA issues at the same moment.  Issued at the start of
        // the tile: the bulk prefetches share the TMA engine with the operand
        // copies, and issuing them mid-tile (or re-warming this tile's rows
        // for the readout) measured 17% slower.
        auto prefetch_tile = [&](int pt) {
          if (pt >= n_tiles) return;
          const int64_t t0 = static_cast<int64_t>(pt) * kObsTile;
          const int64_t rows = min(static_cast<int64_t>(kObsTile), p.N - t0);
          const uintptr_t base = reinterpret_cast<uintptr_t>(p.obs);
          for (int s = lane; s < p.n; s += 32) {
            const uintptr_t a = base + static_cast<uintptr_t>(t0 + static_cast<int64_t>(s) * p.ld) * io_bytes;
            const uintptr_t a0 = a & ~uintptr_t{15}, a1 = (a + rows * io_bytes) & ~uintptr_t{15};
            if (a1 > a0) ptx::prefetch_l2(reinterpret_cast<const void*>(a0), static_cast<uint32_t>(a1 - a0));
          }
        };
        if (!dn && !STAGED) prefetch_tile(tile + gridDim.x);  // staged tiles arrive by TMA
        for (int j = 0; j < T; ++j, r.next()) {
          if (dn) CSB_TL(0, 30, j);
          rwait(&empty[r.idx], r.phase ^ 1);
          if (dn) CSB_TL(0, 31, j);
          ptx::mbar_arrive_expect_tx_elect(&full[r.idx], bytes);
          if (CL > 1) {
            const uint32_t slice = bytes / CL;
            ptx::bulk_g2s_multicast_elect(ring + r.idx * bytes + cl_rank * slice,
                                          src + static_cast<size_t>(j) * bytes + cl_rank * slice, slice,
                                          &full[r.idx], cl_mask);
          } else {
            ptx::bulk_g2s_elect(ring + r.idx * bytes, src + static_cast<size_t>(j) * bytes, bytes, &full[r.idx]);
          }
        }
      }
    }
  } else if (warp == 2 || warp == 3) {
    // ---------------------------------------------------------- MMA issuer
    // (whole warp, converged, warp-uniform operands; one elected lane issues)
    {
      const uint32_t idesc1 = ptx::idesc_f16(128, MT);
      const uint32_t idesc2 = ptx::idesc_f16(128, N2);
      const uint32_t SBO = 128;
      const uint32_t LBO1 = (MT / 8) * 128;  // D_norm^T tile: MT rows x K1
      const uint32_t LBO2 = (N2 / 8) * 128;  // P^T tile: N2 rows x MT
      const uint64_t dn_desc0 = ptx::smem_desc(ptx::smem_u32(dn_ring), LBO1, SBO);
      const uint64_t p_desc0 = ptx::smem_desc(ptx::smem_u32(p_ring), LBO2, SBO);
      const uint64_t dn_lo_off = (static_cast<uint64_t>(MT) * K1 * 2) >> 4;
      const uint64_t p_lo_off = (static_cast<uint64_t>(N2) * MT * 2) >> 4;
      const uint64_t dn_stage_off = p.dn_stage_bytes >> 4, p_stage_off = p.p_stage_bytes >> 4;
      const uint64_t k_step1 = (2 * LBO1) >> 4, k_step2 = (2 * LBO2) >> 4;
      const uint32_t dO = tmem + colO;
      Ring rd(NS), rp(NS);
      uint32_t acc_use[2] = {0, 0}, s_use[2] = {0, 0};
      uint32_t tcount1 = 0, tcount2 = 0;

      auto issue_g1 = [&](int j) {
        const int b = NB == 2 ? (j & 1) : 0;
        CSB_TL(1, 1, j);
        if (j == 0) {
          rwait(x_ready, tcount1 & 1);
          // the tensor pipe runs MMAs in issue order: the next tile's GEMM1
          // goes after this tile's last GEMM2, whose completion (o_full)
          // starts the readout on the critical path
          if (tcount1 > 0) rwait(g2_last, (tcount1 - 1) & 1);
        }
        rwait(&dn_full[rd.idx], rd.phase);
        rwait(&acc_free[b], (acc_use[b] & 1) ^ 1);
        ptx::tc_fence_after();
        CSB_TL(1, 2, j);
        const uint32_t dS = tmem + colAcc + b * MT;
        uint64_t bh = dn_desc0 + rd.idx * dn_stage_off;
        uint64_t bl = bh + dn_lo_off;
        uint32_t ah = tmem + colXh, al = tmem + colXl;
        for (int kk = 0; kk < K1 / 16; ++kk) {
          ptx::mma_f16_ts_elect(dS, al, bh, idesc1, kk > 0 ? 1u : 0u);
#if !CSB_G1_2X
          ptx::mma_f16_ts_elect(dS, ah, bl, idesc1, 1u);
#endif
          ptx::mma_f16_ts_elect(dS, ah, bh, idesc1, 1u);
          bh += k_step1;
          bl += k_step1;
          ah += 8;
          al += 8;
        }
        ptx::tc_commit_elect(&acc_full[b]);
        if (CL > 1) {
          ptx::tc_commit_multicast_elect(&dn_empty[rd.idx], cl_mask);
        } else {
          ptx::tc_commit_elect(&dn_empty[rd.idx]);
        }
        if (j == T - 1) {
          ptx::tc_commit_elect(x_free);
          ++tcount1;
        }
        ++acc_use[b];
        rd.next();
      };
      auto issue_g2 = [&](int j) {
        const int b = SB == 2 ? (j & 1) : 0;
        CSB_TL(4, 3, j);
        rwait(&s_ready[b], s_use[b] & 1);
        rwait(&p_full[rp.idx], rp.phase);
        if (j == 0) rwait(o_free, (tcount2 & 1) ^ 1);
        ptx::tc_fence_after();
        CSB_TL(4, 4, j);
        const uint64_t bh0 = p_desc0 + rp.idx * p_stage_off;
        const uint64_t bl0 = bh0 + p_lo_off;
        uint32_t ah = tmem + colS + b * MT;
        uint32_t al = ah + MT / 2;
#pragma unroll
        for (int kk = 0; kk < MT / 16; ++kk) {
          const uint64_t bh = bh0 + kk * k_step2, bl = bl0 + kk * k_step2;
          ptx::mma_f16_ts_elect(dO, al, bh, idesc2, (j == 0 && kk == 0) ? 0u : 1u);
          ptx::mma_f16_ts_elect(dO, ah, bl, idesc2, 1u);
          ptx::mma_f16_ts_elect(dO, ah, bh, idesc2, 1u);
          ah += 8;
          al += 8;
        }
        if constexpr (SB == 1 && NB == 2) {
          // S is free again for the set that owns the next step
          ptx::tc_commit_elect(&s_free[j + 1 < T ? ((j + 1) & 1) : 0]);
        } else {
          ptx::tc_commit_elect(&s_free[b]);
        }
        if (CL > 1) {
          ptx::tc_commit_multicast_elect(&p_empty[rp.idx], cl_mask);
        } else {
          ptx::tc_commit_elect(&p_empty[rp.idx]);
        }
        if (j == T - 1) {
          ptx::tc_commit_elect(o_full);
          ptx::mbar_arrive_elect(g2_last);
          ++tcount2;
        }
        ++s_use[b];
        rp.next();
      };

      // GEMM1 and GEMM2 are issued by separate warps (2 and 3), each in its
      // own step order: GEMM1(j + NB) goes as soon as the epilogue has read
      // ACC(j), whatever S hand-off GEMM2 is waiting on (one issuing warp
      // serialised the two chains; tools/timeline.py).  Every commit tracks
      // only its own warp's MMAs, and all cross-GEMM dependencies are
      // mbarriers (ACC, S, X, O), so the tensor pipe may interleave freely.
      if (warp == 2) {
        for (int tile = blockIdx.x; tile < tile_end; tile += gridDim.x)
          for (int j = 0; j < T; ++j) issue_g1(j);
      } else {
        for (int tile = blockIdx.x; tile < tile_end; tile += gridDim.x)
          for (int j = 0; j < T; ++j) issue_g2(j);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 4;               // 0..kEpiWarps-1 (every lane quarter
                                           // appears once in each group of four)
    const int q = warp & 3;                // TMEM lane quarter this warp may access
    const int set = NB == 2 ? ew / kSetWarps : 0;  // step parity owned
    const int half = (ew % kSetWarps) >> 2;        // column slice in step
    const bool tl_lead = ew % kSetWarps == 0;      // timeline recorder of the set (CSB_TIMELINE)
    const int tl_slot = 2 + ew / kSetWarps;
    (void)tl_lead;
    (void)tl_slot;
    // Tile edge (x prologue of the next tile, O readout of this one).  Split
    // edge: the set that does not own step T-1 runs the prologue (8 warps)
    // while the owner of T-1 finishes it and reads O out (8 warps); the
    // prologue set posts ||x||^2 per row through shared memory (a_done).
    // Otherwise all 16 warps run both in turn.  A role is kBW warps = kBG
    // groups of four (one warp per TMEM lane quarter); gi is this warp's group.
    const int kBW = kSplitEdge ? kSetWarps : kEpiWarps;
    const int kBG = kBW / 4;
    const int gi = (ew >> 2) & (kBG - 1);
    const int last_set = kSplitEdge ? ((T - 1) & 1) : 0;
    const bool do_pro = !kSplitEdge || set != last_set;
    const bool do_read = !kSplitEdge || set == last_set;
    const int row = 32 * q + lane;
    const uint32_t lane_off = static_cast<uint32_t>(32 * q) << 16;
    const IO* obs = static_cast<const IO*>(p.obs);
    IO* est = static_cast<IO*>(p.est);
    IO* resid = static_cast<IO*>(p.resid);
    const bool gaussian = p.kind == CS_KERNEL_GAUSSIAN;
    const int c0 = half * COLS;

    // normalised observation value (branch-free: out-of-range reads element
    // 0); column n is the constant 1 that multiplies the ||d||^2 column of
    // the packed D_norm^T tiles.
    auto xnorm = [&](int64_t t, int s, bool valid) -> float {
      const bool ok = valid && s < p.n;
      const IO raw = obs[ok ? t + static_cast<int64_t>(s) * p.ld : 0];
      float v;
      if constexpr (sizeof(IO) == 8) {
        v = static_cast<float>(static_cast<double>(raw) * s_inv_d[s]);
      } else {
        v = static_cast<float>(raw) * s_inv_f[s];
      }
      return ok ? v : (s == p.n ? 1.f : 0.f);
    };

    // raw observations of row t, signals 8 c .. 8 c + 7 (rows past N read
    // row 0, signals past n read signal n-1; callers mask both)
    auto load_chunk = [&](int64_t t, bool valid, int c, IO* r) {
      const int64_t tt = valid ? t : 0;
      if ((c + 1) * 8 <= p.n) {
        ptx::ldg8_strided(obs + tt + static_cast<int64_t>(c) * 8 * p.ld, p.ld, r);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) r[e] = obs[tt + static_cast<int64_t>(min(c * 8 + e, p.n - 1)) * p.ld];
      }
    };
    // normalise a raw value of signal s (column n is the constant that
    // multiplies the packed ||d||^2 column)
    auto norm = [&](IO raw, int s, bool valid) -> float {
      float v;
      if constexpr (sizeof(IO) == 8) {
        v = static_cast<float>(static_cast<double>(raw) * s_inv_d[s]);
      } else {
        v = static_cast<float>(raw) * s_inv_f[s];
      }
      return (valid && s < p.n) ? v : (s == p.n ? p.aug_x : 0.f);
    };

    auto wait = [](uint64_t* bar, uint32_t parity) {
      if constexpr (CSB_WAIT_SLEEP >= 1) {
        ptx::mbar_wait_sleep(bar, parity);
      } else {
        ptx::mbar_wait(bar, parity);
      }
    };
    // TMA issuer for the staged tile edge: one fixed thread (bulk groups are per thread)
    const bool issuer_thread = do_read && ew % kBW == 0 && lane == 0;
    float* s_stage = reinterpret_cast<float*>(smem + p.stage_out_off);  // halves A, B: [n][128] each
    const uint32_t xs_bytes = static_cast<uint32_t>(p.n) * kObsTile * 4;
    auto tma_x = [&](int tile_k, float* dst, uint64_t* bar) {
      const int tk = min(tile_k, n_tiles - 1);  // a dummy slot reads a real tile (rows unused)
      ptx::mbar_arrive_expect_tx(bar, xs_bytes);
      ptx::tma_load_2d(dst, &p.tmap_obs, tk * kObsTile, 0, bar);
    };
    uint32_t prologue_count = 0;
    // x prologue: warp group gi normalises, splits and stores K-chunks
    // k8 = gi mod kBG and contributes a partial ||x||^2 for its chunks.
    // Column n + 1 of the operand is
    // ||x||^2 / kXxCol (GEMM1 then yields d2 itself): it is written once the
    // partials are summed.  Returns ||x||^2 of this thread's row and whether
    // the row must be recomputed exactly.
    constexpr int PB = sizeof(IO) == 8 ? 2 : 4;  // chunks per load batch
    const uint32_t w_xx = static_cast<uint32_t>(p.n + 1) / 2;  // f16x2 word holding column n + 1
    auto prologue = [&](int tile, bool& bad_row) -> float {
      if (tl_lead) CSB_TL(tl_slot, 20, tile);
      const int64_t t = static_cast<int64_t>(tile) * kObsTile + row;
      const bool valid = t < p.N;
      float acc = 0.f;
      bool bad = false;  // a value outside the FP16 split's range: recompute the row exactly
      bool waited = false;
      const int kt = tile / static_cast<int>(gridDim.x);  // tile index of this CTA
      const float* xs = nullptr;
      if constexpr (STAGED) {
        wait(xa_full, kt & 1);
        if (tl_lead) CSB_TL(tl_slot, 45, tile);
        xs = s_stage;
      }
      // split and store one normalised 8-column chunk of the operand
      auto put_chunk = [&](int k8, float* xv) {
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (k8 * 8 + e < p.n) acc = fmaf(xv[e], xv[e], acc);
          const bool out = !(fabsf(xv[e]) < kF16Safe);
          bad |= out;
          if (out) xv[e] = 0.f;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) ptx::split_f16x2(xv[2 * e], xv[2 * e + 1], hi[e], lo[e]);
        ptx::tmem_st4(tmem + lane_off + colXh + k8 * 4, hi);
        ptx::tmem_st4(tmem + lane_off + colXl + k8 * 4, lo);
      };
      if (xs) {
        // staged: shared-memory reads, one chunk at a time (no load batches
        // to keep live: batched registers spilled, and with ~220 KB of
        // shared memory the spills missed the small L1)
        wait(x_free, (prologue_count & 1) ^ 1);
        ++prologue_count;
        ptx::tc_fence_after();
        waited = true;
        if (tl_lead) CSB_TL(tl_slot, 21, tile);
        for (int k8 = gi; k8 < K1 / 8; k8 += kBG) {
          float xv[8];
          const int c = min(k8, (p.n - 1) / 8);
#pragma unroll
          for (int e = 0; e < 8; ++e) xv[e] = norm(xs[min(c * 8 + e, p.n - 1) * kObsTile + row], k8 * 8 + e, valid);
          put_chunk(k8, xv);
        }
      } else {
        // global loads: all loads of a batch are issued before any is
        // consumed (one memory latency per batch instead of one per chunk)
        for (int k0 = gi; k0 < K1 / 8; k0 += kBG * PB) {
          float xv[PB][8];
          {
            IO raw[PB][8];
#pragma unroll
            for (int b = 0; b < PB; ++b)
              if (k0 + kBG * b < K1 / 8) load_chunk(t, valid, min(k0 + kBG * b, (p.n - 1) / 8), raw[b]);
#pragma unroll
            for (int b = 0; b < PB; ++b)
#pragma unroll
              for (int e = 0; e < 8; ++e) xv[b][e] = norm(raw[b][e], (k0 + kBG * b) * 8 + e, valid);
          }
          if (!waited) {
            wait(x_free, (prologue_count & 1) ^ 1);
            ++prologue_count;
            ptx::tc_fence_after();
            if (tl_lead) CSB_TL(tl_slot, 21, tile);
            waited = true;
          }
#pragma unroll
          for (int b = 0; b < PB; ++b) {
            if (k0 + kBG * b >= K1 / 8) break;
            put_chunk(k0 + kBG * b, xv[b]);
          }
        }
      }
      if (!waited) {
        wait(x_free, (prologue_count & 1) ^ 1);
        ++prologue_count;
        ptx::tc_fence_after();
      }
      const int par = kt & 1;
      if (tl_lead) CSB_TL(tl_slot, 42, tile);
      float* xx_part = s_xx + par * 4 * kObsTile;
      uint8_t* bad_part = s_bad + par * 4 * kObsTile;
      xx_part[gi * kObsTile + row] = acc;
      bad_part[gi * kObsTile + row] = bad && valid;
      ptx::named_bar_sync(1, kBW * 32);
      if (tl_lead) CSB_TL(tl_slot, 43, tile);
      float xx = 0.f;
#pragma unroll
      for (int g = 0; g < kBG; ++g) {
        xx += xx_part[g * kObsTile + row];
        bad |= bad_part[g * kObsTile + row] != 0;
      }
      const float xc = xx * (1.f / kXxCol);
      bad = (bad || !(xc < kF16Safe)) && valid;
      if (kSplitEdge && gi == 0) {
        s_xx_tot[par * kObsTile + row] = xx;
        s_bad_tot[par * kObsTile + row] = bad;
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(a_done);  // (after the barrier: all reads of A done)
      }
      if (gi == 0) {
        // the word holding column n + 1 (its partner is the ||d||^2 column n
        // or the zero column n + 2)
        const float a = (p.n & 1) ? 0.f : p.aug_x;
        const float c = bad ? 0.f : xc;
        uint32_t hi, lo;
        if (p.n & 1) {
          ptx::split_f16x2(c, 0.f, hi, lo);
        } else {
          ptx::split_f16x2(a, c, hi, lo);
        }
        ptx::tmem_st1(tmem + lane_off + colXh + w_xx, hi);
        ptx::tmem_st1(tmem + lane_off + colXl + w_xx, lo);
      }
      ptx::tc_wait_st();
      ptx::tc_fence_before();
      __syncwarp();
      if (tl_lead) CSB_TL(tl_slot, 22, tile);
      if (lane == 0) ptx::mbar_arrive(x_ready);
      bad_row = bad;
      return xx;
    };
    uint32_t use = 0, tcount = 0;  // uses of this set's TMEM buffers
    uint32_t s_waits = 0;          // SB = 1, NB = 2: waits on this set's s_free
    bool bad_cur = false;  // row of the current tile recomputed exactly
    float xx_cur = 0.f, thr_cur = 0.f;
    // every d2 >= thr clears the exact near-zero criterion; thr > 0, so rows
    // whose minimum passes also need no clamp before the square root
    auto set_thr = [&]() { thr_cur = p.tau * (xx_cur + p.dd_max); };
    // split edge, readout set: ||x||^2 of tile index k posted by the prologue set
    auto fetch_xx = [&](int k) {
      wait(a_done, k & 1);
      xx_cur = s_xx_tot[(k & 1) * kObsTile + row];
      bad_cur = s_bad_tot[(k & 1) * kObsTile + row] != 0;
      set_thr();
    };
    if (n_iter > 0) {
      if (STAGED && issuer_thread) tma_x(blockIdx.x, s_stage, xa_full);  // x(0) for the first prologue
      if (do_pro) {
        xx_cur = prologue(blockIdx.x, bad_cur);
        set_thr();
      } else {
        fetch_xx(0);
      }
    }
    const float inv_h_s = p.inv_h * (1.f / kSScale);  // exact power-of-two rescaling
    const uint32_t a_base = colAcc + set * MT + c0;
    const int sbuf = SB == 2 ? set : 0;
    const uint32_t s_base = colS + sbuf * MT + c0 / 2;  // f16x2: two columns per word
    for (int tile = blockIdx.x; tile < tile_end; tile += gridDim.x, ++tcount) {
      const int64_t t = static_cast<int64_t>(tile) * kObsTile + row;
      const bool valid = t < p.N;
      bool x_due = STAGED && issuer_thread;
      for (int j = set; j < T; j += NB, ++use) {
        const int valid_cols = min(COLS, p.m - (j * MT + c0));
        const float* dd = p.dd + static_cast<size_t>(j) * MT + c0;
        // ACC chunk c -> similarity values in v[0..CH)
        // the whole ACC slice of this warp: all tcgen05.ld issued, one wait
        auto load_acc = [&](float* vall) {
#pragma unroll
          for (int c = 0; c < COLS / CH; ++c) {
            if constexpr (CH == 16) {
              ptx::tmem_ld16(tmem + lane_off + a_base + c * CH, vall + c * CH);
            } else {
              ptx::tmem_ld8(tmem + lane_off + a_base + c * CH, vall + c * CH);
            }
          }
          ptx::tc_wait_ld();
        };
        auto compute_chunk = [&](int c, float* v) {
          // ACC = d2 = ||x||^2 + ||d||^2 - 2 x.d (tensor core).  The
          // prefilter min(d2) < tau (||x||^2 + max ||d||^2) is a superset of
          // the exact near-zero criterion d2 < tau (||x||^2 + ||d||^2),
          // re-checked per entry; recomputed entries are >= 0, all others
          // >= the criterion's bound >= 0.
          float mn = v[0];
#pragma unroll
          for (int e = 1; e < CH; ++e) mn = fminf(mn, v[e]);
          if ((mn < thr_cur || bad_cur) && valid) {  // rare: direct difference, not unrolled
#pragma unroll 1
            for (int e = 0; e < CH; ++e) {
              float cur = 0.f;
#pragma unroll
              for (int ee = 0; ee < CH; ++ee)
                if (ee == e) cur = v[ee];
              const int col = c * CH + e;
              if (col >= valid_cols || (!bad_cur && !(cur < p.tau * (xx_cur + __ldg(dd + col))))) continue;
              const int mem = j * MT + c0 + col;
              float a = 0.f;
              for (int s = 0; s < p.n; ++s) {
                const float d = xnorm(t, s, true) - __ldg(p.dn32 + static_cast<size_t>(mem) * p.n + s);
                a = fmaf(d, d, a);
              }
#pragma unroll
              for (int ee = 0; ee < CH; ++ee)
                if (ee == e) v[ee] = a;
            }
          }
          // S scaled by 2^14 (FP16 split range, pack_tc.cuh)
          if (gaussian) {
#pragma unroll
            for (int e = 0; e < CH; ++e) v[e] = ptx::ex2_approx(-v[e] * p.g_coef) * kSScale;
          } else {
            // 2^14 / (1 + sqrt(d2)/h) = 1 / (2^-14 + sqrt(d2) (2^-14/h)): the
            // scale folds into the FMA exactly.  sqrt on the MUFU pipe; of
            // every four reciprocals CSB_RCP_MUFU go to MUFU, the rest to an
            // FMA-pipe Newton iteration (default: all on MUFU).
#if CSB_MAP2
#pragma unroll
            for (int e = 0; e < CH; e += 2) {
              const float2 x2 = __ffma2_rn(make_float2(ptx::sqrt_approx(v[e]), ptx::sqrt_approx(v[e + 1])),
                                           make_float2(inv_h_s, inv_h_s),
                                           make_float2(1.f / kSScale, 1.f / kSScale));
              if ((e & 3) < CSB_RCP_MUFU) {
                v[e] = ptx::rcp_approx(x2.x);
                v[e + 1] = ptx::rcp_approx(x2.y);
              } else {
                const float2 y = ptx::rcp_newton2(x2);
                v[e] = y.x;
                v[e + 1] = y.y;
              }
            }
#else
#pragma unroll
            for (int e = 0; e < CH; ++e) {
              const float x = fmaf(ptx::sqrt_approx(v[e]), inv_h_s, 1.f / kSScale);
              v[e] = (e & 3) < CSB_RCP_MUFU ? ptx::rcp_approx(x) : ptx::rcp_newton(x);
            }
#endif
          }
          if (valid_cols < (c + 1) * CH) {
#pragma unroll
            for (int e = 0; e < CH; ++e)
              if (c * CH + e >= valid_cols) v[e] = 0.f;
          }
        };
        // v[0..CH) -> TMEM 2^14 S hi | lo (f16x2 words)
        auto store_chunk = [&](int c, const float* v) {
#pragma unroll
          for (int h8 = 0; h8 < CH / 8; ++h8) {
            uint32_t hi[4], lo[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
#if CSB_MAP2
              ptx::split_f16x2_v2(v[h8 * 8 + 2 * e], v[h8 * 8 + 2 * e + 1], hi[e], lo[e]);
#else
              ptx::split_f16x2(v[h8 * 8 + 2 * e], v[h8 * 8 + 2 * e + 1], hi[e], lo[e]);
#endif
            }
            ptx::tmem_st4(tmem + lane_off + s_base + (c * CH + h8 * 8) / 2, hi);
            ptx::tmem_st4(tmem + lane_off + s_base + MT / 2 + (c * CH + h8 * 8) / 2, lo);
          }
        };
        if (tl_lead) CSB_TL(tl_slot, 10, j);
        wait(&acc_full[set], use & 1);
        ptx::tc_fence_after();
        if (tl_lead) CSB_TL(tl_slot, 11, j);
        if constexpr (SB == 1) {
          // single S buffer: release ACC as early as possible (GEMM1 of the
          // next step may start), then wait for GEMM2 of the previous step
          // before overwriting S.  With two epilogue sets sharing S, GEMM2
          // commits to the s_free barrier of the set owning the next step, so
          // each set counts only its own waits (a shared barrier waited on by
          // parity is ambiguous: GEMM1 runs two steps ahead, so a set can
          // reach its wait before the previous phase has completed).
          float vall[COLS];
          load_acc(vall);
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&acc_free[set]);  // GEMM1 may refill ACC now
#pragma unroll
          for (int c = 0; c < COLS / CH; ++c) compute_chunk(c, vall + c * CH);
          if (tl_lead) CSB_TL(tl_slot, 12, j);
          if constexpr (NB == 1) {
            wait(&s_free[0], (use & 1) ^ 1);
          } else if (tcount != 0 || j != 0) {  // the CTA's first step has no predecessor
            wait(&s_free[set], s_waits & 1);
            ++s_waits;
          }
          ptx::tc_fence_after();
          if (tl_lead) CSB_TL(tl_slot, 13, j);
#pragma unroll
          for (int c = 0; c < COLS / CH; ++c) store_chunk(c, vall + c * CH);
        } else {
          // double buffers: read the ACC slice and release it at once (GEMM1
          // two steps ahead overlaps the kernel map), then map and store S
          float vall[COLS];
          load_acc(vall);
          if (tl_lead) CSB_TL(tl_slot, 46, j);
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&acc_free[set]);
          // map first, then wait for GEMM2(j - 2) to have read S[set]
#pragma unroll
          for (int c = 0; c < COLS / CH; ++c) compute_chunk(c, vall + c * CH);
          if (tl_lead) CSB_TL(tl_slot, 12, j);
          wait(&s_free[set], (use & 1) ^ 1);
          ptx::tc_fence_after();
          if (tl_lead) CSB_TL(tl_slot, 13, j);
#pragma unroll
          for (int c = 0; c < COLS / CH; ++c) store_chunk(c, vall + c * CH);
        }
        ptx::tc_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (tl_lead) CSB_TL(tl_slot, 14, j);
        if (lane == 0) ptx::mbar_arrive(&s_ready[sbuf]);
        if (x_due) {  // staged issuer, first step of the tile: stage x(k + 1) and x(k)
          ptx::bulk_wait_read0();  // the previous edge's stores have read both halves
          ptx::fence_proxy_async_smem();
          if (tile + static_cast<int>(gridDim.x) < tile_end) tma_x(tile + gridDim.x, s_stage, xa_full);
          tma_x(tile, s_stage + p.n * kObsTile, xb_full);
          x_due = false;
        }
      }
      // next tile's x prologue overlaps this tile's last GEMM2
      const int next = tile + gridDim.x;
      float xx_next = 0.f;
      bool bad_next = false;
      if (do_pro && next < tile_end) xx_next = prologue(next, bad_next);

      // readout: estimate = scale .* O, residual = x - estimate.  The raw
      // observations of a batch are loaded before waiting for O.
      const bool issuer = issuer_thread;
      if (do_read) {
        if (tl_lead) CSB_TL(tl_slot, 23, tile);
        float* s_out = s_stage;  // est -> half A, resid -> half B (over x)
        bool o_ready = false;
        if constexpr (STAGED) {
          {
            // x(k) is in half B: one chunk at a time from shared memory
            float* xb = s_stage + p.n * kObsTile;
            wait(xb_full, tcount & 1);
            // half A holds x(k + 1) until the prologue set has staged it
            if (kSplitEdge && next < tile_end) wait(a_done, (tcount + 1) & 1);
            wait(o_full, tcount & 1);
            ptx::tc_fence_after();
            if (tl_lead) CSB_TL(tl_slot, 24, tile);
            o_ready = true;
            // O read CSB_RD_BATCH chunks per TMEM wait
            constexpr int OB = CSB_RD_BATCH;
            for (int c0 = gi; c0 < N2 / 8; c0 += OB * kBG) {
              float o[OB][8];
#pragma unroll
              for (int b = 0; b < OB; ++b)
                if (c0 + b * kBG < N2 / 8) ptx::tmem_ld8(tmem + lane_off + colO + (c0 + b * kBG) * 8, o[b]);
              ptx::tc_wait_ld();
              if (tl_lead && c0 == gi) CSB_TL(tl_slot, 44, tile);
#pragma unroll
              for (int b = 0; b < OB; ++b) {
                const int c = c0 + b * kBG;
                if (c >= N2 / 8) break;
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                  const int s = c * 8 + e;
                  if (s < p.n) {
                    const float ev = o[b][e] * s_scale_f[s];
                    s_out[s * kObsTile + row] = ev;
                    xb[s * kObsTile + row] -= ev;
                  }
                }
              }
            }
          }
        } else {
          // x loads of all of a thread's chunks are issued before O is waited
          // for (one latency); O is read a chunk at a time (register pressure)
          constexpr int RB = PB;  // (plain edge: four groups)
          for (int cb = gi; cb < N2 / 8; cb += kBG * RB) {
            IO xr[RB][8];
#pragma unroll
            for (int b = 0; b < RB; ++b)
              if (cb + kBG * b < N2 / 8) load_chunk(t, valid, min(cb + kBG * b, (p.n - 1) / 8), xr[b]);
            if (!o_ready) {
              wait(o_full, tcount & 1);
              ptx::tc_fence_after();
              if (tl_lead) CSB_TL(tl_slot, 24, tile);
              o_ready = true;
            }
#pragma unroll
            for (int b = 0; b < RB; ++b) {
              const int c = cb + kBG * b;
              if (c >= N2 / 8) break;
              float o[8];
              ptx::tmem_ld8_wait(tmem + lane_off + colO + c * 8, o);
              if (tl_lead && c == gi) CSB_TL(tl_slot, 44, tile);
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const int s = c * 8 + e;
                const bool ok = valid && s < p.n;
                const int64_t idx = t + static_cast<int64_t>(s) * p.ld;
                if constexpr (sizeof(IO) == 8) {
                  const double ev = static_cast<double>(o[e]) * s_scale_d[s];
                  if (ok && est) est[idx] = ev;
                  if (ok && resid) resid[idx] = xr[b][e] - ev;
                } else {
                  const float ev = o[e] * s_scale_f[s];
                  if (ok && est) est[idx] = ev;
                  if (ok && resid) resid[idx] = xr[b][e] - ev;
                }
              }
            }
          }
        }
        if (!o_ready) {
          wait(o_full, tcount & 1);
          ptx::tc_fence_after();
        }
        if (tl_lead) CSB_TL(tl_slot, 27, tile);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(o_free);  // O read: the next tile's GEMM2 may start
        if constexpr (STAGED) {
          ptx::fence_proxy_async_smem();
          ptx::named_bar_sync(2, kBW * 32);
          if (issuer && tile < n_tiles) {  // (a dummy slot has nothing to store)
            const int t0 = tile * kObsTile;
            if (est) ptx::tma_store_2d(&p.tmap_est, t0, 0, s_out);
            if (resid) ptx::tma_store_2d(&p.tmap_res, t0, 0, s_out + p.n * kObsTile);
            ptx::bulk_commit();
          }
        }
        if (tl_lead) CSB_TL(tl_slot, 25, tile);
      }
      if (next < tile_end) {
        if (do_pro) {
          xx_cur = xx_next;
          bad_cur = bad_next;
          set_thr();
        } else {
          fetch_xx(tcount + 1);
        }
      }
      if (tl_lead) CSB_TL(tl_slot, 26, tile);
    }
    if (STAGED && issuer_thread) ptx::bulk_wait0();  // stores complete before exit
  }
  __syncthreads();
  if (CL > 1) ptx::cluster_sync();  // no CTA leaves while peers may still signal it
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kTmemCols);
  }
}

}  // namespace csb
