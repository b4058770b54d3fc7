// selection.cuh -- bit-exact memory-vector selection on the device
// (select_memory_vectors, mset.cpp:72-137).
//
//  * distinct-row count: FNV-1a over each row's raw bytes (mset.cpp:22-42),
//    one thread per row (column-major input -> coalesced across threads),
//    radix sort of the 64-bit hashes, adjacent-difference count.  Hash
//    collisions count as duplicates, exactly as the reference's
//    unordered_set of hashes does.
//  * stage 1: per-signal argmin / argmax, earliest index on ties
//    (strict < / > scan, mset.cpp:99-104) as a (value, index) block
//    reduction; the min-before-max dedupe over signals (first occurrence
//    of each row in candidate order) by atomicMin + an ordered block
//    compaction.
//  * stage 2: Eigen row(r).norm() is a left-to-right sum of squares
//    (no FMA) then sqrt; restated with __dmul_rn/__dadd_rn.  Non-negative
//    doubles order like their bit patterns, so sorting (norm, index) pairs is
//    a stable LSD radix sort of the norm bits over rows in index order;
//    already-selected rows get key UINT64_MAX and sort past the pool.
#pragma once

#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

namespace csb {

__global__ void row_hash_kernel(const double* __restrict__ X, int64_t N, int64_t n,
                                unsigned long long* __restrict__ hashes) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= N) return;
  unsigned long long h = 1469598103934665603ULL;
  auto mix = [&h](unsigned long long bits) {
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      h ^= (bits >> (8 * b)) & 0xffULL;
      h *= 1099511628211ULL;
    }
  };
  int64_t s = 0;
  // sixteen signals' loads in flight before their bytes enter the (serial) hash
  for (; s + 16 <= n; s += 16) {
    unsigned long long bits[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) bits[k] = static_cast<unsigned long long>(__double_as_longlong(__ldg(X + r + (s + k) * N)));
#pragma unroll
    for (int k = 0; k < 16; ++k) mix(bits[k]);
  }
  for (; s < n; ++s) mix(static_cast<unsigned long long>(__double_as_longlong(__ldg(X + r + s * N))));
  hashes[r] = h;
}

__global__ void count_distinct_kernel(const unsigned long long* __restrict__ sorted, int64_t N,
                                      unsigned long long* __restrict__ count) {
  unsigned long long local = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < N;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    local += (i == 0 || sorted[i] != sorted[i - 1]) ? 1ULL : 0ULL;
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(count, local);
}

// (value, index) ordering for the extrema scan: strictly smaller value wins,
// equal values keep the earlier index -- the result of the reference's
// sequential `if (x[r] < x[imin]) imin = r` loop.
__device__ __forceinline__ void better_min(double& v, int64_t& i, double v2, int64_t i2) {
  if (v2 < v || (!(v < v2) && i2 < i)) { v = v2; i = i2; }
}
__device__ __forceinline__ void better_max(double& v, int64_t& i, double v2, int64_t i2) {
  if (v2 > v || (!(v > v2) && i2 < i)) { v = v2; i = i2; }
}

__global__ void __launch_bounds__(256)
col_extrema_kernel(const double* __restrict__ X, int64_t N, int64_t* __restrict__ imin_out,
                   int64_t* __restrict__ imax_out) {
  const int64_t s = blockIdx.x;
  const double* col = X + s * N;
  double vmin = col[0], vmax = col[0];
  int64_t imin = 0, imax = 0;
  for (int64_t r = threadIdx.x; r < N; r += blockDim.x) {
    const double v = col[r];
    better_min(vmin, imin, v, r);
    better_max(vmax, imax, v, r);
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double v1 = __shfl_xor_sync(0xffffffffu, vmin, o);
    const int64_t i1 = __shfl_xor_sync(0xffffffffu, imin, o);
    const double v2 = __shfl_xor_sync(0xffffffffu, vmax, o);
    const int64_t i2 = __shfl_xor_sync(0xffffffffu, imax, o);
    better_min(vmin, imin, v1, i1);
    better_max(vmax, imax, v2, i2);
  }
  __shared__ double sv[2][8];
  __shared__ int64_t si[2][8];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane == 0) {
    sv[0][warp] = vmin; si[0][warp] = imin;
    sv[1][warp] = vmax; si[1][warp] = imax;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x / 32); ++w) {
      better_min(vmin, imin, sv[0][w], si[0][w]);
      better_max(vmax, imax, sv[1][w], si[1][w]);
    }
    imin_out[s] = imin;
    imax_out[s] = imax;
  }
}

// mset.cpp:99-111: signals in order, min before max, skip already-selected.
// Candidate p = 2 s + j (j = 0 min, 1 max) is picked iff no earlier
// candidate names the same row: first[row] = min p by atomicMin, then a
// block-wide ordered compaction keeps the reference's pick order.  One CTA
// (the sequential walk it replaces was a chain of dependent L2 round trips,
// ~0.3 ms at n = 1000).  `first` holds N entries preset to 0xffffffff.
__global__ void __launch_bounds__(1024) stage1_dedupe_kernel(const int64_t* __restrict__ imin,
                                                             const int64_t* __restrict__ imax, int64_t n,
                                                             unsigned char* __restrict__ selected,
                                                             int64_t* __restrict__ picked,
                                                             int64_t* __restrict__ npicked,
                                                             unsigned* __restrict__ first) {
  __shared__ int warp_sum[32];
  __shared__ int64_t running;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int64_t C = 2 * n;
  auto row_of = [&](int64_t p) { return (p & 1) ? imax[p >> 1] : imin[p >> 1]; };
  for (int64_t p = tid; p < C; p += blockDim.x) atomicMin(first + row_of(p), static_cast<unsigned>(p));
  if (tid == 0) running = 0;
  __syncthreads();
  for (int64_t base = 0; base < C; base += blockDim.x) {
    const int64_t p = base + tid;
    int64_t r = 0;
    bool keep = false;
    if (p < C) {
      r = row_of(p);
      keep = __ldcg(first + r) == static_cast<unsigned>(p);
    }
    const unsigned ballot = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) warp_sum[warp] = __popc(ballot);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < nw; ++w) {
      before += w < warp ? warp_sum[w] : 0;
      total += warp_sum[w];
    }
    const int64_t at = running + before + __popc(ballot & ((1u << lane) - 1u));
    if (keep) {
      picked[at] = r;
      selected[r] = 1;
    }
    __syncthreads();  // everyone has read warp_sum / running
    if (tid == 0) running += total;
    __syncthreads();
  }
  if (tid == 0) *npicked = running;
}

__global__ void row_norm_key_kernel(const double* __restrict__ X, int64_t N, int64_t n,
                                    const unsigned char* __restrict__ selected,
                                    unsigned long long* __restrict__ keys,
                                    int64_t* __restrict__ rows) {
  const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (r >= N) return;
  rows[r] = r;
  if (selected[r]) {
    keys[r] = ~0ULL;
    return;
  }
  double s2 = 0.0;
  for (int64_t s = 0; s < n; ++s) {
    const double v = X[r + s * N];
    s2 = __dadd_rn(s2, __dmul_rn(v, v));
  }
  keys[r] = static_cast<unsigned long long>(__double_as_longlong(sqrt(s2)));
}

// mset.cpp:123-128: pos = i*(pool-1)/(remaining-1) over the sorted pool.
__global__ void stride_pick_kernel(const int64_t* __restrict__ sorted_rows, int64_t N,
                                   int64_t m, const int64_t* __restrict__ npicked_dev,
                                   int64_t* __restrict__ picked) {
  const int64_t np = *npicked_dev;
  const int64_t remaining = m - np;
  const int64_t pool = N - np;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < remaining;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t pos = remaining == 1 ? (pool - 1) / 2 : i * (pool - 1) / (remaining - 1);
    picked[np + i] = sorted_rows[pos];
  }
}

// D(:, c) = training.row(picked[c])  (mset.cpp:131-135)
__global__ void gather_memory_kernel(const double* __restrict__ X, int64_t N, int64_t n,
                                     const int64_t* __restrict__ picked, int64_t m,
                                     double* __restrict__ D) {
  const int64_t total = n * m;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = e % n, c = e / n;
    D[e] = X[picked[c] + s * N];
  }
}

}  // namespace csb
