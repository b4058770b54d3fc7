// mma_probe.cu -- measures tcgen05.mma issue/throughput on this part.
//
// One CTA per SM; one warp issues `iters` back-to-back MMAs into a TMEM
// accumulator, then commits and waits.  Reports cycles per MMA and the
// implied dense throughput for kind::tf32 / kind::f16 (bf16), A from TMEM
// ("TS") or shared memory ("SS"), over N.  Used to pin the tensor-pipe
// ceiling the surveillance kernel is compared against (profiles/).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe mma_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2003_08011_b200/csrc/sm100_ptx.cuh"

using namespace csb;

__device__ __forceinline__ uint32_t idesc(int kind, int M, int N) {
  // kind 0: tf32 (a/b format 2), kind 1: f16 (kind::f16, format 0); F32 accumulate
  const uint32_t f = kind == 0 ? 2u : 0u;
  return (1u << 4) | (f << 7) | (f << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_ts(int kind, uint32_t d, uint32_t a, uint64_t b, uint32_t id) {
  if (kind == 0)
    asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;" ::"r"(d), "r"(a), "l"(b), "r"(id));
  else
    asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;" ::"r"(d), "r"(a), "l"(b), "r"(id));
}
__device__ __forceinline__ void mma_ss(int kind, uint32_t d, uint64_t a, uint64_t b, uint32_t id) {
  if (kind == 0)
    asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a), "l"(b), "r"(id));
  else
    asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a), "l"(b), "r"(id));
}

__global__ void __launch_bounds__(128, 1) probe(int kind, int ts, int N, int iters, long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc(&holder, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = holder;
  if (warp == 1) {
    const uint32_t id = idesc(kind, 128, N);
    const uint32_t sb = ptx::smem_u32(smem);
    const uint64_t bdesc = ptx::smem_desc(sb, (N / 8) * 128, 128);
    const uint64_t adesc = ptx::smem_desc(sb + 32768, 16 * 128, 128);
    const long long t0 = clock64();
    if (kind == 0) {
      if (ts) {
        for (int i = 0; i < iters; ++i) ptx::mma_tf32_ts_elect(tmem, tmem + 256 + (i & 7) * 8, bdesc, id, 1u);
      } else {
        for (int i = 0; i < iters; ++i) ptx::mma_tf32_ss_elect(tmem, adesc, bdesc, id, 1u);
      }
    } else {
      if (ts) {
        for (int i = 0; i < iters; ++i) ptx::mma_f16_ts_elect(tmem, tmem + 256 + (i & 7) * 8, bdesc, id, 1u);
      } else {
        for (int i = 0; i < iters; ++i) ptx::mma_f16_ss_elect(tmem, adesc, bdesc, id, 1u);
      }
    }
    ptx::tc_commit_elect(&bar);
    ptx::mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 32) cycles[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 4096;
  printf("{\"sm_clock_khz\": %d, \"results\": [\n", clk);
  bool first = true;
  for (int kind = 0; kind < 2; ++kind)
  for (int ts = 1; ts >= 0; --ts) {
    for (int N : {16, 32, 64, 112, 128, 256}) {
      probe<<<148, 128, 96 * 1024>>>(kind, ts, N, iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (long long v : h) mx = v > mx ? v : mx;
      const double cyc = static_cast<double>(mx) / iters;
      // per SM: 128 x N x K MACs per MMA (K = 8 tf32, 16 f16)
      const double macs_per_clk = 128.0 * N * (kind ? 16 : 8) / cyc;
      const double tflops = 2.0 * macs_per_clk * 148 * clk * 1e3 / 1e12;
      printf("%s {\"form\": \"%s\", \"kind\": \"%s\", \"M\": 128, \"N\": %d, \"cycles_per_mma\": %.2f, "
             "\"mac_per_clk_per_sm\": %.1f, \"tflops_at_base_clock\": %.1f, \"err\": \"%s\"}",
             first ? "" : ",\n", ts ? "TS" : "SS", kind ? "f16" : "tf32", N, cyc, macs_per_clk, tflops,
             cudaGetErrorString(e));
      first = false;
    }
  }
  printf("\n]}\n");
  return 0;
}
