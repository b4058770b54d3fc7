// peaks_probe.cu -- measured FP64 / FP32 / MUFU throughput ceilings of this part.
//
// The train path is FP64 ("FP64 DMMA/DFMA ... measure, do not
// assume") and the C1 surveillance corner is MUFU-bound.  Each
// probe runs a persistent grid (SMs x 4 CTAs of 256 threads) of independent
// dependency chains long enough to hide latency, times it with CUDA events
// and prints one JSON object (profiles/peaks_probe.json):
//   dmma_f64_tflops   mma.sync.aligned.m8n8k4.row.col.f64 (2*8*8*4 flops/warp-op)
//   dfma_f64_tflops   fma.rn.f64 (2 flops/thread-op)
//   ffma_f32_tflops   fma.rn.f32
//   mufu_rsqrt_gops   rsqrt.approx.f32 results/s
//   mufu_ex2_gops     ex2.approx.f32 results/s
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks_probe peaks_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

constexpr int kChains = 8;

__global__ void dmma_kernel(int iters, double* out) {
  double acc[kChains][2];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c][0] = acc[c][1] = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c][0] + acc[c][1];
  if (s == 123.456) out[0] = s;
}

__global__ void dfma_kernel(int iters, double* out) {
  double acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = c;
  const double a = 1.0 + threadIdx.x * 1e-12, b = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 123.456) out[0] = s;
}

__global__ void ffma_kernel(int iters, double* out) {
  float acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = c;
  const float a = 1.0f + threadIdx.x * 1e-7f, b = 1e-6f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = fmaf(acc[c], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 123.456f) out[0] = s;
}

template <int OP>
__global__ void mufu_kernel(int iters, double* out) {
  float acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = 1.0f + c + threadIdx.x * 1e-3f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      float r;
      if (OP == 0)
        asm volatile("rsqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(acc[c]));
      else
        asm volatile("ex2.approx.f32 %0, %1;" : "=f"(r) : "f"(acc[c]));
      acc[c] = r;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 123.456f) out[0] = s;
}

template <typename K>
double time_it(K kernel, int blocks, int threads, int iters, double* out) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kernel<<<blocks, threads>>>(iters / 10, out);  // warm-up (clocks up, module load)
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    kernel<<<blocks, threads>>>(iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return best * 1e-3;
}

int main() {
  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  double* out;
  cudaMalloc(&out, 8);
  const int blocks = sms * 4, threads = 256;
  const double warps = static_cast<double>(blocks) * threads / 32;
  const double lanes = static_cast<double>(blocks) * threads;
  const int it_dmma = 4096, it_fma = 8192, it_mufu = 4096;
  const double t_dmma = time_it(dmma_kernel, blocks, threads, it_dmma, out);
  const double t_dfma = time_it(dfma_kernel, blocks, threads, it_fma, out);
  const double t_ffma = time_it(ffma_kernel, blocks, threads, it_fma, out);
  const double t_rsq = time_it(mufu_kernel<0>, blocks, threads, it_mufu, out);
  const double t_ex2 = time_it(mufu_kernel<1>, blocks, threads, it_mufu, out);
  const double dmma = warps * it_dmma * kChains * 2.0 * 8 * 8 * 4 / t_dmma / 1e12;
  const double dfma = lanes * it_fma * kChains * 2.0 / t_dfma / 1e12;
  const double ffma = lanes * it_fma * kChains * 2.0 / t_ffma / 1e12;
  const double rsq = lanes * it_mufu * kChains / t_rsq / 1e9;
  const double ex2 = lanes * it_mufu * kChains / t_ex2 / 1e9;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  std::printf(
      "{\"device\": \"%s\", \"sms\": %d, \"clock_khz_attr\": %d, \"dmma_f64_tflops\": %.3f, "
      "\"dfma_f64_tflops\": %.3f, \"ffma_f32_tflops\": %.3f, \"mufu_rsqrt_gops\": %.1f, \"mufu_ex2_gops\": %.1f, "
      "\"how\": \"tools/peaks_probe.cu: %d CTAs x %d threads, %d independent chains per thread, best of 5 "
      "(CUDA events)\", \"err\": \"%s\"}\n",
      prop.name, sms, clk, dmma, dfma, ffma, rsq, ex2, blocks, threads, kChains,
      cudaGetErrorString(cudaGetLastError()));
  return 0;
}
