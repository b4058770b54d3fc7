// dmma_bench.cu -- standalone timing / correctness probe of the FP64 DMMA
// train kernels (paper_2003_08011_b200/csrc/train_f64.cu): Gram, GEMM,
// Cholesky leaf and the recursive Cholesky inverse.  Development tool.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
//        -I include -I paper_2003_08011_b200/csrc tools/dmma_bench.cu -o tools/dmma_bench
//   tools/dmma_bench [m ...]
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CSB_LEAF_PROFILE 1
#include "../paper_2003_08011_b200/csrc/train_f64.cu"

using namespace csb;

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)

// median of `reps` individually event-timed calls (after one warm-up)
template <class F>
float time_ms(cudaStream_t st, int reps, F f) {
  f();
  CK(cudaStreamSynchronize(st));
  std::vector<float> t;
  for (int i = 0; i < reps; ++i) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
    f();
    cudaEventRecord(b, st);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    t.push_back(ms);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  std::sort(t.begin(), t.end());
  return t[t.size() / 2];
}

int main(int argc, char** argv) {
  std::vector<int> ms;
  for (int i = 1; i < argc; ++i) ms.push_back(std::atoi(argv[i]));
  if (ms.empty()) ms = {1000, 4000, 8000};
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  alloc_stream() = st;
  configure_pool(0);
  for (int m : ms) {
    const int n = m / 4;
    std::vector<double> h(static_cast<size_t>(n) * m);
    std::mt19937_64 rng(7);
    std::normal_distribution<double> nd;
    for (auto& v : h) v = nd(rng);
    double *Dn, *G, *Gi, *E;
    CK(cudaMalloc(&Dn, sizeof(double) * n * m));
    CK(cudaMalloc(&G, sizeof(double) * m * m));
    CK(cudaMalloc(&Gi, sizeof(double) * m * m));
    CK(cudaMalloc(&E, sizeof(double) * m * m));
    CK(cudaMemcpy(Dn, h.data(), sizeof(double) * n * m, cudaMemcpyHostToDevice));
    const double hbw = std::sqrt(static_cast<double>(n));
    const float t_gram = time_ms(st, 9, [&] { dmma_gram(st, Dn, n, m, 0, hbw, G); });
    const float t_gemm = time_ms(st, 9, [&] { dmma_gemm(st, 0, m, m, m, 1.0, G, m, G, m, 0.0, E, m); });
    const float t_p = time_ms(st, 9, [&] { dmma_gemm(st, 0, n, m, m, 1.0, Dn, n, G, m, 0.0, E, n); });
    bool ok = true;
    const float t_inv = time_ms(st, 7, [&] { ok = dmma_chol_inverse(st, G, m, Gi) && ok; });
    // leaf alone: m/128 sequential launches on the diagonal blocks
    int* fail;
    CK(cudaMalloc(&fail, sizeof(int)));
    CK(cudaMemset(fail, 0, sizeof(int)));
    cudaFuncSetAttribute(chol_inv_leaf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kLeafSmem));
    const int nleaf = m / kLeaf;
    const float t_leaf = time_ms(st, 7, [&] {
      for (int b = 0; b < nleaf; ++b)
        chol_inv_leaf_kernel<<<1, kLeafThreads, kLeafSmem, st>>>(G, m, static_cast<int64_t>(b) * kLeaf, kLeaf, E, m,
                                                                  fail);
    });
    {
      long long clk[64];
      CK(cudaMemcpyFromSymbol(clk, g_leaf_clk, sizeof clk));
      std::printf("leaf phases (cycles from start): load %lld", clk[1] - clk[0]);
      for (int kb = 0; kb < 4; ++kb)
        std::printf(" | kb%d warp0 %lld panel %lld trail %lld", kb, clk[2 + 3 * kb] - clk[0], clk[3 + 3 * kb] - clk[0],
                    clk[4 + 3 * kb] - clk[0]);
      for (int kb = 0; kb < 4; ++kb)
        std::printf(" | kb%d factor-done %lld inv-start %lld", kb, clk[20 + kb] - clk[0], clk[24 + kb] - clk[0]);
      std::printf(" | inv d1 %lld d2 %lld d3 %lld | end %lld\n", clk[15] - clk[0], clk[16] - clk[0], clk[17] - clk[0],
                  clk[18] - clk[0]);
    }
    // residual: G Gi - I
    dmma_gemm(st, 0, m, m, m, 1.0, G, m, Gi, m, 0.0, E, m);
    std::vector<double> e(static_cast<size_t>(m) * m);
    CK(cudaMemcpyAsync(e.data(), E, sizeof(double) * m * m, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    double err = 0;
    for (int j = 0; j < m; ++j)
      for (int i = 0; i < m; ++i) err = std::fmax(err, std::fabs(e[i + static_cast<size_t>(j) * m] - (i == j)));
    const double fg = 2.0 * m * m * n / 2, fm = 2.0 * m * m * m, fp = 2.0 * n * m * m, fi = 1.0 * m * m * m;
    std::printf(
        "m=%d n=%d  gram %.3f ms (%.1f TF/s lower half)  gemm mxmxm %.3f ms (%.1f TF/s)  P nxmxm %.3f ms (%.1f TF/s)  "
        "chol_inverse %.3f ms (%.1f TF/s of m^3)  %d leaves %.3f ms (%.1f us each)  ok=%d  max|G Gi - I| %.2e\n",
        m, n, t_gram, fg / t_gram / 1e9, t_gemm, fm / t_gemm / 1e9, t_p, fp / t_p / 1e9, t_inv, fi / t_inv / 1e9,
        nleaf, t_leaf, 1e3 * t_leaf / nleaf, ok ? 1 : 0, err);
    cudaFree(Dn);
    cudaFree(G);
    cudaFree(Gi);
    cudaFree(E);
    cudaFree(fail);
  }
  return 0;
}
