// Microbenchmark: Γ^{-1} (blocked Gauss-Jordan, launch_gamma_inverse) and the fused update in
// isolation; CPD_GJ_DBG bits skip phases (1 pivot block, 2 panel, 4 rank-16 update).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include tools/bench_ginv.cu
//        paper_2010_12056_b200/csrc/small.cu -o tools/bench_ginv
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2010_12056_b200/csrc/kernels.h"
namespace cpd { std::atomic<long long> g_launches{0}; }
int main(int argc, char** argv) {
  const int N = 4;
  for (int R : {32, 64, 100, 128}) {
    std::vector<double> S(N * R * R);
    for (int k = 0; k < N; k++)
      for (int i = 0; i < R; i++)
        for (int j = 0; j < R; j++) S[k * R * R + i * R + j] = (i == j ? 2.0 * R : 0.0) + 1.0 / (1 + i + j);
    double *dS, *G;
    int* st;
    cudaMalloc(&dS, S.size() * 8);
    cudaMemcpy(dS, S.data(), S.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&G, (size_t)R * R * 8);
    cudaMalloc(&st, 64);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 3; w++) cpd::launch_gamma_inverse(dS, N, 0, R, G, st, s);
    cudaEventRecord(a, s);
    for (int w = 0; w < 20; w++) cpd::launch_gamma_inverse(dS, N, 0, R, G, st, s);
    cudaEventRecord(b, s);
    cudaStreamSynchronize(s);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("R=%d gamma_inverse %.1f us  (%s)\n", R, 1e3 * ms / 20, cudaGetErrorString(cudaGetLastError()));
    cudaFree(dS);
    cudaFree(G);
  }
  return 0;
}
