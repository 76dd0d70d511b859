// Microbenchmark of the small R x R kernels (Cholesky, solve) in isolation.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2010_12056_b200/csrc/kernels.h"
int main(int argc, char** argv) {
  int R = argc > 1 ? atoi(argv[1]) : 64;
  int rows = argc > 2 ? atoi(argv[2]) : 1024;
  int N = 3;
  std::vector<double> S(N * R * R);
  for (int k = 0; k < N; k++)
    for (int i = 0; i < R; i++)
      for (int j = 0; j < R; j++) S[k * R * R + i * R + j] = (i == j ? R : 0.0) + 1.0 / (1 + i + j);
  double *dS, *Lp, *M, *X;
  int* st;
  cudaMalloc(&dS, S.size() * 8);
  cudaMemcpy(dS, S.data(), S.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&Lp, (R * R + R) * 8);
  cudaMalloc(&M, (size_t)rows * R * 8);
  cudaMalloc(&X, (size_t)rows * R * 8);
  cudaMemset(M, 0, (size_t)rows * R * 8);
  cudaMalloc(&st, 64);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; w++) cpd::launch_gamma_chol(dS, N, 0, R, Lp, st, s);
  cudaStreamSynchronize(s);
  float ms;
  cudaEventRecord(a, s);
  for (int it = 0; it < 100; it++) cpd::launch_gamma_chol(dS, N, 0, R, Lp, st, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("R=%d chol: %.2f us/launch (%s)\n", R, ms * 10, cudaGetErrorString(cudaGetLastError()));
  for (int w = 0; w < 3; w++) cpd::launch_trisolve(Lp, M, rows, R, X, s);
  cudaEventRecord(a, s);
  for (int it = 0; it < 100; it++) cpd::launch_trisolve(Lp, M, rows, R, X, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("R=%d rows=%d trisolve: %.2f us/launch\n", R, rows, ms * 10);
  // empty-kernel floor
  return 0;
}
