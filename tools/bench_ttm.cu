// Microbenchmark of the first-level TTM kernel on BASELINE-shaped problems.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include "../paper_2010_12056_b200/csrc/kernels.h"
int main() {
  struct Case { const char* name; long pre, K, post; int R; };
  Case cases[] = {{"C2 root j=3 (KC)", 1L << 20, 1024, 1, 64}, {"C2 root j=1 (MC)", 1, 1024, 1L << 20, 64},
                  {"C2 root j=2 (MC batched)", 1024, 1024, 1024, 64}, {"C3 root j=4 (KC)", 8000000, 200, 1, 100},
                  {"C3 root j=2 (MC)", 200, 200, 40000, 100}, {"C4 root j=5 (KC)", 16777216, 64, 1, 32},
                  {"C5-like KC R=200", 1L << 20, 2048, 1, 200}};
  size_t maxT = 0, maxO = 0, maxA = 0;
  for (auto& c : cases) {
    size_t t = (size_t)c.pre * c.K * c.post, o = (size_t)c.pre * c.post * c.R, a = (size_t)c.K * c.R;
    if (t > maxT) maxT = t; if (o > maxO) maxO = o; if (a > maxA) maxA = a;
  }
  double *T, *O, *A;
  cudaMalloc(&T, maxT * 8); cudaMalloc(&O, maxO * 8); cudaMalloc(&A, maxA * 8);
  cudaMemset(T, 0, maxT * 8); cudaMemset(A, 0, maxA * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (auto& c : cases) {
    for (int w = 0; w < 2; w++) cpd::launch_ttm(T, c.pre, c.K, c.post, A, c.R, O, 0, 0);
    cudaEventRecord(a);
    int it = 5;
    for (int i = 0; i < it; i++) cpd::launch_ttm(T, c.pre, c.K, c.post, A, c.R, O, 0, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= it;
    double fl = 2.0 * c.pre * c.post * c.K * c.R;
    printf("%-28s %8.3f ms  %6.2f TF/s  (%s)\n", c.name, ms, fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
