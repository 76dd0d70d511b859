// FP64 peak microbenchmarks on sm_100a: DMMA (mma.sync .f64) issue rate, DFMA rate, HBM read stream.
// Used once to fill the FP64 roofline denominators in MEASURED_FP64.json (MEASURED_PEAKS.json has none).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)

__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; i++) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
__global__ void dmma_m16n8k8(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = 1.0 + threadIdx.x * 1e-4, b1 = b0 + 1;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) c[i][j] = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; i++) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}
__global__ void dfma_loop(double* out, int iters) {
  double x[8];
  double a = 1.0000001, b = 1e-9 * threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; i++) x[i] = i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += x[i];
  if (s == 12345.678) out[0] = s;
}
__global__ void read_stream(const double2* __restrict__ p, size_t n2, double* out) {
  double acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n2; i += 4 * stride) {
    double2 v0 = __ldcs(p + i), v1 = __ldcs(p + i + stride), v2 = __ldcs(p + i + 2 * stride), v3 = __ldcs(p + i + 3 * stride);
    acc += v0.x + v0.y + v1.x + v1.y + v2.x + v2.y + v3.x + v3.y;
  }
  for (; i < n2; i += stride) { double2 v = p[i]; acc += v.x + v.y; }
  if (acc == 12345.678) out[0] = acc;
}
int main() {
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0));
  int sms = pr.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d", pr.name, sms);
  double* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  int iters = 20000;
  for (int bpsm : {4, 8}) {
    int grid = sms * bpsm, thr = 256;
    dmma_m8n8k4<<<grid, thr>>>(out, 100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dmma_m8n8k4<<<grid, thr>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = (double)grid * (thr / 32) * iters * 8 * 512.0;
    printf(", \"dmma_m8n8k4_tflops_b%d\": %.2f", bpsm, fl / ms / 1e9);
    dmma_m16n8k8<<<grid, thr>>>(out, 100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dmma_m16n8k8<<<grid, thr>>>(out, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    fl = (double)grid * (thr / 32) * iters * 4 * 2048.0;
    printf(", \"dmma_m16n8k8_tflops_b%d\": %.2f", bpsm, fl / ms / 1e9);
    dfma_loop<<<grid, thr>>>(out, 100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dfma_loop<<<grid, thr>>>(out, iters * 4); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    fl = (double)grid * thr * (iters * 4.0) * 8 * 2.0;
    printf(", \"dfma_tflops_b%d\": %.2f", bpsm, fl / ms / 1e9);
  }
  size_t bytes = (size_t)8 << 30;
  double2* p; CK(cudaMalloc(&p, bytes)); CK(cudaMemset(p, 0, bytes));
  float best = 1e30f;
  for (int r = 0; r < 6; r++) {
    cudaEventRecord(e0); read_stream<<<sms * 8, 512>>>(p, bytes / 16, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf(", \"hbm_read_gbs\": %.1f", bytes / best / 1e6);
  printf("}\n");
  return 0;
}
