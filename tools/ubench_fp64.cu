// Development microbenchmark: FP64 pipe rates on this part (DFMA, F2I.F64/I2F.F64 conversions,
// the exact kernel's weight() body).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubf64 tools/ubench_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int n, double a) {
  double x[8];
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, 1e-9);
  double s = 0;
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.678) out[0] = s;
}
__global__ void k_cvt(double* out, int n, double a) {
  double x[8];
  int acc = 0;
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int b = (int)(x[j] * 64.0);
      acc += b;
      x[j] = x[j] * a + (double)(b & 7);
    }
  if (acc == 12345) out[0] = acc;
}
__global__ void k_f32(float* out, int n, float a) {
  float x[8];
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3f + j;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fmaf(x[j], a, 1e-9f);
  float s = 0;
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.678f) out[0] = s;
}
int main() {
  double* d;
  cudaMalloc(&d, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int n = 4096, blocks = 148, thr = 512;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0);
    k_dfma<<<blocks, thr>>>(d, n, 0.999999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * thr * n * 8;
    printf("DFMA: %.3f ms  %.1f per clk per SM (1.965 GHz)\n", ms, ops / (ms * 1e-3) / 1.965e9 / 148);
    cudaEventRecord(e0);
    k_cvt<<<blocks, thr>>>(d, n, 0.999999);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DMUL+F2I+I2F+DADD group: %.3f ms  %.2f groups per clk per SM\n", ms, ops / (ms * 1e-3) / 1.965e9 / 148);
    cudaEventRecord(e0);
    k_f32<<<blocks, thr>>>((float*)d, n, 0.999999f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA: %.3f ms  %.1f per clk per SM\n", ms, ops / (ms * 1e-3) / 1.965e9 / 148);
  }
  return 0;
}
