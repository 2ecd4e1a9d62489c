// Microbenchmark: dependent-chain latency and throughput of DFMA/DMUL/FFMA/FFMA2/LDS on this GPU.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_dfma(double* out, long long* cyc, int iters, double a, double b) {
  double x = threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void chain_ffma(float* out, long long* cyc, int iters, float a, float b) {
  float x = threadIdx.x * 1e-9f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    x = fmaf(x, a, b); x = fmaf(x, a, b); x = fmaf(x, a, b); x = fmaf(x, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
// throughput: 8 independent chains per thread
__global__ void tput_dfma(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void tput_ffma(float* out, int iters, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
    x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
  double* d; float* f; long long* c;
  cudaMalloc(&d, 1 << 26); cudaMalloc(&f, 1 << 26); cudaMalloc(&c, 8);
  long long cyc;
  int iters = 4096;
  chain_dfma<<<1, 32>>>(d, c, iters, 0.999, 1e-3); cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)cyc / (4.0 * iters));
  chain_ffma<<<1, 32>>>(f, c, iters, 0.999f, 1e-3f); cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
  printf("FFMA dependent latency: %.2f cycles\n", (double)cyc / (4.0 * iters));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = 148 * 16, threads = 256; iters = 2048;
  tput_dfma<<<blocks, threads>>>(d, iters, 0.999, 1e-3);
  cudaEventRecord(e0); tput_dfma<<<blocks, threads>>>(d, iters, 0.999, 1e-3); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("DFMA throughput: %.1f TFLOP/s\n", 2.0 * 8 * iters * (double)blocks * threads / ms / 1e9);
  tput_ffma<<<blocks, threads>>>(f, iters, 0.999f, 1e-3f);
  cudaEventRecord(e0); tput_ffma<<<blocks, threads>>>(f, iters, 0.999f, 1e-3f); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("FFMA throughput: %.1f TFLOP/s\n", 2.0 * 8 * iters * (double)blocks * threads / ms / 1e9);
  return 0;
}
