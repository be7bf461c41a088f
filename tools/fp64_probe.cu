// FP64 throughput / latency probe: DFMA chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* out, int iters, double a, double b) {
  double x[CH];
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  double s = 0;
  for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
void run(int blocks, int threads) {
  double* o; cudaMalloc(&o, blocks * threads * 8);
  int iters = 4096;
  k<CH><<<blocks, threads>>>(o, iters, 1.0000001, 1e-9);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<CH><<<blocks, threads>>>(o, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double dfma = (double)blocks * threads * iters * CH;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("CH=%d blocks=%d threads=%d: %.3f ms, %.1f GDFMA/s, %.2f DFMA/clk/SM (clk %d MHz)\n", CH,
         blocks, threads, ms, dfma / ms / 1e6, dfma / (ms * 1e-3) / (clk * 1e3) / 148, clk / 1000);
  cudaFree(o);
}
int main() {
  run<1>(148, 32);    // latency: one warp per SM, one chain
  run<4>(148, 32);
  run<8>(148, 128);
  run<8>(148 * 4, 256);
  return 0;
}
