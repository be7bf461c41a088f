// Latency of dependent FP64 sqrt / division / DFMA chains (one thread), in clock cycles.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double x, int n) {
  double a = x, b = x, c = x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = sqrt(a + 1.0);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) b = 1.0 / (b + 1.0);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) c = fma(c, 0.999, 1e-3);
  long long t3 = clock64();
  volatile __shared__ double s[64];
  s[threadIdx.x] = x;
  __syncthreads();
  long long t4 = clock64();
  double d = 0;
  for (int i = 0; i < n; ++i) d += s[(int)d & 7];
  long long t5 = clock64();
  out[0] = a + b + c + d;
  cyc[0] = (t1 - t0) / n, cyc[1] = (t2 - t1) / n, cyc[2] = (t3 - t2) / n, cyc[3] = (t5 - t4) / n;
}
__global__ void kb(long long* cyc, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0) / n;
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 8); cudaMallocManaged(&c, 8 * 8);
  k<<<1, 1>>>(o, c, 2.0, 1000);
  kb<<<1, 1024>>>(c, 1000);
  cudaDeviceSynchronize();
  printf("cycles per dependent op: sqrt %lld, div %lld, dfma %lld, lds.64(+dadd) %lld, syncthreads(1024) %lld\n",
         c[0], c[1], c[2], c[3], c[4]);
  return 0;
}
