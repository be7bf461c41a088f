// latency of the f64 pivot chain (IEEE sqrt + reciprocal, -prec-sqrt/-prec-div) and of a
// 1024-thread barrier: the per-column floor of the finalize kernels
#include <cstdio>
__global__ void chain(double* out, int iters, double x0, int mode) {
  double x = x0;
  long long t0 = clock64();
  if (mode == 0) for (int i = 0; i < iters; ++i) { double l = sqrt(x); x = 1.0 / l + 1.0; }
  else if (mode == 1) for (int i = 0; i < iters; ++i) { x = sqrt(x) + 1.0; }
  else if (mode == 2) for (int i = 0; i < iters; ++i) { x = 1.0 / x + 1.0; }
  else if (mode == 3) for (int i = 0; i < iters; ++i) { double r = rsqrt(x); x = r * 3.0 + 1.0; }
  else if (mode == 4) for (int i = 0; i < iters; ++i) { x = __dmul_rn(x, 1.0000001) + 1e-9; }
  else if (mode == 5) for (int i = 0; i < iters; ++i) { __syncthreads(); x += 1.0; }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = x; out[1] = (double)(t1 - t0) / iters; }
}
int main() {
  double* d; cudaMalloc(&d, 16);
  const char* names[] = {"sqrt + 1/l chain", "sqrt chain", "1/x chain", "rsqrt chain", "dmul+dadd chain", "syncthreads x1024 thr"};
  for (int m = 0; m < 6; ++m) {
    int thr = m == 5 ? 1024 : 1;
    chain<<<1, thr>>>(d, 10, 2.0, m);
    chain<<<1, thr>>>(d, 1000, 2.0, m);
    double h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-24s %7.1f cycles/iter\n", names[m], h[1]);
  }
}
