// Per-step cost of a barrier-synchronised loop where each warp updates K register-held
// row chunks per step (LDS V[t] + broadcast LDS V[i], 3 DMUL, DADD), thread 0 doing a
// sqrt + div pivot chain; 1 CTA of NT threads.  Prints cycles per step.
#include <cstdio>
#include <cuda_runtime.h>
template <int NT, int K>
__global__ void k(double* out, long long* cyc, int steps, int mode) {
  __shared__ double dg[1024];
  __shared__ double V[2][256];
  double X[K];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int u = 0; u < K; ++u) X[u] = threadIdx.x + u;
  if (threadIdx.x < 256) V[0][threadIdx.x] = 1.0 + threadIdx.x * 1e-3, V[1][threadIdx.x] = 1.0;
  if (threadIdx.x < 1024) dg[threadIdx.x] = 0.5;
  __syncthreads();
  long long t0 = clock64();
  for (int j = 0; j < steps; ++j) {
    __syncthreads();
    const double rl = dg[j];
    if (rl != rl) break;
    const double* Vj = V[j & 1];
    if (threadIdx.x == 0 && mode >= 1) {
      const double v = Vj[j + 1] * rl + 3.0;
      const double l = sqrt(v);
      dg[j + 1] = 1.0 / l * 0.25 + 0.375;
    }
    if (mode >= 2 && warp > 0) {
#pragma unroll
      for (int u = 0; u < K; ++u) {
        const int i = (warp * 7 + u * 13) & 127;
        const int t = (lane + u * 32) & 127;
        const double x = Vj[t] * rl;
        const double lij = Vj[i] * rl;
        X[u] = __dsub_rn(X[u], __dmul_rn(lij, x));
      }
    }
  }
  long long t1 = clock64();
  double a = 0;
#pragma unroll
  for (int u = 0; u < K; ++u) a += X[u];
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / steps;
}
template <int NT, int K>
void run(double* o, long long* c, int mode) {
  k<NT, K><<<1, NT>>>(o, c, 70, mode);
  cudaDeviceSynchronize();
  printf("NT=%4d K=%2d mode=%d: %lld cyc/step\n", NT, K, mode, c[0]);
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 8 * 1024); cudaMallocManaged(&c, 8 * 8);
  for (int m = 0; m < 3; ++m) {
    run<512, 1>(o, c, m); run<512, 2>(o, c, m); run<512, 4>(o, c, m); run<512, 8>(o, c, m);
    run<512, 16>(o, c, m); run<256, 8>(o, c, m); run<128, 8>(o, c, m); run<1024, 4>(o, c, m);
  }
  return 0;
}
