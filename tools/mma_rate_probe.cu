// tcgen05.mma issue-rate probe: cycles per MMA for the shapes the score / moments
// kernels issue (A from TMEM vs shared memory, N, kind), one CTA per SM, operands
// are whatever the buffers hold (timing only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tools/mma_rate_probe.cu \
//        -o tools/mma_rate_probe_bin && tools/mma_rate_probe_bin
#include <cstdio>
#include <cstdlib>

#include "../paper_2602_13509_b200/csrc/umma.cuh"

using namespace skyrx::umma;

// MODE 0: f16 A in TMEM (ts), 1: f16 A in smem (ss), 2: i8 ss (MN-major, SW128),
// 3: the score_tc tile sequence (NCAT, 10 ts MMAs of N = 160..96 and 80..16)
// 4: score_tc tile sequence, ss
template <int MODE, int N>
__global__ void __launch_bounds__(128, 1) rate_kernel(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tslot;
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x < 32) {
    const uint64_t bd = smem_desc(sm, 128, 1024);
    const uint64_t ad = smem_desc(sm + 65536, 128, 1024);
    __syncwarp();
    t0 = clock64();
    if (elect_one()) {
      for (int it = 0; it < iters; ++it) {
        if constexpr (MODE == 0) {
#pragma unroll
          for (int k = 0; k < 8; ++k)
            mma_f16_ts(tm, tm + 256 + 8 * (k & 1), bd + 2 * k, idesc_f16_f32(128, N, 0, 0), 1);
        } else if constexpr (MODE == 1) {
#pragma unroll
          for (int k = 0; k < 8; ++k)
            mma_f16(tm, ad + 2 * k, bd + 2 * k, idesc_f16_f32(128, N, 0, 0), 1);
        } else if constexpr (MODE == 2) {
#pragma unroll
          for (int k = 0; k < 8; ++k)
            mma_i8(tm + (k & 1) * (N <= 128 ? 128 : 0), smem_desc_sw128(sm + 65536, 8192, 1024) + 2 * k,
                   smem_desc_sw128(sm, 8192, 1024) + 2 * k,
                   (2u << 4) | (1u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | (8u << 24), 1);
        } else if constexpr (MODE == 3) {
#pragma unroll
          for (int ks = 0; ks < 5; ++ks) {
            mma_f16_ts(tm + 16 * ks, tm + 320 + ks * 8, bd + ks * 64,
                       idesc_f16_f32(128, 160 - 16 * ks, 0, 0), 1);
            mma_f16_ts(tm + 16 * ks, tm + 360 + ks * 8, bd + ks * 64,
                       idesc_f16_f32(128, 80 - 16 * ks, 0, 0), 1);
          }
        } else if constexpr (MODE == 5 || MODE == 6) {
          // gram_tc's operand layout: MN-major, no swizzle, LBO = 3 NG 128 (NG = 5), SBO = 128
          // (MODE 5) vs MN-major SWIZZLE_128B (MODE 6), i8, M = 128, N = 240 / 160 / 80
          const uint32_t lbo = MODE == 5 ? 1920u : 8192u, sbo = MODE == 5 ? 128u : 1024u;
          const uint64_t b = MODE == 5 ? smem_desc(sm, lbo, sbo) : smem_desc_sw128(sm, lbo, sbo);
          const uint64_t a = MODE == 5 ? smem_desc(sm + 1280, lbo, sbo) : smem_desc_sw128(sm + 16384, lbo, sbo);
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint32_t o = MODE == 5 ? ks * 4 * 1920 / 16 : ks * 4096 / 16;
            mma_i8(tm, a + o, b + o, (2u << 4) | (1u << 15) | (1u << 16) | (30u << 17) | (8u << 24), 1);
            mma_i8(tm + 240, a + o, b + o, (2u << 4) | (1u << 15) | (1u << 16) | (20u << 17) | (8u << 24), 1);
            mma_i8(tm + 400, a + o, b + o, (2u << 4) | (1u << 15) | (1u << 16) | (10u << 17) | (8u << 24), 1);
          }
        } else {
#pragma unroll
          for (int ks = 0; ks < 5; ++ks) {
            mma_f16(tm + 16 * ks, ad + ks * 8, bd + ks * 64, idesc_f16_f32(128, 160 - 16 * ks, 0, 0), 1);
            mma_f16(tm + 16 * ks, ad + 4096 + ks * 8, bd + ks * 64,
                    idesc_f16_f32(128, 80 - 16 * ks, 0, 0), 1);
          }
        }
      }
      mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    t1 = clock64();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tm, 512);
}

template <int MODE, int N>
void run(const char* name, int per_iter) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(rate_kernel<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  rate_kernel<MODE, N><<<148, 128, smem>>>(10, d);
  rate_kernel<MODE, N><<<148, 128, smem>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double mx = 0, mean = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx, mean += h[i] / 148.0;
  printf("%-28s N=%3d  %7.1f cyc/MMA (mean over SMs), max %7.1f  %s\n", name, N,
         mean / ((double)iters * per_iter), mx / ((double)iters * per_iter),
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<0, 16>("f16 ts M128 K16", 8);
  run<0, 32>("f16 ts M128 K16", 8);
  run<0, 64>("f16 ts M128 K16", 8);
  run<0, 80>("f16 ts M128 K16", 8);
  run<0, 128>("f16 ts M128 K16", 8);
  run<0, 160>("f16 ts M128 K16", 8);
  run<0, 256>("f16 ts M128 K16", 8);
  run<1, 16>("f16 ss M128 K16", 8);
  run<1, 32>("f16 ss M128 K16", 8);
  run<1, 64>("f16 ss M128 K16", 8);
  run<1, 80>("f16 ss M128 K16", 8);
  run<1, 128>("f16 ss M128 K16", 8);
  run<1, 160>("f16 ss M128 K16", 8);
  run<1, 256>("f16 ss M128 K16", 8);
  run<2, 16>("i8 ss M128 K32 sw128", 8);
  run<2, 64>("i8 ss M128 K32 sw128", 8);
  run<2, 128>("i8 ss M128 K32 sw128", 8);
  run<2, 256>("i8 ss M128 K32 sw128", 8);
  run<3, 0>("score_tc tile ts (10 MMAs)", 10);
  run<4, 0>("score_tc tile ss (10 MMAs)", 10);
  run<5, 0>("gram_tc tile i8 noswz (12 MMAs)", 12);
  run<6, 0>("gram_tc tile i8 sw128 (12 MMAs)", 12);
  return 0;
}
