// Hardware probe for the hand-written tcgen05 layer (csrc/umma.cuh).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I include \
//        tools/umma_probe.cu -o build/umma_probe && build/umma_probe
// Checks (1) f16 K-major x K-major, (2) s8 MN-major x MN-major descriptor
// encodings against a CPU GEMM, and (3) how the f32 accumulator rounds
// (round-to-nearest vs truncation) — the precision budget of DESIGN.md
// depends on it.
#include <cuda_fp16.h>
#include <stdio.h>
#include <stdlib.h>

#include <cmath>
#include <vector>

#include "../paper_2602_13509_b200/csrc/umma.cuh"

using namespace skyrx::umma;

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

// generic probe kernel: copies pre-laid-out operand bytes to smem, runs a list
// of MMAs, dumps D (128 lanes x ncols f32/s32) to global
struct MmaOp {
  uint32_t a_off, b_off, lbo_a, sbo_a, lbo_b, sbo_b, idesc, dcol, accumulate, kind;  // kind 0 f16, 1 i8
};

__global__ void probe_kernel(const uint8_t* __restrict__ ops_bytes, int nbytes, const MmaOp* ops,
                             int nops, int ncols, uint32_t* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t taddr_s;
  for (int i = threadIdx.x; i < nbytes; i += blockDim.x) sm[i] = ops_bytes[i];
  fence_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if ((threadIdx.x >> 5) == 0) tmem_alloc(&taddr_s, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = taddr_s;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nops; ++i) {
      const MmaOp o = ops[i];
      const uint64_t a = smem_desc(sm + o.a_off, o.lbo_a, o.sbo_a);
      const uint64_t b = smem_desc(sm + o.b_off, o.lbo_b, o.sbo_b);
      if (o.kind == 0) mma_f16(tbase + o.dcol, a, b, o.idesc, o.accumulate);
      else mma_i8(tbase + o.dcol, a, b, o.idesc, o.accumulate);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int w = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int c = 0; c < ncols; c += 16) {
    uint32_t r[16];
    tmem_ld16(tbase + ((uint32_t)(32 * w) << 16) + c, r);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) out[(32 * w + lane) * ncols + c + j] = r[j];
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(tbase, 512);
}

static void run(std::vector<uint8_t>& bytes, std::vector<MmaOp>& ops, int ncols,
                std::vector<uint32_t>& out) {
  uint8_t* db;
  MmaOp* dops;
  uint32_t* dout;
  CK(cudaMalloc(&db, bytes.size()));
  CK(cudaMalloc(&dops, ops.size() * sizeof(MmaOp)));
  CK(cudaMalloc(&dout, 128 * ncols * 4));
  CK(cudaMemcpy(db, bytes.data(), bytes.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dops, ops.data(), ops.size() * sizeof(MmaOp), cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000));
  probe_kernel<<<1, 128, bytes.size()>>>(db, (int)bytes.size(), dops, (int)ops.size(), ncols, dout);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  out.resize(128 * ncols);
  CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
  cudaFree(db);
  cudaFree(dops);
  cudaFree(dout);
}

static uint16_t h16(float f) {
  __half h = __float2half_rn(f);
  return *reinterpret_cast<uint16_t*>(&h);
}

int test_f16_kmajor() {
  const int M = 128, N = 80, K = 80;
  std::vector<float> A(M * K), B(N * K);
  srand(1);
  for (auto& v : A) v = (float)((rand() % 2001) - 1000) / 64.0f;  // exact in f16
  for (auto& v : B) v = (float)((rand() % 2001) - 1000) / 128.0f;
  // K-major interleave: (r/8)*SBO + (k/8)*LBO + (r%8)*16 + (k%8)*2 ; LBO=128, SBO=(K/8)*128
  const uint32_t LBO = 128, SBO_A = (K / 8) * 128, SBO_B = (K / 8) * 128;
  const uint32_t a_off = 0, b_off = M * K * 2;
  std::vector<uint8_t> bytes(b_off + N * K * 2 + 4096, 0);
  auto put = [&](uint32_t base, uint32_t sbo, int r, int k, float v) {
    uint16_t h = h16(v);
    uint32_t off = base + (r / 8) * sbo + (k / 8) * LBO + (r % 8) * 16 + (k % 8) * 2;
    bytes[off] = h & 0xff;
    bytes[off + 1] = h >> 8;
  };
  for (int r = 0; r < M; ++r)
    for (int k = 0; k < K; ++k) put(a_off, SBO_A, r, k, A[r * K + k]);
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) put(b_off, SBO_B, n, k, B[n * K + k]);
  std::vector<MmaOp> ops;
  for (int ks = 0; ks < K / 16; ++ks)
    ops.push_back({a_off + ks * 2 * LBO, b_off + ks * 2 * LBO, LBO, SBO_A, LBO, SBO_B,
                   idesc_f16_f32(M, N, 0, 0), 0, (uint32_t)(ks > 0), 0});
  std::vector<uint32_t> out;
  run(bytes, ops, 80, out);
  double maxerr = 0;
  for (int r = 0; r < M; ++r)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)A[r * K + k] * B[n * K + k];
      float got;
      memcpy(&got, &out[r * 80 + n], 4);
      maxerr = fmax(maxerr, fabs(got - ref));
    }
  printf("f16 K-major 128x80x80: max abs err %.3g %s\n", maxerr, maxerr < 1e-2 ? "OK" : "FAIL");
  return maxerr < 1e-2;
}

// A from TMEM (tcgen05.st by the 128 threads, 2 f16 per 32-bit column, even k
// in the low half) x B K-major in smem: the layout the score kernel relies on
__global__ void ts_kernel(const uint32_t* __restrict__ apack, const uint8_t* __restrict__ bbytes,
                          int nb, int K, int N, uint32_t idesc, uint32_t* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t taddr_s;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) sm[i] = bbytes[i];
  fence_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if ((threadIdx.x >> 5) == 0) tmem_alloc(&taddr_s, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = taddr_s;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, r = threadIdx.x;
  const uint32_t lanebase = tbase + ((uint32_t)(32 * w) << 16);
  // A occupies columns [256, 256 + K/2)
  for (int c = 0; c < K / 2; c += 4)
    tmem_st4(lanebase + 256 + c, apack[r * (K / 2) + c], apack[r * (K / 2) + c + 1],
             apack[r * (K / 2) + c + 2], apack[r * (K / 2) + c + 3]);
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t SBO = (K / 8) * 128;
    for (int ks = 0; ks < K / 16; ++ks)
      mma_f16_ts(tbase, tbase + 256 + ks * 8, smem_desc(sm + ks * 256, 128, SBO), idesc, ks > 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < N; c += 16) {
    uint32_t v[16];
    tmem_ld16(lanebase + c, v);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) out[r * N + c + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(tbase, 512);
}

int test_f16_a_in_tmem() {
  const int M = 128, N = 80, K = 80;
  std::vector<float> A(M * K), B(N * K);
  srand(3);
  for (auto& v : A) v = (float)((rand() % 2001) - 1000) / 64.0f;
  for (auto& v : B) v = (float)((rand() % 2001) - 1000) / 128.0f;
  std::vector<uint32_t> apack(M * K / 2);
  for (int r = 0; r < M; ++r)
    for (int k = 0; k < K; k += 2)
      apack[r * (K / 2) + k / 2] = (uint32_t)h16(A[r * K + k]) | ((uint32_t)h16(A[r * K + k + 1]) << 16);
  const uint32_t LBO = 128, SBO = (K / 8) * 128;
  std::vector<uint8_t> bytes(N * K * 2, 0);
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) {
      uint16_t h = h16(B[n * K + k]);
      uint32_t off = (n / 8) * SBO + (k / 8) * LBO + (n % 8) * 16 + (k % 8) * 2;
      bytes[off] = h & 0xff;
      bytes[off + 1] = h >> 8;
    }
  uint32_t *da, *dout;
  uint8_t* db;
  CK(cudaMalloc(&da, apack.size() * 4));
  CK(cudaMalloc(&db, bytes.size()));
  CK(cudaMalloc(&dout, M * N * 4));
  CK(cudaMemcpy(da, apack.data(), apack.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, bytes.data(), bytes.size(), cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(ts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000));
  ts_kernel<<<1, 128, bytes.size()>>>(da, db, (int)bytes.size(), K, N, idesc_f16_f32(M, N, 0, 0),
                                      dout);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<uint32_t> out(M * N);
  CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0;
  for (int r = 0; r < M; ++r)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)A[r * K + k] * B[n * K + k];
      float got;
      memcpy(&got, &out[r * N + n], 4);
      maxerr = fmax(maxerr, fabs(got - ref));
    }
  printf("f16 A-in-TMEM 128x80x80: max abs err %.3g %s\n", maxerr, maxerr < 1e-2 ? "OK" : "FAIL");
  return maxerr < 1e-2;
}

int test_i8_mnmajor() {
  // Gram-shaped: A = D^T (M = bands, MN-major), B = D^T (N = bands), K = pixels
  const int M = 128, N = 80, K = 128, MV = 80;
  std::vector<int> D(K * MV);
  srand(2);
  for (auto& v : D) v = (rand() % 255) - 127;
  // MN-major interleave: (mn/16)*SBO + (k/8)*LBO + (k%8)*16 + (mn%16); SBO=128, LBO=(MV/16)*128
  const uint32_t SBO = 128, LBO = (MV / 16) * 128;
  std::vector<uint8_t> bytes(K / 8 * LBO + 8192, 0x7f);  // junk beyond the valid bands
  for (int k = 0; k < K; ++k)
    for (int m = 0; m < MV; ++m)
      bytes[(m / 16) * SBO + (k / 8) * LBO + (k % 8) * 16 + (m % 16)] = (uint8_t)(int8_t)D[k * MV + m];
  std::vector<MmaOp> ops;
  for (int ks = 0; ks < K / 32; ++ks)
    ops.push_back({ks * 4 * LBO, ks * 4 * LBO, LBO, SBO, LBO, SBO, idesc_s8_s32(M, N, 1, 1), 0,
                   (uint32_t)(ks > 0), 1});
  std::vector<uint32_t> out;
  run(bytes, ops, 80, out);
  long bad = 0;
  for (int i = 0; i < MV; ++i)
    for (int j = 0; j < N; ++j) {
      long ref = 0;
      for (int k = 0; k < K; ++k) ref += (long)D[k * MV + i] * D[k * MV + j];
      if ((int32_t)out[i * 80 + j] != ref) ++bad;
    }
  printf("s8 MN-major Gram 80x80 over 128 px: %ld mismatches %s\n", bad, bad ? "FAIL" : "OK");
  return bad == 0;
}

void test_rounding() {
  // D = sum of products; inspect how f32 accumulation rounds
  const int M = 128, N = 16, K = 16;
  struct Case {
    const char* name;
    float a[4], b[4];
    int split;  // 1: product 0 in first MMA, rest accumulated by a second MMA
  } cases[] = {
      {"1 + 0.75ulp in one MMA", {1.f, 3.f / 8192.f, 0, 0}, {1.f, 1.f / 4096.f, 0, 0}, 0},
      {"1 + 0.75ulp across MMAs", {1.f, 3.f / 8192.f, 0, 0}, {1.f, 1.f / 4096.f, 0, 0}, 1},
      {"1 + 0.25ulp across MMAs", {1.f, 1.f / 8192.f, 0, 0}, {1.f, 1.f / 4096.f, 0, 0}, 1},
      {"-1 - 0.75ulp across MMAs", {-1.f, -3.f / 8192.f, 0, 0}, {1.f, 1.f / 4096.f, 0, 0}, 1},
      {"1 + 3 x 0.375ulp in one MMA", {1.f, 3.f / 16384.f, 3.f / 16384.f, 3.f / 16384.f},
       {1.f, 1.f / 4096.f, 1.f / 4096.f, 1.f / 4096.f}, 0},
  };
  for (auto& c : cases) {
    const uint32_t LBO = 128, SBO = 256;
    std::vector<uint8_t> bytes(2 * M * K * 2 + 4096, 0);
    const uint32_t b_off = M * K * 2;
    auto put = [&](uint32_t base, int r, int k, float v) {
      uint16_t h = h16(v);
      uint32_t off = base + (r / 8) * SBO + (k / 8) * LBO + (r % 8) * 16 + (k % 8) * 2;
      bytes[off] = h & 0xff;
      bytes[off + 1] = h >> 8;
    };
    // operand copy 1 (first MMA) at offset 0 / b_off; copy 2 for the split case after
    const uint32_t a2 = 2 * M * K * 2 + 0, b2 = a2 + M * K * 2;
    bytes.resize(b2 + M * K * 2 + 4096, 0);
    for (int k = 0; k < 4; ++k) {
      if (c.split) {
        if (k == 0) {
          put(0, 0, 0, c.a[0]);
          put(b_off, 0, 0, c.b[0]);
        } else {
          put(a2, 0, k, c.a[k]);
          put(b2, 0, k, c.b[k]);
        }
      } else {
        put(0, 0, k, c.a[k]);
        put(b_off, 0, k, c.b[k]);
      }
    }
    std::vector<MmaOp> ops;
    ops.push_back({0, b_off, LBO, SBO, LBO, SBO, idesc_f16_f32(M, N, 0, 0), 0, 0, 0});
    if (c.split) ops.push_back({a2, b2, LBO, SBO, LBO, SBO, idesc_f16_f32(M, N, 0, 0), 0, 1, 0});
    std::vector<uint32_t> out;
    run(bytes, ops, 16, out);
    float got;
    memcpy(&got, &out[0], 4);
    double exact = 0;
    for (int k = 0; k < 4; ++k) exact += (double)c.a[k] * c.b[k];
    float rn = (float)exact;
    printf("rounding %-30s got %.10g (bits %08x)  RN %.10g  trunc %.10g\n", c.name, got, out[0],
           rn, (double)(exact > 0 ? nextafterf(rn, 0) : nextafterf(rn, 0)));
  }
}

int main() {
  int ok = test_f16_kmajor();
  ok &= test_i8_mnmajor();
  ok &= test_f16_a_in_tmem();
  test_rounding();
  printf(ok ? "PROBE OK\n" : "PROBE FAIL\n");
  return ok ? 0 : 1;
}
