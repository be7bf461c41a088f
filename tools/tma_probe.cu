// Raw-streaming probe: how fast can one persistent CTA per SM pull a 2 GB u16
// cube into shared memory with 1-D bulk copies, for the tile orders the score
// and moments kernels use?  Compare with a plain LDG.128 streaming read.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tma_probe tools/tma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2602_13509_b200/csrc/tma.cuh"
using namespace skyrx::umma;
using skyrx::tma_load_2d;

__global__ void ldg_kernel(const uint4* __restrict__ p, size_t n, unsigned long long* out) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldg(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) atomicAdd(out, 1ull);
}

// mode 0: tile t = chunk (blockIdx + t*grid) of consecutive `seg`-byte chunks (streaming)
// mode 1: score order: tile = line (round-robin) of sample block b: addr = line*pitch + b*seg
// nseg: copies per tile (mode 2: 4 lines x seg)
__global__ void bulk_kernel(const uint8_t* base, int mode, uint32_t seg, int lines_per_tile,
                            int64_t lines, int64_t pitch, int nblocks, int64_t ntiles, int nst,
                            unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + nst * seg * lines_per_tile);
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int64_t n = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  uint32_t acc = 0;
  auto issue = [&](int64_t t) {
    const int s = t % nst;
    const int64_t item = blockIdx.x + t * gridDim.x;
    mbar_arrive_expect_tx(&full[s], seg * lines_per_tile);
    for (int li = 0; li < lines_per_tile; ++li) {
      const uint8_t* src;
      if (mode == 0) src = base + (item * lines_per_tile + li) * (int64_t)seg;
      else {
        const int64_t per_block = lines / lines_per_tile;
        const int64_t b = item / per_block, g = item % per_block;
        src = base + (g * lines_per_tile + li) * pitch + b * (int64_t)seg;
      }
      bulk_g2s(sm + (s * lines_per_tile + li) * seg, src, seg, &full[s]);
    }
  };
  for (int64_t t = 0; t < n && t < nst; ++t) issue(t);
  for (int64_t t = 0; t < n; ++t) {
    const int s = t % nst;
    mbar_wait(&full[s], (t / nst) & 1);
    acc += sm[s * seg * lines_per_tile + 5];
    if (t + nst < n) issue(t + nst);
  }
  if (acc == 0xFFFFFFFFu) atomicAdd(out, 1ull);
}

// gram_raw order: unit u -> (window w = u % nwin, line split = u / nwin); each tile = a
// box of `boxw` bytes x `boxl` lines at byte offset w*winstride of each line (2-D map)
__global__ void tensor_kernel(const __grid_constant__ CUtensorMap map, int nwin, int winstride,
                              int boxw, int boxl, int natom, int64_t lines, int nst,
                              unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t stage = (uint32_t)boxw * boxl * natom;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + nst * stage);
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int64_t per = lines / boxl;
  const int64_t ntiles = (int64_t)nwin * per;
  int64_t n = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  uint32_t acc = 0;
  auto issue = [&](int64_t t) {
    const int s = t % nst;
    const int64_t item = blockIdx.x + t * gridDim.x;
    const int w = item % nwin;
    const int64_t g = item / nwin;
    mbar_arrive_expect_tx(&full[s], stage);
    for (int a = 0; a < natom; ++a)
      tma_load_2d(sm + s * stage + a * boxw * boxl, &map, ((w * winstride) & ~15) + a * boxw, (int)(g * boxl),
                  &full[s]);
  };
  for (int64_t t = 0; t < n && t < nst; ++t) issue(t);
  for (int64_t t = 0; t < n; ++t) {
    const int s = t % nst;
    mbar_wait(&full[s], (t / nst) & 1);
    acc += sm[s * stage + 5];
    if (t + nst < n) issue(t + nst);
  }
  if (acc == 0xFFFFFFFFu) atomicAdd(out, 1ull);
}

int main() {
  const int64_t L = 16384, S = 900, B = 70;
  const int64_t pitch = S * B * 2;        // 126000 B per line
  const size_t bytes = (size_t)L * pitch;  // 2.06 GB
  uint8_t* buf;
  unsigned long long* out;
  cudaMalloc(&buf, bytes + (1 << 20));
  cudaMalloc(&out, 8);
  cudaMemset(buf, 1, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto time = [&](auto fn) {
    fn();
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) fn();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
  };
  float ms = time([&] { ldg_kernel<<<148 * 8, 512>>>((const uint4*)buf, bytes / 16, out); });
  printf("ldg128 stream: %.3f ms  %.0f GB/s\n", ms, bytes / ms / 1e6);
  struct Cfg { int mode; uint32_t seg; int lpt; int nst; const char* name; };
  Cfg cfgs[] = {
      {0, 17920, 1, 4, "contiguous 17.9KB x4"},  {0, 17920, 1, 8, "contiguous 17.9KB x8"},
      {0, 8192, 1, 16, "contiguous 8KB x16"},    {0, 32768, 1, 4, "contiguous 32KB x4"},
      {1, 17920, 1, 4, "score W=128 x4"},        {1, 17920, 1, 8, "score W=128 x8"},
      {1, 4480, 4, 4, "score W=32 4 lines x4"},  {1, 4480, 4, 8, "score W=32 4 lines x8"},
      {1, 8960, 2, 6, "W=64 2 lines x6"},
  };
  for (auto& c : cfgs) {
    int64_t ntiles = c.mode == 0 ? bytes / (c.seg * (size_t)c.lpt)
                                 : (pitch / (c.seg)) * (L / c.lpt);
    size_t smem = (size_t)c.nst * c.seg * c.lpt + 8 * c.nst + 64;
    if (smem > 232448) { printf("%s: smem too big\n", c.name); continue; }
    cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    ms = time([&] {
      bulk_kernel<<<148, 32, smem>>>(buf, c.mode, c.seg, c.lpt, L, pitch, (int)(pitch / c.seg),
                                     ntiles, c.nst, out);
    });
    double moved = (double)ntiles * c.seg * c.lpt;
    printf("%-28s %.3f ms  %.0f GB/s  (%.2f GB)\n", c.name, ms, moved / ms / 1e6, moved / 1e9);
  }
  {
    struct TC { int boxw, boxl, natom, nst, swz; const char* name; };
    TC tcs[] = {{128, 128, 2, 4, 1, "gram: 2x(128B x128 lines) sw128 x4"},
                {128, 256, 2, 3, 1, "gram: 2x(128B x256 lines) sw128 x3"},
                {128, 64, 2, 8, 1, "gram: 2x(128B x64 lines) sw128 x8"},
                {256, 64, 1, 8, 0, "256B x 64 lines x8"}};
    for (auto& c : tcs) {
      const cuuint64_t line_bytes = (cuuint64_t)pitch;
      cuuint64_t dims[2] = {line_bytes, (cuuint64_t)L};
      cuuint64_t strides[1] = {line_bytes};
      cuuint32_t box[2] = {(cuuint32_t)c.boxw, (cuuint32_t)c.boxl};
      cuuint32_t estr[2] = {1, 1};
      CUtensorMap map;
      CUresult r = skyrx::tensor_map_encoder()(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims,
          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          c.swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("%s: encode failed %d\n", c.name, (int)r); continue; }
      const int nwin = 900;  // one window per sample (140 B of 2 x 128 B boxes)
      size_t smem = (size_t)c.nst * c.boxw * c.boxl * c.natom + 8 * c.nst + 64;
      cudaFuncSetAttribute(tensor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      ms = time([&] { tensor_kernel<<<148, 32, smem>>>(map, nwin, 140, c.boxw, c.boxl, c.natom, L,
                                                         c.nst, out); });
      double moved = (double)nwin * (L / c.boxl) * c.boxl * c.boxw * c.natom;
      printf("%-36s %.3f ms  %.0f GB/s fetched (%.2f GB), useful %.0f GB/s\n", c.name, ms,
             moved / ms / 1e6, moved / 1e9, (double)bytes / ms / 1e6);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
