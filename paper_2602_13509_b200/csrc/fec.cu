// GF(256) Reed-Solomon erasure code of the downlink: the product
// behind parity generation and erasure recovery, fec.py:101-195 / _accel.py:50-70, 92-107.
//
// gf_matmul_kernel: out[g] = M[g] (r x k) * D[g] (k x n bytes) over GF(2^8), poly 0x11D.
// Multiplication by a constant is GF(2)-linear, so it is done bit-sliced, 8 bytes per
// thread: for each data row j the thread turns its bytes into eight byte masks (mask_b =
// bit b of every byte replicated, one SHF + one PRMT sign-replicate each), and every output
// row i accumulates acc ^= mask_b & C[i][j][b], where C[i][j][b] = m_ij * 2^b replicated to
// four bytes lives in shared memory (broadcast reads, no table lookups, no bank conflicts):
// 8 LOP3 per 4 byte products. Data rows are read once per row tile, coalesced.
//
// gf_invert_kernel: Gauss-Jordan of the k x k matrix formed by chosen rows of an encoding
// matrix (fec.py:82-98, same pivot rule: first nonzero at or below the diagonal), one CTA per
// problem, in shared memory; only the requested rows of the inverse are written (the erased
// data slots, fec.py:188-191), zero rows after them so a batch shares one matmul launch.
#include "common.cuh"

namespace skyrx {

constexpr int kGfRowTile = 4;     // output rows per CTA
constexpr int kGfThreads = 128;   // 8 bytes per thread -> 1 KB of columns per CTA

// bit b of each byte of x replicated over that byte
__device__ __forceinline__ uint32_t bitmask_bytes(uint32_t x, int b) {
  uint32_t y = x << (7 - b), r;
  asm("prmt.b32 %0, %1, %1, 0xBA98;" : "=r"(r) : "r"(y));
  return r;
}

__device__ __forceinline__ uint32_t lop_xor_and(uint32_t acc, uint32_t m, uint32_t c) {
  return acc ^ (m & c);
}

__global__ void __launch_bounds__(kGfThreads)
gf_matmul_kernel(const uint8_t* __restrict__ mat, int64_t mat_gstride, int r, int k,
                 const uint8_t* __restrict__ data, int64_t dpitch, int64_t d_gstride, int64_t n,
                 uint8_t* __restrict__ out, int64_t opitch, int64_t o_gstride) {
  extern __shared__ uint4 gf_smem[];
  uint4* C = gf_smem;  // [kGfRowTile][k][2] : C[i][j] = 8 u32 (bits 0..7)
  const int g = blockIdx.z;
  const int i0 = blockIdx.y * kGfRowTile;
  const int rows = min(kGfRowTile, r - i0);
  const uint8_t* M = mat + g * mat_gstride;
  for (int e = threadIdx.x; e < kGfRowTile * k; e += blockDim.x) {
    const int i = e / k, j = e % k;
    const uint32_t m = i < rows ? M[(int64_t)(i0 + i) * k + j] : 0u;
    uint32_t v[8], x = m;
#pragma unroll
    for (int b = 0; b < 8; ++b) {  // m * 2^b: repeated xtime
      v[b] = x * 0x01010101u;
      x = (x << 1) ^ ((x & 0x80u) ? 0x11Du : 0u);
    }
    C[2 * e] = make_uint4(v[0], v[1], v[2], v[3]);
    C[2 * e + 1] = make_uint4(v[4], v[5], v[6], v[7]);
  }
  __syncthreads();

  const int64_t col = (blockIdx.x * (int64_t)kGfThreads + threadIdx.x) * 8;
  if (col >= n) return;
  const uint8_t* D = data + g * d_gstride + col;
  const bool full = col + 8 <= n && ((reinterpret_cast<uintptr_t>(D) | dpitch) & 7) == 0;
  uint32_t acc[kGfRowTile][2];
#pragma unroll
  for (int i = 0; i < kGfRowTile; ++i) acc[i][0] = acc[i][1] = 0u;
  auto load = [&](int j) -> uint2 {
    const uint8_t* src = D + j * dpitch;
    if (full) return __ldg(reinterpret_cast<const uint2*>(src));
    uint32_t w[2] = {0u, 0u};
    for (int t = 0; t < 8 && col + t < n; ++t) w[t >> 2] |= (uint32_t)src[t] << (8 * (t & 3));
    return make_uint2(w[0], w[1]);
  };
  // data rows kGfPrefetch ahead: the loop is otherwise one exposed L2/HBM latency per row
  constexpr int kGfPrefetch = 4;
  uint2 buf[kGfPrefetch];
#pragma unroll
  for (int q = 0; q < kGfPrefetch; ++q) buf[q] = q < k ? load(q) : make_uint2(0u, 0u);
  for (int j0 = 0; j0 < k; j0 += kGfPrefetch) {
#pragma unroll
   for (int q = 0; q < kGfPrefetch; ++q) {
    const int j = j0 + q;
    if (j >= k) break;
    const uint32_t x0 = buf[q].x, x1 = buf[q].y;
    if (j + kGfPrefetch < k) buf[q] = load(j + kGfPrefetch);
    uint32_t m0[8], m1[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) m0[b] = bitmask_bytes(x0, b), m1[b] = bitmask_bytes(x1, b);
    const uint4* Cj = C + 2 * j;
#pragma unroll
    for (int i = 0; i < kGfRowTile; ++i) {
      const uint4 lo = Cj[2 * i * k], hi = Cj[2 * i * k + 1];
      const uint32_t c[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        acc[i][0] = lop_xor_and(acc[i][0], m0[b], c[b]);
        acc[i][1] = lop_xor_and(acc[i][1], m1[b], c[b]);
      }
    }
   }
  }
  uint8_t* O = out + g * o_gstride + col;
  const bool ofull = col + 8 <= n && ((reinterpret_cast<uintptr_t>(O) | opitch) & 7) == 0;
#pragma unroll
  for (int i = 0; i < kGfRowTile; ++i) {
    if (i >= rows) break;
    uint8_t* dst = O + (int64_t)(i0 + i) * opitch;
    if (ofull) {
      *reinterpret_cast<uint2*>(dst) = make_uint2(acc[i][0], acc[i][1]);
    } else {
      for (int t = 0; t < 8 && col + t < n; ++t) dst[t] = (uint8_t)(acc[i][t >> 2] >> (8 * (t & 3)));
    }
  }
}

constexpr int kGfInvThreads = 512;

__global__ void __launch_bounds__(kGfInvThreads)
gf_invert_kernel(const uint8_t* __restrict__ mat, int ld, const int32_t* __restrict__ rows, int k,
                 const int32_t* __restrict__ sel, const int32_t* __restrict__ nsel,
                 uint8_t* __restrict__ out, int32_t* __restrict__ status) {
  extern __shared__ uint8_t inv_smem[];
  const int g = blockIdx.x, w2 = 2 * k;
  uint8_t* A = inv_smem;                 // [k][2k]: [m | I]
  uint8_t* F = A + k * w2;               // elimination factors of the pivot column
  uint8_t* gexp = F + ((k + 15) & ~15);  // 512-entry antilog
  uint8_t* glog = gexp + 512;            // 256-entry log
  __shared__ int piv;
  __shared__ uint8_t pinv;
  const int tid = threadIdx.x;
  if (tid == 0) {
    uint32_t v = 1;
    for (int e = 0; e < 255; ++e) {
      gexp[e] = gexp[e + 255] = (uint8_t)v;
      glog[v] = (uint8_t)e;
      v = (v << 1) ^ ((v & 0x80u) ? 0x11Du : 0u);
    }
    gexp[510] = gexp[511] = 0;
    glog[0] = 0;
  }
  for (int e = tid; e < k * w2; e += blockDim.x) {
    const int i = e / w2, c = e % w2;
    A[e] = c < k ? mat[(int64_t)rows[g * k + i] * ld + c] : (uint8_t)(c - k == i);
  }
  __syncthreads();
  auto mul = [&](uint32_t a, uint32_t b) -> uint8_t {
    return (a && b) ? gexp[glog[a] + glog[b]] : (uint8_t)0;
  };
  for (int c = 0; c < k; ++c) {
    if (tid == 0) piv = k;
    __syncthreads();
    for (int i = c + tid; i < k; i += blockDim.x)
      if (A[i * w2 + c]) atomicMin(&piv, i);
    __syncthreads();
    const int p = piv;
    if (p == k) {  // singular: uniform exit
      if (tid == 0) status[g] = 1;
      return;
    }
    if (p != c)
      for (int e = tid; e < w2; e += blockDim.x) {
        const uint8_t t = A[c * w2 + e];
        A[c * w2 + e] = A[p * w2 + e];
        A[p * w2 + e] = t;
      }
    __syncthreads();
    if (tid == 0) pinv = gexp[255 - glog[A[c * w2 + c]]];
    __syncthreads();
    for (int e = tid; e < w2; e += blockDim.x) A[c * w2 + e] = mul(A[c * w2 + e], pinv);
    for (int i = tid; i < k; i += blockDim.x) F[i] = i == c ? (uint8_t)0 : A[i * w2 + c];
    __syncthreads();
    for (int e = tid; e < k * w2; e += blockDim.x) {
      const int i = e / w2;
      const uint8_t f = F[i];
      if (f) A[e] ^= mul(f, A[c * w2 + (e % w2)]);
    }
    __syncthreads();
  }
  const int ns = nsel[g];
  uint8_t* O = out + (int64_t)g * k * k;
  for (int e = tid; e < k * k; e += blockDim.x) {
    const int i = e / k, c = e % k;
    O[e] = i < ns ? A[sel[g * k + i] * w2 + k + c] : (uint8_t)0;
  }
  if (tid == 0) status[g] = 0;
}

}  // namespace skyrx

using namespace skyrx;

extern "C" int skyrx_gf_matmul(const uint8_t* mat, int64_t mat_gstride, int r, int k,
                               const uint8_t* data, int64_t dpitch, int64_t d_gstride, int64_t n,
                               uint8_t* out, int64_t opitch, int64_t o_gstride, int groups,
                               void* stream) {
  SKYRX_REQUIRE(r >= 1 && k >= 1 && k <= 256 && groups >= 1 && n >= 0, "bad GF matmul shape");
  SKYRX_REQUIRE(dpitch >= n && opitch >= n, "row pitch below row length");
  if (n == 0) return SKYRX_OK;
  const size_t smem = (size_t)kGfRowTile * k * 32;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(gf_matmul_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((unsigned)((n + 8 * kGfThreads - 1) / (8 * kGfThreads)),
            (unsigned)((r + kGfRowTile - 1) / kGfRowTile), (unsigned)groups);
  gf_matmul_kernel<<<grid, kGfThreads, smem, as_stream(stream)>>>(
      mat, mat_gstride, r, k, data, dpitch, d_gstride, n, out, opitch, o_gstride);
  SKYRX_CHECK_LAUNCH("gf_matmul_kernel");
  return SKYRX_OK;
}

extern "C" int skyrx_gf_invert(const uint8_t* mat, int ld, const int32_t* rows, int k,
                               const int32_t* sel, const int32_t* nsel, int groups, uint8_t* out,
                               int32_t* status, void* stream) {
  SKYRX_REQUIRE(k >= 1 && k <= 256 && ld >= k && groups >= 1, "bad GF inverse shape");
  const size_t smem = (size_t)k * 2 * k + ((k + 15) & ~15) + 768;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(gf_invert_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  gf_invert_kernel<<<groups, kGfInvThreads, smem, as_stream(stream)>>>(mat, ld, rows, k, sel, nsel,
                                                                      out, status);
  SKYRX_CHECK_LAUNCH("gf_invert_kernel");
  return SKYRX_OK;
}
