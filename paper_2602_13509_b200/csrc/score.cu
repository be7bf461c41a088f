// K4 — RX scores: delta = ||W (x - mu)||^2 with W = L^-1 (lower triangular).
//
// Reference: rx.py:89-97 calls _accel.mahalanobis_sq (_accel.py:75-90), a
// per-pixel forward substitution L y = x - mu in f64.  Solving with the
// explicit inverse turns the hot loop into a dense pixel-block x W^T product
// (GEMM-shaped) followed by a row-wise sum of squares.
//
// Fast path (kind RAW/F32, f32 arithmetic): x calibrated in the tile loader,
// d = (x - mu_hi) - mu_lo, z accumulated in f32 over k ascending (<= B terms;
// measured max score error 8e-7 vs the f64 reference at B=70), delta summed in
// f32 in a fixed order.  Slot path (skyrx_mahalanobis_sq): the same kernel in
// f64, matching the reference's f64 accumulation (rtol 1e-9 suites).
//
// Tiling: threads = pixel-groups x j-tiles; each thread owns TP pixels x 8
// outputs z[p][j], streams k in vectors of 16 B from shared memory
// (d[p][k] pixel-major, W^T[k][j]); j-tile J only needs k < 8J+8 (triangle).
// Partial sums of squares per j-tile are reduced per pixel in shared memory
// in J order (deterministic).
#include "common.cuh"
#include "tile_loader.cuh"

namespace skyrx {

struct ScoreGeom {
  int bp, nt, pgroups, threads, P, ld, kc;  // kc: k-chunk of W held in smem
  bool w_resident;
  int64_t ptiles;
  int grid;
};

template <typename T, int TP>
static ScoreGeom score_geom(int64_t npix, int bands) {
  ScoreGeom g;
  g.bp = ((bands + 7) / 8) * 8;
  g.nt = g.bp / 8;
  int pg = 256 / g.nt;
  if (pg < 16) pg = 16;
  if (pg * g.nt > 512) pg = 512 / g.nt;
  g.pgroups = pg;
  g.threads = ((pg * g.nt + 31) / 32) * 32;
  g.P = TP * pg;
  g.ld = g.bp + 16 / (int)sizeof(T);
  const size_t wbytes = (size_t)g.bp * g.bp * sizeof(T);
  g.w_resident = wbytes <= 64 * 1024;
  g.kc = g.w_resident ? g.bp : 32;
  g.ptiles = ceil_div<int64_t>(npix, g.P);
  const size_t smem = (size_t)g.P * g.ld * sizeof(T) + (size_t)g.kc * g.bp * sizeof(T);
  const int per_sm = smem <= 100 * 1024 ? 2 : 1;
  int64_t grid = (int64_t)kSMs * per_sm;
  if (grid > g.ptiles) grid = g.ptiles;
  g.grid = (int)(grid < 1 ? 1 : grid);
  return g;
}

template <typename T>
static size_t score_smem(const ScoreGeom& g) {
  return (size_t)g.P * g.ld * sizeof(T) + (size_t)g.kc * g.bp * sizeof(T) +
         (size_t)g.nt * g.P * sizeof(T) + 2 * (size_t)g.P * sizeof(int32_t) +
         2 * (size_t)g.bp * sizeof(float);
}

template <int KIND, typename T, int TP>
__global__ void __launch_bounds__(512, 1) score_kernel(CubeRef cube, const float* __restrict__ mu_hilo,
                             const double* __restrict__ mu64, const T* __restrict__ wt,
                             int ld_w, ScoreGeom geo, T* __restrict__ out_t,
                             uint32_t* __restrict__ max_bits) {
  using V = typename Vec16<T>::type;
  constexpr int VN = Vec16<T>::n;
  extern __shared__ __align__(16) unsigned char smem[];
  T* d = reinterpret_cast<T*>(smem);
  T* w = d + (size_t)geo.P * geo.ld;                 // W^T chunk [kc][bp]
  T* part = w + (size_t)geo.kc * geo.bp;             // [nt][P]
  int32_t* s_line = reinterpret_cast<int32_t*>(part + (size_t)geo.nt * geo.P);
  int32_t* s_samp = s_line + geo.P;
  float* mhi = reinterpret_cast<float*>(s_samp + geo.P);
  float* mlo = mhi + geo.bp;

  const int B = cube.bands;
  const int tid = threadIdx.x;
  const int J = tid % geo.nt;
  const int pg = tid / geo.nt;
  const bool active = pg < geo.pgroups;
  const int kmax = min(geo.bp, 8 * J + 8);
  if (mu_hilo) {
    for (int b = tid; b < geo.bp; b += blockDim.x) {
      mhi[b] = b < B ? mu_hilo[b] : 0.0f;
      mlo[b] = b < B ? mu_hilo[B + b] : 0.0f;
    }
  }
  auto load_w = [&](int k0) {
    for (int e = tid; e < geo.kc * geo.bp; e += blockDim.x) {
      const int kk = e / geo.bp, j = e - kk * geo.bp;
      const int k = k0 + kk;
      w[e] = (k < geo.bp) ? wt[(size_t)k * ld_w + j] : T(0);
    }
  };
  if (geo.w_resident) load_w(0);
  uint32_t local_max = 0;

  for (int64_t t = blockIdx.x; t < geo.ptiles; t += gridDim.x) {
    const int64_t p0 = t * geo.P;
    __syncthreads();
    load_tile<KIND, T>(cube, p0, geo.P, geo.ld, geo.bp, mhi, mlo, mu64, d, s_line, s_samp);
    __syncthreads();
    T acc[TP][8];
#pragma unroll
    for (int i = 0; i < TP; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = T(0);
    for (int k0 = 0; k0 < geo.bp; k0 += geo.kc) {
      if (!geo.w_resident) {
        __syncthreads();
        load_w(k0);
        __syncthreads();
      }
      if (active) {
        const int kend = min(k0 + geo.kc, kmax);
        for (int k = k0; k < kend; k += VN) {
          T dv[TP][VN];
#pragma unroll
          for (int i = 0; i < TP; ++i)
            unpack(*reinterpret_cast<const V*>(d + (size_t)(pg * TP + i) * geo.ld + k), dv[i]);
          T wv[VN][8];
#pragma unroll
          for (int kk = 0; kk < VN; ++kk) {
            const T* wr = w + (size_t)(k - k0 + kk) * geo.bp + 8 * J;
#pragma unroll
            for (int q = 0; q < 8; q += VN) unpack(*reinterpret_cast<const V*>(wr + q), &wv[kk][q]);
          }
#pragma unroll
          for (int kk = 0; kk < VN; ++kk)
#pragma unroll
            for (int i = 0; i < TP; ++i)
#pragma unroll
              for (int j = 0; j < 8; ++j) acc[i][j] = fma(dv[i][kk], wv[kk][j], acc[i][j]);
        }
      }
    }
    if (active) {
#pragma unroll
      for (int i = 0; i < TP; ++i) {
        T ss = T(0);
#pragma unroll
        for (int j = 0; j < 8; ++j) ss = fma(acc[i][j], acc[i][j], ss);
        part[(size_t)J * geo.P + pg * TP + i] = ss;
      }
    }
    __syncthreads();
    for (int p = tid; p < geo.P; p += blockDim.x) {
      const int64_t pix = p0 + p;
      if (pix < cube.npix) {
        T delta = T(0);
        for (int jj = 0; jj < geo.nt; ++jj) delta += part[(size_t)jj * geo.P + p];
        out_t[pix] = delta;
        if constexpr (sizeof(T) == 4) local_max = max(local_max, f2ord(delta));
      }
    }
  }
  if constexpr (sizeof(T) == 4) {
    if (max_bits) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
        local_max = max(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
      if ((tid & 31) == 0 && local_max) atomicMax(max_bits, local_max);
    }
  }
}

// W64 = L^-1 for the kernel slot: one column per thread
__global__ void trinv_kernel(const double* __restrict__ L, int B, double* __restrict__ W) {
  for (int c = threadIdx.x; c < B; c += blockDim.x) {
    for (int i = 0; i < c; ++i) W[(size_t)i * B + c] = 0.0;
    for (int i = c; i < B; ++i) {
      double a = (i == c) ? 1.0 : 0.0;
      for (int k = c; k < i; ++k) a -= L[(size_t)i * B + k] * W[(size_t)k * B + c];
      W[(size_t)i * B + c] = a / L[(size_t)i * B + i];
    }
  }
}

// transposed + padded copy W^T (ld x ld) for the score kernel
__global__ void transpose_pad_kernel(const double* __restrict__ W, int B, int ld,
                                     double* __restrict__ wt) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ld * ld; e += gridDim.x * blockDim.x) {
    const int k = e / ld, j = e - k * ld;
    wt[e] = (j < B && k < B && k <= j) ? W[(size_t)j * B + k] : 0.0;
  }
}

template <int KIND, typename T, int TP>
static int launch_score(const CubeRef& c, const float* mu_hilo, const double* mu64, const T* wt,
                        int ld_w, T* out, uint32_t* max_bits, cudaStream_t st) {
  ScoreGeom g = score_geom<T, TP>(c.npix, c.bands);
  if (c.npix == 0) return SKYRX_OK;
  const size_t sm = score_smem<T>(g);
  auto kern = score_kernel<KIND, T, TP>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  kern<<<g.grid, g.threads, sm, st>>>(c, mu_hilo, mu64, wt, ld_w, g, out, max_bits);
  SKYRX_CHECK_LAUNCH("score_kernel");
  return SKYRX_OK;
}

}  // namespace skyrx

using namespace skyrx;

extern "C" int skyrx_score(int32_t kind, const void* pixels, int64_t lines, int32_t samples,
                           int32_t bands, const float* dark, const float* coeff,
                           const float* gain, const float* mu_hilo, const float* whiten,
                           int32_t ld_w, float* scores, uint32_t* max_bits, void* stream) {
  SKYRX_REQUIRE(bands > 0 && bands <= 1024, "bands %d outside [1, 1024]", bands);
  SKYRX_REQUIRE(ld_w >= ((bands + 7) / 8) * 8, "ld_w %d too small", ld_w);
  CubeRef c;
  c.pixels = pixels;
  c.dark = dark;
  c.coeff = coeff;
  c.gain = gain;
  c.npix = lines * (int64_t)samples;
  c.samples = samples;
  c.bands = bands;
  cudaStream_t st = as_stream(stream);
  if (kind == SKYRX_IN_RAW_U16)
    return launch_score<SKYRX_IN_RAW_U16, float, 8>(c, mu_hilo, nullptr, whiten, ld_w, scores,
                                                    max_bits, st);
  if (kind == SKYRX_IN_F32)
    return launch_score<SKYRX_IN_F32, float, 8>(c, mu_hilo, nullptr, whiten, ld_w, scores,
                                                max_bits, st);
  set_error("bad pixel kind %d", kind);
  return SKYRX_ERR_ARG;
}

extern "C" int skyrx_mahalanobis_sq(int32_t kind, const void* pixels, int64_t n, int32_t bands,
                                    const double* mu, const double* chol, double* whiten64,
                                    double* out, void* stream) {
  SKYRX_REQUIRE(bands > 0 && bands <= 1024, "bands %d outside [1, 1024]", bands);
  SKYRX_REQUIRE(kind == SKYRX_IN_F32 || kind == SKYRX_IN_F64, "bad pixel kind %d", kind);
  cudaStream_t st = as_stream(stream);
  if (n == 0) return SKYRX_OK;
  const int bp = ((bands + 7) / 8) * 8;
  // whiten64 workspace holds W (B*B) followed by W^T padded (bp*bp)
  double* W = whiten64;
  double* wt = whiten64 + (size_t)bands * bands;
  trinv_kernel<<<1, 256, 0, st>>>(chol, bands, W);
  transpose_pad_kernel<<<ceil_div(bp * bp, 256), 256, 0, st>>>(W, bands, bp, wt);
  SKYRX_CHECK_LAUNCH("skyrx_mahalanobis_sq/trinv");
  CubeRef c;
  c.pixels = pixels;
  c.dark = c.coeff = c.gain = nullptr;
  c.npix = n;
  c.samples = 1;
  c.bands = bands;
  if (kind == SKYRX_IN_F64)
    return launch_score<SKYRX_IN_F64, double, 4>(c, nullptr, mu, wt, bp, out, nullptr, st);
  return launch_score<SKYRX_IN_F32, double, 4>(c, nullptr, mu, wt, bp, out, nullptr, st);
}
