// K2 background moments and K3 batched factorisation.
//
// Reference: rx.py:42-86 (compute_stats).  The reference makes two passes
// (f64 mean, then f64 dgemm of centred pixels).  Here one pass accumulates
// shifted moments s = sum(x-c), Q = sum((x-c)(x-c)^T) around a per-band shift
// c close to the mean (skyrx_stats_shift), so the raw cube is read once:
//   mu = c + s/n,  sigma = (Q - s s^T / n) / (n - 1)      (identical algebra).
//
// Precision plan (measured in numpy emulation on the c1 generator, kappa ~6e3,
// DESIGN.md §numerics): FP32 products and FP32 running sums of at most ~200
// products per accumulator, promoted to FP64 registers, FP64 across threads
// and CTAs in a fixed order (no float atomics -> bit-reproducible).
//
// Gram layout: B padded to BP = 8*nt; the lower triangle of nt x nt 8x8
// tiles is distributed over threads (tile, pixel-group); each thread keeps an
// 8x8 FP32 + 8x8 FP64 register accumulator and reads its two 8-band slices of
// every pixel of its group from the shared-memory tile (4 LDS.128 / 64 FFMA).
#include <cstdlib>

#include "common.cuh"
#include "tile_loader.cuh"

namespace skyrx {

constexpr int kGramThreads = 256;
constexpr int kGramTileP = 64;       // pixels per shared-memory tile
constexpr int kFlushProducts = 16;  // FP32 products per accumulator before FP64 promotion

struct GramGeom {
  int bp, nt, ntiles, parts, groups, tiles_per_part, ld, grid;
  int64_t ptiles;
};

static GramGeom gram_geom(int64_t npix, int bands, size_t tsize = 4) {
  GramGeom g;
  g.bp = ((bands + 7) / 8) * 8;
  g.nt = g.bp / 8;
  g.ntiles = g.nt * (g.nt + 1) / 2;
  if (g.ntiles <= kGramThreads) {
    g.parts = 1;
    g.groups = kGramThreads / g.ntiles;
    g.tiles_per_part = g.ntiles;
  } else {
    g.parts = ceil_div(g.ntiles, kGramThreads);
    g.groups = 1;
    g.tiles_per_part = kGramThreads;
  }
  g.ld = g.bp + (int)(16 / tsize);
  g.ptiles = ceil_div<int64_t>(npix, kGramTileP);
  int64_t grid = g.ptiles < kSMs ? g.ptiles : kSMs;
  g.grid = (int)(grid < 1 ? 1 : grid);
  return g;
}

static size_t gram_smem(const GramGeom& g, size_t tsize) {
  return (size_t)kGramTileP * g.ld * tsize + (size_t)g.bp * sizeof(double) +
         (size_t)(g.groups > 1 ? g.tiles_per_part * 64 : 0) * sizeof(double) +
         (size_t)g.bp * sizeof(float) + 2 * kGramTileP * sizeof(int32_t);
}

// workspace: per-CTA partials [grid][ntiles*64] + [grid][bp] doubles
static size_t gram_ws(const GramGeom& g) {
  return ((size_t)g.grid * g.ntiles * 64 + (size_t)g.grid * g.bp) * sizeof(double);
}

__device__ __forceinline__ void tri_decode(int t, int& I, int& J) {
  int i = (int)((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  while (i * (i + 1) / 2 > t) --i;
  I = i;
  J = t - i * (i + 1) / 2;
}

template <int KIND, typename T>
__global__ void __launch_bounds__(kGramThreads, 1) gram_kernel(
    CubeRef cube, const double* __restrict__ shift, GramGeom geo, double* __restrict__ part_q,
    double* __restrict__ part_s, int32_t* __restrict__ flags) {
  constexpr bool kFast = sizeof(T) == 4;  // f32 products, FP64 promotion; else all-f64
  extern __shared__ __align__(16) unsigned char smem[];
  T* d = reinterpret_cast<T*>(smem);
  double* c64 = reinterpret_cast<double*>(d + kGramTileP * geo.ld);
  double* red = c64 + geo.bp;
  float* c_f = reinterpret_cast<float*>(red + (geo.groups > 1 ? geo.tiles_per_part * 64 : 0));
  int32_t* s_line = reinterpret_cast<int32_t*>(c_f + geo.bp);
  int32_t* s_samp = s_line + kGramTileP;

  const int B = cube.bands;
  const int tid = threadIdx.x;
  for (int b = tid; b < geo.bp; b += kGramThreads) {
    const double c = b < B ? shift[b] : 0.0;
    c64[b] = c;
    c_f[b] = (float)c;  // shift is f32-representable (skyrx_stats_shift)
  }

  const int part = blockIdx.y;
  const int tiles_here = min(geo.tiles_per_part, geo.ntiles - part * geo.tiles_per_part);
  const int group = tid / tiles_here;
  const int tl = tid - group * tiles_here;
  const bool active = group < geo.groups;
  int I = 0, J = 0;
  if (active) tri_decode(part * geo.tiles_per_part + tl, I, J);
  // band sums: thread b owns bands b and b + 256 (bp <= 512 covers B <= 512)
  const bool do_s = (part == 0) && tid < geo.bp;
  const bool do_s2 = (part == 0) && tid + kGramThreads < geo.bp;

  T acc[8][8];
  double acc64[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = T(0), acc64[i][j] = 0.0;
  double s64 = 0.0, s64b = 0.0;
  int since_flush = 0;
  bool finite_ok = true;
  bool clamped = false;
  const int per_thread = ceil_div(kGramTileP, geo.groups);

  for (int64_t t = blockIdx.x; t < geo.ptiles; t += gridDim.x) {
    __syncthreads();
    finite_ok &= load_tile<KIND, T>(cube, t * kGramTileP, kGramTileP, geo.ld, geo.bp, c_f,
                                    nullptr, c64, d, s_line, s_samp, &clamped);
    __syncthreads();
    if (do_s) {  // band sums over the tile, then FP64 across tiles
      T cs = T(0);
      for (int p = 0; p < kGramTileP; ++p) cs += d[p * geo.ld + tid];
      s64 += (double)cs;
      if (do_s2) {
        T cs2 = T(0);
        for (int p = 0; p < kGramTileP; ++p) cs2 += d[p * geo.ld + tid + kGramThreads];
        s64b += (double)cs2;
      }
    }
    if (active) {
      const T* rowI = d + 8 * I;
      const T* rowJ = d + 8 * J;
      for (int p = group; p < kGramTileP; p += geo.groups) {
        T av[8], bv[8];
        load8(rowI + p * geo.ld, av);
        load8(rowJ + p * geo.ld, bv);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
        if (kFast && ++since_flush == kFlushProducts) {  // promote short f32 runs to f64
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc64[i][j] += (double)acc[i][j], acc[i][j] = T(0);
          since_flush = 0;
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc64[i][j] += (double)acc[i][j];

  // combine pixel groups in a fixed order, then one partial per CTA
  double* pq = part_q + (size_t)blockIdx.x * geo.ntiles * 64 +
               (size_t)(part * geo.tiles_per_part) * 64;
  if (geo.groups > 1) {
    __syncthreads();
    for (int g = 0; g < geo.groups; ++g) {
      if (active && group == g) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            double* r = red + tl * 64 + i * 8 + j;
            *r = (g == 0) ? acc64[i][j] : *r + acc64[i][j];
          }
      }
      __syncthreads();
    }
    for (int e = tid; e < tiles_here * 64; e += kGramThreads) pq[e] = red[e];
  } else if (active) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) pq[tl * 64 + i * 8 + j] = acc64[i][j];
  }
  if (do_s) part_s[(size_t)blockIdx.x * geo.bp + tid] = s64;
  if (do_s2) part_s[(size_t)blockIdx.x * geo.bp + tid + kGramThreads] = s64b;
  if (!finite_ok) atomicOr(flags, 1);
  // 128: the general path's clamp check ran; 64: a raw value was below dark
  if (KIND == SKYRX_IN_RAW_U16) {
    if (blockIdx.x == 0 && tid == 0) atomicOr(flags, 128);
    if (__any_sync(0xffffffffu, clamped) && (tid & 31) == 0) atomicOr(flags, 64);
  }
}

// moments[0] = n, moments[1..B] = s, moments[1+B ..] = Q (full, symmetric)
__global__ void gram_reduce_kernel(const double* __restrict__ part_q,
                                   const double* __restrict__ part_s, GramGeom geo, int bands,
                                   double n, double* __restrict__ moments) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const int nq = geo.ntiles * 64;
  double* s_out = moments + 1;
  double* q_out = moments + 1 + bands;
  if (e < nq) {
    double v = 0.0;
    for (int c = 0; c < geo.grid; ++c) v += part_q[(size_t)c * nq + e];
    const int t = e >> 6, r = (e >> 3) & 7, cc = e & 7;
    int I, J;
    tri_decode(t, I, J);
    const int row = 8 * I + r, col = 8 * J + cc;
    if (row < bands && col < bands && (I != J || r >= cc)) {
      q_out[(size_t)row * bands + col] = v;
      q_out[(size_t)col * bands + row] = v;
    }
  } else if (e < nq + bands) {
    const int b = e - nq;
    double v = 0.0;
    for (int c = 0; c < geo.grid; ++c) v += part_s[(size_t)c * geo.bp + b];
    s_out[b] = v;
  } else if (e == nq + bands) {
    moments[0] = n;
  }
}

// shift: f32-rounded f64 mean of a strided sample of <= 4096 pixels
// one CTA per band, 256 threads over the sample, fixed-order tree reduction
template <int KIND>
__global__ void __launch_bounds__(256) shift_kernel(CubeRef cube, double* __restrict__ shift) {
  __shared__ double part[8];
  const int64_t n = cube.npix;
  const int64_t step = n > 4096 ? n / 4096 : 1;
  const int64_t m = n > 0 ? (n + step - 1) / step : 0;
  const int B = cube.bands;
  const int b = blockIdx.x;
  auto value = [&](int64_t i) -> float {
    const int64_t pix = i * step;
    const int64_t gi = pix * B + b;
    if constexpr (KIND == SKYRX_IN_RAW_U16) {
      const int64_t line = pix / cube.samples;
      const int64_t tb = (pix - line * cube.samples) * B + b;
      return calib((float)__ldg(reinterpret_cast<const uint16_t*>(cube.pixels) + gi),
                   __ldg(cube.dark + tb), __ldg(cube.coeff + tb), __ldg(cube.gain + line));
    } else {
      return __ldg(reinterpret_cast<const float*>(cube.pixels) + gi);
    }
  };
  // the strided sample is scattered over the whole cube: issue 8 loads before
  // summing (same order as a plain loop, so the shift is unchanged)
  double acc = 0.0;
  int64_t i = threadIdx.x;
  for (; i + 7 * (int64_t)blockDim.x < m; i += 8 * (int64_t)blockDim.x) {
    float x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = value(i + q * (int64_t)blockDim.x);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc += (double)x[q];
  }
  for (; i < m; i += blockDim.x) acc += (double)value(i);
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += part[w];
    shift[b] = m > 0 ? (double)(float)(s / (double)m) : 0.0;
  }
}

__global__ void fold_kernel(double* __restrict__ state, const double* __restrict__ chunk,
                            int64_t len, double forget, double* __restrict__ prev) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < len) {
    const double v = state[i];
    if (prev) prev[i] = v;  // the undo point of a chunk that must be redone
    state[i] = forget * v + chunk[i];
  }
}

// ------------------------------------------------------------------ K3
constexpr int kFinThreads = 512;
// -DSKYRX_FIN_PROFILE: clock64 at the phase boundaries of matrix 0 (skyrx_fin_profile)
#ifdef SKYRX_FIN_PROFILE
__device__ long long fin_prof[8];
__device__ long long fin_acc[4];
#define FIN_T(k)                                                    \
  do {                                                              \
    __syncthreads();                                                \
    if (blockIdx.x == 0 && threadIdx.x == 0) fin_prof[k] = clock64(); \
  } while (0)
extern "C" __attribute__((visibility("default"))) int skyrx_fin_profile(long long* out) {
  cudaMemcpyFromSymbol(out + 8, fin_acc, sizeof(fin_acc));
  return (int)cudaMemcpyFromSymbol(out, fin_prof, sizeof(fin_prof));
}
#else
#define FIN_T(k) \
  do {           \
  } while (0)
#endif
constexpr int kSmemCholMaxB = 160;
constexpr int kSmemInvMaxB = 118;  // L and W = L^-1 both in shared memory (2 B^2 doubles)

__device__ __forceinline__ double block_sum_fixed(double v, double* scratch) {
  // deterministic: warp tree then serial over warps
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) scratch[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r += scratch[i];
    scratch[32] = r;
  }
  __syncthreads();
  r = scratch[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kFinThreads) finalize_kernel(
    const double* __restrict__ moments_all, const double* __restrict__ shift_all,
    const int32_t* __restrict__ flags_all, int bands, double* __restrict__ mu_all,
    double* __restrict__ sigma_all, double* __restrict__ chol_all,
    double* __restrict__ inv_all, double* __restrict__ w64_all, float* __restrict__ wf_all,
    int ld_w, float* __restrict__ mhl_all, double* __restrict__ ridge_all,
    int32_t* __restrict__ status_all, int do_inverse) {
  extern __shared__ __align__(16) double fsm[];
  __shared__ double scratch[40];
  __shared__ int s_fail;
  const int B = bands;
  const size_t BB = (size_t)B * B;
  const int m = blockIdx.x;
  const double* mom = moments_all + (size_t)m * (1 + B + BB);
  const double* shift = shift_all + (size_t)m * B;
  double* mu = mu_all + (size_t)m * B;
  double* sigma = sigma_all + (size_t)m * BB;
  double* chol = chol_all + (size_t)m * BB;
  double* inv = inv_all + (size_t)m * BB;
  double* w64 = w64_all + (size_t)m * BB;
  float* wf = wf_all + (size_t)m * ld_w * ld_w;
  float* mhl = mhl_all + (size_t)m * 2 * B;
  const int tid = threadIdx.x;
  const int NT = blockDim.x;
  FIN_T(0);

  const double n = mom[0];
  const double* s = mom + 1;
  const double* q = mom + 1 + B;
  int status = SKYRX_OK;
  // 2: int8 quantiser overflow, 4: a value clamped at 0 on the raw-byte path
  if (flags_all && flags_range(flags_all[m])) status = SKYRX_ERR_RANGE;
  if (flags_all && (flags_all[m] & 1)) status = SKYRX_ERR_NONFINITE;
  if (!(n > (double)B)) status = SKYRX_ERR_INSUFFICIENT;  // rx.py:51 checks size first
  if (status != SKYRX_OK) {
    if (tid == 0) {
      status_all[m] = status;
      ridge_all[m] = 0.0;
    }
    return;
  }
  // mu, sigma (rx.py:59, 65-66)
  for (int b = tid; b < B; b += NT) {
    const double mb = shift[b] + s[b] / n;
    mu[b] = mb;
    const float hi = (float)mb;
    mhl[b] = hi;
    mhl[B + b] = (float)(mb - (double)hi);
  }
  // (row, column) loops: a warp per row, lanes along it (no 64-bit index divisions)
  const int nwarp = NT >> 5, wrp = tid >> 5, lan = tid & 31;
  for (int i = wrp; i < B; i += nwarp)
    for (int j = lan; j < B; j += 32) {
    const size_t e = (size_t)i * B + j;
    const double vij = (q[(size_t)i * B + j] - s[i] * s[j] / n) / (n - 1.0);
    const double vji = (q[(size_t)j * B + i] - s[j] * s[i] / n) / (n - 1.0);
    sigma[e] = (vij + vji) / 2.0;
  }
  __syncthreads();
  __threadfence_block();
  double tr = 0.0;
  for (int b = tid; b < B; b += NT) tr += sigma[(size_t)b * B + b];
  const double trace = block_sum_fixed(tr, scratch);
  const double scale = trace > 0.0 ? trace / B : 1.0;

  // dynamic shared memory: [l_jj | 1 / l_jj] (2B), then A (B <= kSmemCholMaxB), then W
  double* dg = fsm;
  FIN_T(1);
  double* A = (B <= kSmemCholMaxB) ? fsm + 2 * B : chol;  // working factor
  // row stride of A: odd in shared memory, so a column walk (lanes over rows) spreads over
  // the banks instead of hitting every 4th one (B = 70: stride 140 words)
  const int la = (A != chol) ? (B | 1) : B;
  const double eps_tab[6] = {0.0, 1e-10, 1e-9, 1e-8, 1e-7, 1e-6};
  double ridge = 0.0;
  bool ok = false;
  for (int a = 0; a < 6 && !ok; ++a) {
    ridge = eps_tab[a] * scale;
    for (int i = wrp; i < B; i += nwarp)
      for (int j = lan; j < B; j += 32)
        A[(size_t)i * la + j] = (j <= i) ? sigma[(size_t)i * B + j] + (i == j ? ridge : 0.0) : 0.0;
    if (tid == 0) s_fail = 0;
    if (A == chol) {  // ---- wide B: the factor lives in global memory (L2): blocked
      // Panels of NBP columns in shared memory (column-major P[jj * B + row]); the panel is
      // factored there and the trailing matrix gets the panel's NBP updates per element in
      // one read-modify-write, applied in the same order, with the same rounded l values
      // and FMA-free operations as the unblocked loop below: bit-identical factors, a
      // fraction of the L2 traffic of one column at a time.
      double* P = fsm + 2 * B;
      const int NBP = B <= 750 ? 32 : 16;
      __syncthreads();
      for (int p0 = 0; p0 < B && !s_fail; p0 += NBP) {
        const int nb = min(NBP, B - p0), rows = B - p0;
        for (int e = tid; e < nb * rows; e += NT) {
          const int jj = e / rows, r = p0 + (e - jj * rows);
          P[jj * B + r] = (r >= p0 + jj) ? A[(size_t)r * B + p0 + jj] : 0.0;
        }
        __syncthreads();
#ifdef SKYRX_FIN_PROFILE
        const long long pt0 = clock64();
#endif
        // the panel: a thread per row r, one barrier per column; the owner of row j+1 takes
        // the next pivot right after its update (lookahead), column jj is scaled one step
        // later (when nobody reads it any more)
        auto piv = [&](int j, double v) {
          if (!(v > 0.0)) {
            s_fail = 1;
            return;
          }
          const double l = sqrt(v);
          dg[j] = l, dg[B + j] = 1.0 / l;
        };
        if (tid == 0) piv(p0, P[p0]);
        __syncthreads();
        const int nw = NT >> 5, wid = tid >> 5, ln = tid & 31;
        for (int jj = 0; jj < nb; ++jj) {
          if (s_fail) break;  // uniform: set before the previous barrier
          const int j = p0 + jj;
          const double rl = dg[B + j];
          if (jj > 0)  // delayed scaling of column jj-1 (rows >= j)
            for (int r = j + tid; r < B; r += NT) P[(jj - 1) * B + r] *= dg[B + j - 1];
          // a warp per panel column jj2 > jj, lanes along the rows r >= p0 + jj2; each lane
          // loads up to 8 of its rows before it stores any
          for (int jj2 = jj + 1 + wid; jj2 < nb; jj2 += nw) {
            const double lkj = P[jj * B + p0 + jj2] * rl;
            double* Pc = P + jj2 * B;
            const double* Pj = P + jj * B;
            for (int r0 = p0 + jj2 + ln; r0 < B; r0 += 256) {
              double x[8], y[8];
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const int r = r0 + 32 * q;
                if (r < B) x[q] = Pc[r], y[q] = Pj[r];
              }
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const int r = r0 + 32 * q;
                if (r < B) {
                  const double v = __dsub_rn(x[q], __dmul_rn(y[q] * rl, lkj));
                  Pc[r] = v;
                  if (jj2 == jj + 1 && r == j + 1) piv(r, v);  // the next pivot
                }
              }
            }
          }
          __syncthreads();
        }
        if (!s_fail) {
          for (int r = p0 + nb - 1 + tid; r < B; r += NT)  // the last column's scaling
            if (r > p0 + nb - 1) P[(nb - 1) * B + r] *= dg[B + p0 + nb - 1];
          for (int jj = tid; jj < nb; jj += NT) P[jj * B + p0 + jj] = dg[p0 + jj];
        }
        __syncthreads();
        if (s_fail) break;
        for (int e = tid; e < nb * rows; e += NT) {  // the finished panel of L
          const int jj = e / rows, r = p0 + (e - jj * rows);
          if (r >= p0 + jj) A[(size_t)r * B + p0 + jj] = P[jj * B + r];
        }
#ifdef SKYRX_FIN_PROFILE
        __syncthreads();
        const long long pt1 = clock64();
        if (tid == 0 && blockIdx.x == 0) fin_acc[0] += pt1 - pt0;
#endif
        // trailing update: a warp per row i, lanes along k <= i, the nb updates in order
        const int q0 = p0 + nb;
        for (int i = q0 + wid; i < B; i += nw)
          for (int k0 = q0 + ln; k0 <= i; k0 += 128) {  // 4 independent chains per lane
            double v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int k = k0 + 32 * q;
              v[q] = k <= i ? A[(size_t)i * B + k] : 0.0;
            }
            for (int jj = 0; jj < nb; ++jj) {
              const double lij = P[jj * B + i];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const int k = min(k0 + 32 * q, i);
                v[q] = __dsub_rn(v[q], __dmul_rn(lij, P[jj * B + k]));
              }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int k = k0 + 32 * q;
              if (k <= i) A[(size_t)i * B + k] = v[q];
            }
          }
        __syncthreads();
#ifdef SKYRX_FIN_PROFILE
        if (tid == 0 && blockIdx.x == 0) fin_acc[1] += clock64() - pt1;
#endif
      }
      __syncthreads();
      ok = (s_fail == 0);
      __syncthreads();
      continue;
    }
    // right-looking Cholesky, lower triangle, ONE barrier per column: the trailing update
    // uses l_ij = a_ij / l_jj on the fly (FMA-free, so an exactly rank-deficient input
    // still meets an exactly zero pivot and fails like LAPACK potrf), and column j is
    // scaled in place one step later, when nobody reads it any more. The pivot j+1 is
    // final as soon as step j has updated it: the thread that does so takes its root and
    // reciprocal right away (lookahead), the other warps read them after the barrier.
    const int nw = NT >> 5, wid = tid >> 5, ln = tid & 31;
    auto pivot = [&](int jj, double v) {
      if (!(v > 0.0)) {  // LAPACK potrf: non-positive or NaN pivot fails
        s_fail = 1;
        return;
      }
      const double l = sqrt(v);
      dg[jj] = l, dg[B + jj] = 1.0 / l;
    };
    __syncthreads();
    if (tid == 0) pivot(0, A[0]);
    __syncthreads();
    for (int j = 0; j < B; ++j) {
      if (s_fail) break;  // uniform: written before the previous barrier
      const double rl = dg[B + j];
      const int r = B - j - 1;  // trailing order
      // warp 0: rows j and j+1 (the lookahead pivot, a serial root + reciprocal), the
      // other warps: the trailing rows j+2.. (a warp per row)
      for (int ii = wid == 0 ? 0 : wid + 1; ii <= r; ii += wid == 0 ? 1 : nw - 1) {
        if (wid == 0 && ii > 1) break;
        const int i = j + ii;
        double* Ai = A + i * la;
        if (j > 0 && ln == 0) Ai[j - 1] *= dg[B + j - 1];
        if (ii == 0) continue;
        const double lij = Ai[j] * rl;
        if (ii == 1) {  // row j+1 has one entry: the next pivot
          if (ln == 0) {
            const double v = __dsub_rn(Ai[j + 1], __dmul_rn(lij, lij));
            Ai[j + 1] = v;
            pivot(i, v);
          }
          continue;
        }
        // up to 4 of the lane's entries: all loads, then the updates (the stores would
        // otherwise order every next load behind them)
        for (int k0 = j + 1; k0 <= i; k0 += 128) {
          double x[4], z[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int k = k0 + ln + 32 * q;
            if (k <= i) x[q] = Ai[k], z[q] = A[k * la + j];
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int k = k0 + ln + 32 * q;
            if (k <= i) Ai[k] = __dsub_rn(x[q], __dmul_rn(lij, z[q] * rl));
          }
        }
      }
      __syncthreads();
    }
    __syncthreads();
    ok = (s_fail == 0);
    if (ok)
      for (int j = tid; j < B; j += NT) A[j * la + j] = dg[j];
    __syncthreads();
  }
  if (!ok) {
    if (tid == 0) {
      status_all[m] = SKYRX_ERR_NOT_PD;
      ridge_all[m] = ridge;
    }
    return;
  }
  FIN_T(2);
  if (A != chol)
    for (int i = wrp; i < B; i += nwarp)
      for (int j = lan; j < B; j += 32) chol[(size_t)i * B + j] = A[(size_t)i * la + j];
  __syncthreads();
  if (!do_inverse) {  // wide matrices: W, Sigma^-1 and wf by the multi-CTA kernels below
    if (tid == 0) {
      status_all[m] = SKYRX_OK;
      ridge_all[m] = ridge;
    }
    return;
  }
  // W = L^-1 in shared memory next to L when both fit (so the O(B^3) loops never touch
  // global memory), right-looking: after step j row j of W is final (R_j * 1/l_jj, scaled
  // in place one step later) and every later row has subtracted l_ij * W_j; one barrier per
  // row, the (i, c) updates of a step spread over the whole CTA
  double* Wm = (A != chol && B <= kSmemInvMaxB) ? A + (size_t)B * la : w64;
  for (int i = wrp; i < B; i += nwarp)
    for (int c = lan; c < B; c += 32) Wm[i * B + c] = (i == c) ? 1.0 : 0.0;
  __syncthreads();
  {
    const int nw = NT >> 5, wid = tid >> 5, ln = tid & 31;
    for (int j = 0; j < B; ++j) {
      const double rj = dg[B + j];
      if (j > 0 && wid == nw - 1)
        for (int c = ln; c < j; c += 32) Wm[(j - 1) * B + c] *= dg[B + j - 1];
      const double* Wj = Wm + j * B;
      for (int i = j + 1 + wid; i < B; i += nw) {  // a warp per row, lanes along c <= j
        const double lij = A[i * la + j];
        double* Wi = Wm + i * B;
        for (int c0 = 0; c0 <= j; c0 += 128) {
          double x[4], z[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int c = c0 + ln + 32 * q;
            if (c <= j) x[q] = Wi[c], z[q] = Wj[c];
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int c = c0 + ln + 32 * q;
            if (c <= j) Wi[c] = __dsub_rn(x[q], __dmul_rn(lij, z[q] * rj));  // FMA-free
          }
        }
      }
      __syncthreads();
    }
  }
  for (int c = tid; c < B; c += NT) Wm[(size_t)(B - 1) * B + c] *= dg[B + B - 1];
  __syncthreads();
  FIN_T(3);
  if (Wm != w64)
    for (size_t e = tid; e < BB; e += NT) w64[e] = Wm[e];
  __threadfence_block();
  FIN_T(4);
  // sigma_inv = W^T W (= cho_solve(L, I)), exactly symmetric by construction
  {  // a warp per row i (rows dealt so the long dot products spread), lanes along j <= i
    const int nw = NT >> 5, wid = tid >> 5, ln = tid & 31;
    for (int i = wid; i < B; i += nw)
      for (int j = ln; j <= i; j += 32) {
        double a0 = 0.0, a1 = 0.0;
        int k = i;
        for (; k + 1 < B; k += 2) {
          a0 += Wm[k * B + i] * Wm[k * B + j];
          a1 += Wm[(k + 1) * B + i] * Wm[(k + 1) * B + j];
        }
        if (k < B) a0 += Wm[k * B + i] * Wm[k * B + j];
        const double acc = a0 + a1;
        inv[(size_t)i * B + j] = acc;
        inv[(size_t)j * B + i] = acc;
      }
  }
  FIN_T(5);
  // f32 whitening matrix, transposed (wf[k * ld_w + j] = W[j][k]) for K4
  for (size_t e = tid; e < (size_t)ld_w * ld_w; e += NT) {
    const int k = (int)(e / ld_w), j = (int)(e - (size_t)k * ld_w);
    wf[e] = (j < B && k < B && k <= j) ? (float)Wm[(size_t)j * B + k] : 0.0f;
  }
  FIN_T(6);
  if (tid == 0) {
    status_all[m] = SKYRX_OK;
    ridge_all[m] = ridge;
  }
}

// Wide matrices (B > kSmemInvMaxB): W = L^-1 with one WARP per column (lanes split the
// forward-substitution dot products, the column's solution in shared memory), the
// columns spread over CTAs; then Sigma^-1 = W^T W and the f32 copy, one thread per entry.
__global__ void __launch_bounds__(1024) wide_trinv_kernel(const double* __restrict__ chol_all,
                                                          int B, double* __restrict__ w64_all,
                                                          const int32_t* __restrict__ status_all) {
  extern __shared__ double xs[];  // [32 warps][B]
  const int m = blockIdx.y;
  if (status_all[m] != SKYRX_OK) return;
  const double* L = chol_all + (size_t)m * B * B;
  double* W = w64_all + (size_t)m * B * B;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * 32 + w;
  if (c >= B) return;
  double* x = xs + (size_t)w * B;
  for (int i = lane; i < c; i += 32) W[(size_t)i * B + c] = 0.0;
  for (int i = c; i < B; ++i) {
    double a = 0.0;
    for (int k = c + lane; k < i; k += 32) a += L[(size_t)i * B + k] * x[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    const double xi = ((i == c ? 1.0 : 0.0) - a) / L[(size_t)i * B + i];
    if (lane == 0) {
      x[i] = xi;
      W[(size_t)i * B + c] = xi;
    }
    __syncwarp();
  }
}

__global__ void wide_inv_kernel(const double* __restrict__ w64_all, int B,
                                double* __restrict__ inv_all, float* __restrict__ wf_all, int ld_w,
                                const int32_t* __restrict__ status_all) {
  const int m = blockIdx.y;
  if (status_all[m] != SKYRX_OK) return;
  const double* W = w64_all + (size_t)m * B * B;
  double* inv = inv_all + (size_t)m * B * B;
  float* wf = wf_all + (size_t)m * ld_w * ld_w;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e < (int64_t)B * B) {
    const int i = (int)(e / B), j = (int)(e - (int64_t)i * B);
    if (j <= i) {  // sigma_inv = W^T W, exactly symmetric by construction
      double acc = 0.0;
      for (int k = i; k < B; ++k) acc += W[(size_t)k * B + i] * W[(size_t)k * B + j];
      inv[(size_t)i * B + j] = acc;
      inv[(size_t)j * B + i] = acc;
    }
  }
  if (e < (int64_t)ld_w * ld_w) {  // f32 whitening matrix, transposed (wf[k, j] = W[j][k])
    const int k = (int)(e / ld_w), j = (int)(e - (int64_t)k * ld_w);
    wf[e] = (j < B && k < B && k <= j) ? (float)W[(size_t)j * B + k] : 0.0f;
  }
}

// W = L^-1 (f64, one column per thread), its f32 transposed padded copy and
// mu hi/lo, for scoring with caller-supplied stats (rx_scores(cube, stats)).
__global__ void whiten_prepare_kernel(const double* __restrict__ L, const double* __restrict__ mu,
                                      int B, double* __restrict__ W, float* __restrict__ wf,
                                      int ld_w, float* __restrict__ mhl) {
  for (int c = threadIdx.x; c < B; c += blockDim.x) {
    for (int i = 0; i < c; ++i) W[(size_t)i * B + c] = 0.0;
    for (int i = c; i < B; ++i) {
      double a = (i == c) ? 1.0 : 0.0;
      for (int k = c; k < i; ++k) a -= L[(size_t)i * B + k] * W[(size_t)k * B + c];
      W[(size_t)i * B + c] = a / L[(size_t)i * B + i];
    }
    const float hi = (float)mu[c];
    mhl[c] = hi;
    mhl[B + c] = (float)(mu[c] - (double)hi);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < ld_w * ld_w; e += blockDim.x) {
    const int k = e / ld_w, j = e - k * ld_w;
    wf[e] = (j < B && k < B && k <= j) ? (float)W[(size_t)j * B + k] : 0.0f;
  }
}

// sigma_inv = W^T W and the f32 whitening copy for the wide paths
static int launch_wide_inv(const double* w64, int B, int batch, double* sigma_inv, float* wf,
                           int ld_w, const int32_t* status, cudaStream_t st) {
  const int64_t work = std::max((int64_t)B * B, (int64_t)ld_w * ld_w);
  wide_inv_kernel<<<dim3((int)ceil_div<int64_t>(work, 256), batch), 256, 0, st>>>(
      w64, B, sigma_inv, wf, ld_w, status);
  SKYRX_CHECK_LAUNCH("skyrx_stats_finalize/wide");
  return SKYRX_OK;
}

int launch_finalize_wide(const double* moments, const double* shift, const int32_t* flags, int B,
                         int batch, double* mu, double* sigma, double* chol, double* w64,
                         float* mhl, double* ridge, int32_t* status, cudaStream_t st);
int launch_finalize_panel(const double* moments, const double* shift, const int32_t* flags,
                          int B, int batch, double* mu, double* sigma, double* chol,
                          double* sigma_inv, double* w64, float* wf, int ld_w, float* mhl,
                          double* ridge, int32_t* status, cudaStream_t st);
int launch_finalize_small(const double* moments, const double* shift, const int32_t* flags,
                          int B, int batch, double* mu, double* sigma, double* chol,
                          double* sigma_inv, double* w64, float* wf, int ld_w, float* mhl,
                          double* ridge, int32_t* status, cudaStream_t st);

}  // namespace skyrx

using namespace skyrx;

extern "C" int skyrx_whiten_prepare(const double* chol, const double* mu, int32_t bands,
                                    double* whiten64, float* whiten, int32_t ld_w,
                                    float* mu_hilo, void* stream) {
  SKYRX_REQUIRE(bands > 0 && bands <= 1024 && ld_w >= bands, "bad whiten arguments");
  whiten_prepare_kernel<<<1, 512, 0, as_stream(stream)>>>(chol, mu, bands, whiten64, whiten,
                                                          ld_w, mu_hilo);
  SKYRX_CHECK_LAUNCH("skyrx_whiten_prepare");
  return SKYRX_OK;
}

extern "C" size_t skyrx_moments_len(int32_t bands) {
  return 1 + (size_t)bands + (size_t)bands * bands;
}

static CubeRef make_ref(const void* px, int64_t lines, int32_t samples, int32_t bands,
                        const float* dark, const float* coeff, const float* gain) {
  CubeRef c;
  c.pixels = px;
  c.dark = dark;
  c.coeff = coeff;
  c.gain = gain;
  c.npix = lines * (int64_t)samples;
  c.samples = samples;
  c.bands = bands;
  return c;
}

extern "C" int skyrx_stats_shift(int32_t kind, const void* pixels, int64_t lines,
                                 int32_t samples, int32_t bands, const float* dark,
                                 const float* coeff, const float* gain, double* shift,
                                 void* stream) {
  SKYRX_REQUIRE(bands > 0 && lines >= 0 && samples >= 0, "bad cube shape");
  SKYRX_REQUIRE(kind == SKYRX_IN_RAW_U16 || kind == SKYRX_IN_F32, "bad pixel kind %d", kind);
  CubeRef c = make_ref(pixels, lines, samples, bands, dark, coeff, gain);
  cudaStream_t st = as_stream(stream);
  if (kind == SKYRX_IN_RAW_U16)
    shift_kernel<SKYRX_IN_RAW_U16><<<bands, 256, 0, st>>>(c, shift);
  else
    shift_kernel<SKYRX_IN_F32><<<bands, 256, 0, st>>>(c, shift);
  SKYRX_CHECK_LAUNCH("skyrx_stats_shift");
  return SKYRX_OK;
}

extern "C" int skyrx_stats_workspace(int64_t lines, int32_t samples, int32_t bands,
                                     size_t* bytes) {
  SKYRX_REQUIRE(bands > 0 && bytes, "bad arguments");
  *bytes = gram_ws(gram_geom(lines * (int64_t)samples, bands));  // grid independent of T
  return SKYRX_OK;
}

template <int KIND, typename T>
static void launch_gram(const CubeRef& c, const double* shift, const GramGeom& g, double* pq,
                        double* ps, int32_t* flags, cudaStream_t st) {
  const size_t sm = gram_smem(g, sizeof(T));
  cudaFuncSetAttribute(gram_kernel<KIND, T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sm);
  gram_kernel<KIND, T><<<dim3(g.grid, g.parts), kGramThreads, sm, st>>>(c, shift, g, pq, ps,
                                                                        flags);
}

extern "C" int skyrx_stats_accumulate(int32_t kind, const void* pixels, int64_t lines,
                                      int32_t samples, int32_t bands, const float* dark,
                                      const float* coeff, const float* gain,
                                      const double* shift, int32_t precise, double* moments,
                                      int32_t* flags, void* workspace, size_t workspace_bytes,
                                      void* stream) {
  SKYRX_REQUIRE(bands > 0 && bands <= 320, "bands %d outside [1, 320]", bands);
  SKYRX_REQUIRE(kind == SKYRX_IN_RAW_U16 || kind == SKYRX_IN_F32, "bad pixel kind %d", kind);
  const int64_t npix = lines * (int64_t)samples;
  const size_t ts = precise ? sizeof(double) : sizeof(float);
  GramGeom g = gram_geom(npix, bands, ts);
  SKYRX_REQUIRE(workspace_bytes >= gram_ws(g), "stats workspace too small (%zu < %zu)",
                workspace_bytes, gram_ws(g));
  CubeRef c = make_ref(pixels, lines, samples, bands, dark, coeff, gain);
  double* part_q = reinterpret_cast<double*>(workspace);
  double* part_s = part_q + (size_t)g.grid * g.ntiles * 64;
  cudaStream_t st = as_stream(stream);
  if (kind == SKYRX_IN_RAW_U16) {
    if (precise) launch_gram<SKYRX_IN_RAW_U16, double>(c, shift, g, part_q, part_s, flags, st);
    else launch_gram<SKYRX_IN_RAW_U16, float>(c, shift, g, part_q, part_s, flags, st);
  } else {
    if (precise) launch_gram<SKYRX_IN_F32, double>(c, shift, g, part_q, part_s, flags, st);
    else launch_gram<SKYRX_IN_F32, float>(c, shift, g, part_q, part_s, flags, st);
  }
  SKYRX_CHECK_LAUNCH("skyrx_stats_accumulate/gram");
  const int work = g.ntiles * 64 + bands + 1;
  gram_reduce_kernel<<<ceil_div(work, 256), 256, 0, st>>>(part_q, part_s, g, bands,
                                                          (double)npix, moments);
  SKYRX_CHECK_LAUNCH("skyrx_stats_accumulate/reduce");
  return SKYRX_OK;
}

extern "C" int skyrx_moments_fold(double* state, const double* chunk, int32_t bands,
                                  double forget, void* stream) {
  SKYRX_REQUIRE(bands > 0, "bad bands");
  const int64_t len = (int64_t)skyrx_moments_len(bands);
  fold_kernel<<<(int)ceil_div<int64_t>(len, 256), 256, 0, as_stream(stream)>>>(state, chunk,
                                                                               len, forget, nullptr);
  SKYRX_CHECK_LAUNCH("skyrx_moments_fold");
  return SKYRX_OK;
}

extern "C" int skyrx_moments_fold_keep(double* state, const double* chunk, int32_t bands,
                                       double forget, double* prev, void* stream) {
  SKYRX_REQUIRE(bands > 0 && prev != nullptr, "bad bands or prev");
  const int64_t len = (int64_t)skyrx_moments_len(bands);
  fold_kernel<<<(int)ceil_div<int64_t>(len, 256), 256, 0, as_stream(stream)>>>(state, chunk,
                                                                               len, forget, prev);
  SKYRX_CHECK_LAUNCH("skyrx_moments_fold_keep");
  return SKYRX_OK;
}

extern "C" int skyrx_stats_finalize(const double* moments, const double* shift,
                                    const int32_t* flags, int32_t bands, int32_t batch,
                                    double* mu, double* sigma, double* chol, double* sigma_inv,
                                    double* whiten64, float* whiten, int32_t ld_w,
                                    float* mu_hilo, double* ridge, int32_t* status,
                                    void* stream) {
  SKYRX_REQUIRE(bands > 0 && bands <= 1024, "bands %d outside [1, 1024]", bands);
  SKYRX_REQUIRE(batch >= 1, "batch must be >= 1");
  SKYRX_REQUIRE(ld_w >= bands, "ld_w %d < bands %d", ld_w, bands);
  const bool general = getenv("SKYRX_B200_FIN_GENERAL") != nullptr;
  if (bands <= 128 && !general && getenv("SKYRX_B200_FIN_SLOT") == nullptr)  // finalize_panel.cu
    return launch_finalize_panel(moments, shift, flags, bands, batch, mu, sigma, chol, sigma_inv,
                                 whiten64, whiten, ld_w, mu_hilo, ridge, status,
                                 as_stream(stream));
  if (bands <= 80 && !general)  // the per-column latency kernel (finalize_small.cu)
    return launch_finalize_small(moments, shift, flags, bands, batch, mu, sigma, chol, sigma_inv,
                                 whiten64, whiten, ld_w, mu_hilo, ridge, status,
                                 as_stream(stream));
  cudaStream_t st = as_stream(stream);
  const bool wide = bands > kSmemInvMaxB;
  if (bands > 128 && bands <= 288 && !general) {  // finalize_wide.cu, then W^T W below
    const int rc = launch_finalize_wide(moments, shift, flags, bands, batch, mu, sigma, chol,
                                        whiten64, mu_hilo, ridge, status, st);
    if (rc != SKYRX_OK) return rc;
    return launch_wide_inv(whiten64, bands, batch, sigma_inv, whiten, ld_w, status, st);
  }
  const size_t sm = 2 * (size_t)bands * sizeof(double) +
                    (bands <= kSmemInvMaxB ? ((size_t)bands * (bands | 1) + (size_t)bands * bands) *
                                                 sizeof(double)
                     : bands <= kSmemCholMaxB
                         ? (size_t)bands * (bands | 1) * sizeof(double)
                         : (size_t)(bands <= 750 ? 32 : 16) * bands * sizeof(double));  // panel
  cudaFuncSetAttribute(finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  finalize_kernel<<<batch, kFinThreads, sm, st>>>(moments, shift, flags, bands, mu, sigma, chol,
                                                  sigma_inv, whiten64, whiten, ld_w, mu_hilo,
                                                  ridge, status, wide ? 0 : 1);
  SKYRX_CHECK_LAUNCH("skyrx_stats_finalize");
  if (wide) {
    const size_t xs = 32 * (size_t)bands * sizeof(double);
    cudaFuncSetAttribute(wide_trinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xs);
    wide_trinv_kernel<<<dim3(ceil_div(bands, 32), batch), 1024, xs, st>>>(chol, bands, whiten64,
                                                                          status);
    return launch_wide_inv(whiten64, bands, batch, sigma_inv, whiten, ld_w, status, st);
  }
  return SKYRX_OK;
}
