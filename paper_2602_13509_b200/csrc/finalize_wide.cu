// K3 for 128 < B <= 288 (BASELINE config 3, B = 270): blocked factorisation, one CTA of
// 1024 threads per background, then a column-blocked L^-1 over ceil(B/32) CTAs.
//
// Replaces rx.py:56-86 like finalize_kernel (stats.cu), whose wide form factors one
// column per barrier with the trailing matrix in global memory (644 us at B = 270) and
// solves W = L^-1 one row per L2 round trip (270 us).  Here:
//   fw_factor_kernel  left-looking panels of 32 columns.  A panel's 32 x (B - p0) entries
//                     live in registers (lane = panel column, warp = row slice) and take
//                     the updates of every finished column k < p0 in ascending k from
//                     32-column chunks of L staged in shared memory (cp.async, double
//                     buffered); the panel is then
//                     factored in shared memory column by column (one barrier per column,
//                     the next pivot taken by the thread that finalises it).  Every entry
//                     sees a_ik -= l_ij l_kj for ascending j, FMA-free, with the same l
//                     values (a * (1 / l_jj)) as the right-looking column algorithm, so L is
//                     bit-identical to finalize_kernel (tests/test_gpu_finalize.py) and an
//                     exactly rank-deficient input meets the same zero pivot (potrf);
//   fw_trinv_kernel   W = L^-1 by 32-column blocks, one CTA each: block row I of the
//                     block column J is T = L_I,[J,I) X_[J,I) (one entry per thread, a
//                     dot product over shared memory) followed by a 32-step substitution
//                     with L_II (one warp per column, lane = row, L_II read from shared memory);
//   wide_inv_kernel   (stats.cu) sigma_inv = W^T W and the f32 copy.
#include "common.cuh"

namespace skyrx {

constexpr int kFwThreads = 1024;
constexpr int kFwMaxB = 288;  // two L chunks + the panel in shared memory
constexpr int kFwMaxQ = (kFwMaxB + 31) / 32;  // row slices per warp
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__constant__ double kFwRidgeEps[6] = {0.0, 1e-10, 1e-9, 1e-8, 1e-7, 1e-6};  // rx.py:23

constexpr int kFwLdc = 34;

// one 32-column chunk of the left-looking update for the Q row slices of this warp: rows
// r = warp + 32 qq of the panel column `lane` (lt: the column's own l_jk, transposed)
template <int Q>
__device__ __forceinline__ void fw_left_chunk(double (&acc)[kFwMaxQ], const double* Lcur,
                                              const double* lt, int warp, int nr) {
#pragma unroll 2
  for (int kk = 0; kk < 32; kk += 2) {
    const double l0 = lt[kk * 32], l1 = lt[(kk + 1) * 32];
#pragma unroll
    for (int qq = 0; qq < Q; ++qq) {
      const int r = warp + 32 * qq;
      if (qq < Q - 1 || r < nr) {
        const double2 a = *reinterpret_cast<const double2*>(Lcur + r * kFwLdc + kk);
        acc[qq] = __dsub_rn(acc[qq], __dmul_rn(a.x, l0));
        acc[qq] = __dsub_rn(acc[qq], __dmul_rn(a.y, l1));
      }
    }
  }
}

// -DSKYRX_FW_PROFILE: cycles of matrix 0 spent in the left-looking updates, the panel
// factorisations and the write-backs (skyrx_fw_profile; tools/fw_profile.sh)
#ifdef SKYRX_FW_PROFILE
__device__ long long fw_prof[4];
#define FW_MARK(t) \
  __syncthreads(); \
  const long long t = clock64()
#define FW_ACC(k, a, b) \
  if (blockIdx.x == 0 && threadIdx.x == 0) fw_prof[k] += (b) - (a)
extern "C" __attribute__((visibility("default"))) int skyrx_fw_profile(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, fw_prof, sizeof(fw_prof));
}
#else
#define FW_MARK(t)
#define FW_ACC(k, a, b)
#endif

// the trace exactly as finalize_kernel sums it with its 512 threads (per-thread entry, warp
// tree, serial over the 16 warps): the ridge (and so L) must not depend on the CTA size
__device__ __forceinline__ double fw_trace(const double* sigma, int B, double* scratch) {
  double v = 0.0;
  if (threadIdx.x < 512)
    for (int b = threadIdx.x; b < B; b += 512) v += sigma[(size_t)b * B + b];
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0 && w < 16) scratch[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int i = 0; i < 16; ++i) r += scratch[i];
    scratch[32] = r;
  }
  __syncthreads();
  const double r = scratch[32];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(kFwThreads, 1) fw_factor_kernel(
    const double* __restrict__ moments_all, const double* __restrict__ shift_all,
    const int32_t* __restrict__ flags_all, int B, double* __restrict__ mu_all,
    double* __restrict__ sigma_all, double* __restrict__ chol_all, float* __restrict__ mhl_all,
    double* __restrict__ ridge_all, int32_t* __restrict__ status_all) {
  extern __shared__ __align__(16) double fws[];
  __shared__ double scratch[40];
  __shared__ int s_fail;
  const int ldc = kFwLdc;        // chunk row stride (even: 16-B rows)
  const int ldp = B | 1;         // panel column stride
  const size_t chunk = (size_t)B * kFwLdc;
  double* Lc = fws;              // [2][B][34]: 32 finished columns of L, rows p0..B-1
  double* LT = Lc + 2 * chunk;   // [2][32][32]: the chunk's first 32 rows, transposed
  // [32][ldp]: the panel, column-major, absolute rows p0.. (index p0 + r, r < B - p0); it
  // aliases the chunk buffers, which are idle between the left-looking update and the next
  // panel's first fetch
  double* P = Lc;
  const size_t BB = (size_t)B * B;
  const int m = blockIdx.x;
  const double* mom = moments_all + (size_t)m * (1 + B + BB);
  const double* shift = shift_all + (size_t)m * B;
  double* mu = mu_all + (size_t)m * B;
  double* sigma = sigma_all + (size_t)m * BB;
  double* chol = chol_all + (size_t)m * BB;
  float* mhl = mhl_all + (size_t)m * 2 * B;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  const double n = mom[0];
  const double* s = mom + 1;
  const double* q = mom + 1 + B;
  int status = SKYRX_OK;
  if (flags_all && flags_range(flags_all[m])) status = SKYRX_ERR_RANGE;
  if (flags_all && (flags_all[m] & 1)) status = SKYRX_ERR_NONFINITE;
  if (!(n > (double)B)) status = SKYRX_ERR_INSUFFICIENT;  // rx.py:51 checks size first
  if (status != SKYRX_OK) {
    if (tid == 0) status_all[m] = status, ridge_all[m] = 0.0;
    return;
  }
  for (int b = tid; b < B; b += kFwThreads) {  // rx.py:59
    const double mb = shift[b] + s[b] / n;
    mu[b] = mb;
    const float hi = (float)mb;
    mhl[b] = hi;
    mhl[B + b] = (float)(mb - (double)hi);
  }
  // sigma (rx.py:65-66) with finalize_kernel's expression: a warp per row
  for (int i = warp; i < B; i += kFwThreads / 32)
    for (int j = lane; j < B; j += 32) {
      const double vij = (q[(size_t)i * B + j] - s[i] * s[j] / n) / (n - 1.0);
      const double vji = (q[(size_t)j * B + i] - s[j] * s[i] / n) / (n - 1.0);
      sigma[(size_t)i * B + j] = (vij + vji) / 2.0;
    }
  __syncthreads();
  const double trace = fw_trace(sigma, B, scratch);
  const double scale = trace > 0.0 ? trace / B : 1.0;

  double ridge = 0.0;
  bool ok = false;
  for (int a = 0; a < 6 && !ok; ++a) {
    ridge = kFwRidgeEps[a] * scale;
    if (tid == 0) s_fail = 0;
    __syncthreads();
    for (int p0 = 0; p0 < B; p0 += 32) {
      const int nb = min(32, B - p0), nr = B - p0;
      FW_MARK(ta);
      // ---- panel entries (row p0 + r, column p0 + lane) in registers, rows r = warp + 32 qq
      double acc[kFwMaxQ];
#pragma unroll
      for (int qq = 0; qq < kFwMaxQ; ++qq) {
        const int r = warp + 32 * qq;
        acc[qq] = 0.0;
        if (r < nr && lane < nb && r >= lane)
          acc[qq] = sigma[(size_t)(p0 + r) * B + p0 + lane] + (r == lane ? ridge : 0.0);
      }
      // ---- left-looking update by the finished columns k < p0, 32 at a time, ascending;
      // chunk c + 1 streams into the other buffer (cp.async) while chunk c is applied.  A
      // chunk is L[p0.., c0..c0+31] row-major (rows 16-B aligned: two k per broadcast load)
      // plus its first 32 rows transposed (the panel columns' own l_jk, one per lane)
      const int ne = nr * 32;  // chunk entries (row, column)
      auto fetch = [&](int c0, int buf) {
        double* dst = Lc + buf * chunk;
        double* dt = LT + buf * 1024;
        for (int e = tid; e < ne; e += kFwThreads) {
          const double* src = chol + (size_t)(p0 + (e >> 5)) * B + c0 + (e & 31);
          cp_async8(dst + (e >> 5) * ldc + (e & 31), src);
          if (e < 1024) cp_async8(dt + (e & 31) * 32 + (e >> 5), src);
        }
        cp_async_commit();
      };
      if (p0 > 0) fetch(0, 0);
      const int nq = (nr + 31) / 32;  // row slices of the busiest warp (CTA-uniform)
      for (int c0 = 0; c0 < p0; c0 += 32) {
        const int buf = (c0 >> 5) & 1;
        if (c0 + 32 < p0) {
          fetch(c0 + 32, buf ^ 1);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncthreads();
        if (lane < nb) {
          const double* Lcur = Lc + buf * chunk;
          const double* lt = LT + buf * 1024 + lane;
          switch (nq) {  // only the row slices this panel has (no predicated-off FP64 work)
#define FW_LEFT(Q) \
  case Q: fw_left_chunk<Q>(acc, Lcur, lt, warp, nr); break;
            FW_LEFT(1) FW_LEFT(2) FW_LEFT(3) FW_LEFT(4) FW_LEFT(5) FW_LEFT(6) FW_LEFT(7)
            FW_LEFT(8) FW_LEFT(9)
#undef FW_LEFT
          }
        }
        __syncthreads();
      }
#pragma unroll
      for (int qq = 0; qq < kFwMaxQ; ++qq) {
        const int r = warp + 32 * qq;
        if (r < nr) P[lane * ldp + p0 + r] = acc[qq];
      }
      __syncthreads();
      FW_MARK(tb);
      FW_ACC(0, ta, tb);
      // ---- factor the panel: warp w owns panel column w in registers (lanes = rows
      // p0 + lane + 32 u).  Step jj: warp jj's column is final — it takes the pivot (sqrt,
      // 1 / l), scales its rows and publishes the column; one barrier; every warp w > jj
      // subtracts l_rj l_wj (the right-looking order and rounding, FMA-free)
      double x[kFwMaxQ];
#pragma unroll
      for (int u = 0; u < kFwMaxQ; ++u) {
        const int r = lane + 32 * u;
        x[u] = (warp < nb && r < nr) ? P[warp * ldp + p0 + r] : 0.0;
      }
      for (int jj = 0; jj < nb; ++jj) {
        if (warp == jj) {
          const double v = __shfl_sync(0xffffffffu, x[0], jj);
          if (!(v > 0.0)) {  // LAPACK potrf: non-positive or NaN pivot fails
            if (lane == 0) s_fail = 1;
          } else {
            const double l = sqrt(v), rl = 1.0 / l;
#pragma unroll
            for (int u = 0; u < kFwMaxQ; ++u) {
              const int r = lane + 32 * u;
              if (r < nr && r > jj) {
                x[u] = x[u] * rl;
                P[jj * ldp + p0 + r] = x[u];
              }
            }
            if (lane == jj) x[0] = l, P[jj * ldp + p0 + jj] = l;
          }
        }
        __syncthreads();
        if (s_fail) break;  // uniform: set before the barrier
        if (warp > jj && warp < nb) {
          const double* lj = P + jj * ldp + p0;
          const double lwj = lj[warp];
#pragma unroll
          for (int u = 0; u < kFwMaxQ; ++u) {
            const int r = lane + 32 * u;
            if (r < nr && r >= warp) x[u] = __dsub_rn(x[u], __dmul_rn(lj[r], lwj));
          }
        }
      }
      FW_MARK(tc);
      FW_ACC(1, tb, tc);
      if (s_fail) break;  // uniform
      // the finished panel of L -> global (row-major), a warp per row, lanes along columns
      for (int r = p0 + warp; r < B; r += kFwThreads / 32)
        if (lane < nb && r >= p0 + lane) chol[(size_t)r * B + p0 + lane] = P[lane * ldp + r];
      __syncthreads();
      FW_MARK(td);
      FW_ACC(2, tc, td);
    }
    ok = (s_fail == 0);
    __syncthreads();
  }
  if (!ok) {
    if (tid == 0) status_all[m] = SKYRX_ERR_NOT_PD, ridge_all[m] = ridge;
    return;
  }
  for (int i = warp; i < B; i += kFwThreads / 32)  // the strict upper triangle
    for (int j = i + 1 + lane; j < B; j += 32) chol[(size_t)i * B + j] = 0.0;
  if (tid == 0) status_all[m] = SKYRX_OK, ridge_all[m] = ridge;
}

// W = L^-1, block column J (32 columns) per CTA: rows 32 J.. by 32-row blocks
__global__ void __launch_bounds__(kFwThreads, 1) fw_trinv_kernel(
    const double* __restrict__ chol_all, int B, double* __restrict__ w64_all,
    const int32_t* __restrict__ status_all) {
  extern __shared__ __align__(16) double tws[];
  const int m = blockIdx.y;
  if (status_all[m] != SKYRX_OK) return;
  const int J = blockIdx.x, c0 = 32 * J;
  const int nc = min(32, B - c0);
  const int ldx = 33;
  const int ldl = (B - c0) | 1;
  double* X = tws;                            // [B - c0][33]: rows c0.. of the block column
  double* Lb = X + (size_t)(B - c0) * ldx;    // [32][ldl]: rows of block I, columns c0..
  double* T = Lb + 32 * (size_t)ldl;          // [32][33]
  const double* L = chol_all + (size_t)m * B * B;
  double* W = w64_all + (size_t)m * B * B;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = warp; i < c0; i += 32)  // rows above the block: zero
    if (lane < nc) W[(size_t)i * B + c0 + lane] = 0.0;
  for (int i0 = c0; i0 < B; i0 += 32) {
    const int nrow = min(32, B - i0), kw = i0 + nrow - c0;  // L block columns c0 .. i0 + nrow
    for (int e = tid; e < nrow * kw; e += kFwThreads) {
      const int r = e / kw, k = e - r * kw;
      Lb[r * ldl + k] = L[(size_t)(i0 + r) * B + c0 + k];
    }
    __syncthreads();
    // T[r][c] = sum_{k in [c0, i0)} L[i0 + r][k] X[k][c]  (warp = r, lane = c)
    {
      double t0 = 0.0, t1 = 0.0;
      if (warp < nrow) {
        const double* lr = Lb + warp * ldl;
        int k = 0;
        for (; k + 1 < i0 - c0; k += 2) {
          t0 = fma(lr[k], X[k * ldx + lane], t0);
          t1 = fma(lr[k + 1], X[(k + 1) * ldx + lane], t1);
        }
        if (k < i0 - c0) t0 = fma(lr[k], X[k * ldx + lane], t0);
      }
      T[warp * 33 + lane] = t0 + t1;
    }
    __syncthreads();
    // L_II X_I = E - T: warp = column c, lane = row r; 32 steps
    {
      const int c = warp, r = lane;
      const double* lrow = Lb + (r < nrow ? r : 0) * ldl + (i0 - c0);  // L_II row r (shared)
      const double rinv = r < nrow ? 1.0 / lrow[r] : 0.0;
      double b = ((i0 == c0 && r == c) ? 1.0 : 0.0) - T[r * 33 + c];
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const double lk = (k < nrow && r > k && r < nrow) ? lrow[k] : 0.0;
        const double xk = __shfl_sync(0xffffffffu, b * rinv, k);
        if (r == k) b = xk;
        else b = fma(-lk, xk, b);
      }
      if (r < nrow) X[(i0 - c0 + r) * ldx + c] = b;
    }
    __syncthreads();
  }
  for (int i = c0 + warp; i < B; i += 32)
    if (lane < nc) W[(size_t)i * B + c0 + lane] = X[(i - c0) * ldx + lane];
}

size_t finalize_wide_factor_smem(int B) {
  return (2 * (size_t)B * kFwLdc + 2 * 1024) * sizeof(double);
}
size_t finalize_wide_trinv_smem(int B) {
  return ((size_t)B * 33 + 32 * (size_t)(B | 1) + 32 * 33) * sizeof(double);
}

// launched by skyrx_stats_finalize for 128 < B <= kFwMaxB; the caller adds wide_inv_kernel
int launch_finalize_wide(const double* moments, const double* shift, const int32_t* flags, int B,
                         int batch, double* mu, double* sigma, double* chol, double* w64,
                         float* mhl, double* ridge, int32_t* status, cudaStream_t st) {
  SKYRX_REQUIRE(B > 32 && B <= kFwMaxB, "finalize_wide: B = %d outside (32, %d]", B, kFwMaxB);
  const size_t sf = finalize_wide_factor_smem(B), sw = finalize_wide_trinv_smem(B);
  cudaFuncSetAttribute(fw_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sf);
  fw_factor_kernel<<<batch, kFwThreads, sf, st>>>(moments, shift, flags, B, mu, sigma, chol, mhl,
                                                   ridge, status);
  SKYRX_CHECK_LAUNCH("skyrx_stats_finalize/wide factor");
  cudaFuncSetAttribute(fw_trinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sw);
  fw_trinv_kernel<<<dim3(ceil_div(B, 32), batch), kFwThreads, sw, st>>>(chol, B, w64, status);
  SKYRX_CHECK_LAUNCH("skyrx_stats_finalize/wide trinv");
  return SKYRX_OK;
}

}  // namespace skyrx
