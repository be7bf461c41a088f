// K3 for B <= 80 — latency-bound factorisation of one background per CTA (B > 80 keeps
// the general kernels: past 10 chunks per warp the slot registers spill).
//
// Replaces rx.py:56-86 (mu, unbiased symmetric sigma, ridge ladder eps * trace / B
// over RIDGE_EPSILONS rx.py:23, Cholesky, sigma_inv = cho_solve(L, I) symmetrised)
// and produces W = L^-1 (f64 and the f32 transposed copy K4 reads).
//
// The general finalize_kernel (stats.cu) walks the matrix in shared memory with a
// warp per row: 1650 cycles per Cholesky column and 1040 per row of L^-1 at B = 70
// (tools/fin_profile.sh), 115 us per matrix for the two loops.  Here the factor and the
// inverse advance together, one barrier per step j.  The lower triangle is a set of
// SLOTS (i, t), t <= i: slot (i, t) holds a_it while t > j (right-looking Cholesky),
// emits l_ij at step j = t and from then on holds R_it, the right-looking forward
// substitution of W = L^-1 (R_i = e_i - sum_{k<j} l_ik W_k).  So row i has i + 1 live
// slots at every step j < i and the work per step is the inherent (B - j)(B + j) / 2.
// Rows are cut into 32-slot chunks dealt to warps 1..15 (registers); warp 0 takes the
// pivots (l_{j+1,j+1} is computed at the start of step j from the slot values of step
// j-1, so its sqrt and division overlap the step), writes column j of L and row j of W.
// The slot matrix is double-buffered in shared memory by step parity: step j reads
// M[j & 1] (column j, row j) and every live slot writes its new value to M[~j & 1].
//   t > j:   a_it -= (a_ij / l_jj)(a_tj / l_jj)      FMA-free, so like LAPACK potrf an
//                                                    exactly rank-deficient input meets
//                                                    an exactly zero pivot and fails;
//   t <= j:  R_it -= (a_ij / l_jj)(R_jt / l_jj);     row j of W = R_j / l_jj is final.
// Operands and rounding are the general kernel's (its W loop is FMA-free as well), so
// sigma, L and W are bit-identical to it; sigma_inv = W^T W is summed over 4 x 4
// register tiles.  B = 70: 67 us per call against the general kernel's 123 us
// (tools/time_finalize.py; the step is bound by the per-step barrier + pivot chain and
// the per-warp chunk chain, ~1500 cycles, tools/fs_profile.sh and tools/step_probe.cu).
#include "common.cuh"

namespace skyrx {

constexpr int kFsThreads = 512;
constexpr int kFsWarps = kFsThreads / 32;
__constant__ double kRidgeEps[6] = {0.0, 1e-10, 1e-9, 1e-8, 1e-7, 1e-6};  // rx.py:23

// -DSKYRX_FIN_PROFILE: clock64 at the phase boundaries of matrix 0 (skyrx_fs_profile)
#ifdef SKYRX_FIN_PROFILE
__device__ long long fs_prof[8];
#define FS_T(k)                                                     \
  do {                                                              \
    __syncthreads();                                                \
    if (blockIdx.x == 0 && threadIdx.x == 0) fs_prof[k] = clock64(); \
  } while (0)
extern "C" __attribute__((visibility("default"))) int skyrx_fs_profile(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, fs_prof, sizeof(fs_prof));
}
#else
#define FS_T(k) \
  do {          \
  } while (0)
#endif

__device__ __forceinline__ int tri_row(int e) {
  int i = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
  while (i * (i + 1) / 2 > e) --i;
  while ((i + 1) * (i + 2) / 2 <= e) ++i;
  return i;
}

// pivot j: LAPACK potrf fails on a non-positive or NaN pivot (marked by a NaN 1/l_jj)
__device__ __forceinline__ void pivot_root(double v, double* dg, int B, int j) {
  if (!(v > 0.0)) {
    dg[B + j] = __longlong_as_double(0x7ff8000000000000LL);
  } else {
    const double l = sqrt(v);
    dg[j] = l, dg[B + j] = 1.0 / l;
  }
}

// number of 32-slot row chunks of a B-band triangle (row i has i + 1 slots)
__host__ __device__ inline int fs_chunks(int B) {
  int c = 0;
  for (int i = 0; i < B; ++i) c += (i + 32) / 32;
  return c;
}

template <int CH>
__global__ void __launch_bounds__(kFsThreads, 1) finalize_small_kernel(
    const double* __restrict__ moments_all, const double* __restrict__ shift_all,
    const int32_t* __restrict__ flags_all, int B, double* __restrict__ mu_all,
    double* __restrict__ sigma_all, double* __restrict__ chol_all,
    double* __restrict__ inv_all, double* __restrict__ w64_all, float* __restrict__ wf_all,
    int ld_w, float* __restrict__ mhl_all, double* __restrict__ ridge_all,
    int32_t* __restrict__ status_all) {
  extern __shared__ __align__(16) double fs[];
  __shared__ double red[kFsWarps];
  const int T = B * (B + 1) / 2;
  // M[2]: the slot matrix (packed lower) after step j-1 (read at step j) and after step j
  // (written at step j); slot (i, t) = a_it while t > j, then R_it (see the header)
  double* M0 = fs;
  double* Wp = M0 + 2 * T;     // packed lower W = L^-1
  double* dg = Wp + T;         // [l_jj | 1 / l_jj (NaN: failed)]
  double* sig = M0;            // packed lower sigma, only until the first attempt starts
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
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  FS_T(0);

  const double n = mom[0];
  const double* s = mom + 1;
  const double* q = mom + 1 + B;
  int status = SKYRX_OK;
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
  for (int b = tid; b < B; b += kFsThreads) {  // rx.py:59
    const double mb = shift[b] + s[b] / n;
    mu[b] = mb;
    const float hi = (float)mb;
    mhl[b] = hi;
    mhl[B + b] = (float)(mb - (double)hi);
  }
  // this warp's row chunks: the chunks (row i, slots t0..t0+31) listed rows descending,
  // dealt round-robin to warps 1..15 (warp 0 takes the pivots); packed (i << 16) | t0,
  // -1 = none
  int cw[CH];
#pragma unroll
  for (int u = 0; u < CH; ++u) cw[u] = -1;
  if (warp > 0) {
    int c = 0;
    for (int i = B - 1; i >= 0; --i)
      for (int t0 = 0; t0 <= i; t0 += 32, ++c)
        if (c % (kFsWarps - 1) == warp - 1) {
          const int u = c / (kFsWarps - 1);
#pragma unroll
          for (int v = 0; v < CH; ++v)
            if (v == u) cw[v] = (i << 16) | t0;
        }
  }
  // sigma (rx.py:65-66), symmetric by construction, and its trace
  for (int e = tid; e < T; e += kFsThreads) {
    const int i = tri_row(e), k = e - i * (i + 1) / 2;
    const double vik = (q[(size_t)i * B + k] - s[i] * s[k] / n) / (n - 1.0);
    const double vki = (q[(size_t)k * B + i] - s[k] * s[i] / n) / (n - 1.0);
    const double v = (vik + vki) / 2.0;
    sig[e] = v;
    sigma[(size_t)i * B + k] = v;
    sigma[(size_t)k * B + i] = v;
  }
  __syncthreads();
  // the trace in the general kernel's order (ridge = eps * trace / B must match it bitwise)
  double tr = 0.0;
  for (int b = tid; b < B; b += kFsThreads) tr += sig[b * (b + 1) / 2 + b];
  tr = warp_sum(tr);
  if (lane == 0) red[warp] = tr;
  __syncthreads();
  double trace = 0.0;
  for (int w = 0; w < kFsWarps; ++w) trace += red[w];  // fixed order: deterministic
  const double scale = trace > 0.0 ? trace / B : 1.0;
  FS_T(1);

  double ridge = 0.0;
  bool ok = false;
  double X[CH];  // slot (i, t0 + lane): a_it while t > j (factor), then R_it (inverse row)
  int po[CH], ptt[CH];  // the slot's packed offset; t (t + 1) / 2 (its column walk)
#pragma unroll
  for (int u = 0; u < CH; ++u) {
    const int i = cw[u] >> 16, t = (cw[u] & 0xffff) + lane;
    po[u] = (cw[u] >= 0 && t <= i) ? i * (i + 1) / 2 + t : -1;
    ptt[u] = t <= i ? t * (t + 1) / 2 : i * (i + 1) / 2;  // dead lanes read in bounds
  }
  __syncthreads();  // sig (= M0) has been read
#pragma unroll 1
  for (int a = 0; a < 6 && !ok; ++a) {
    ridge = kRidgeEps[a] * scale;
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int i = cw[u] >> 16, t = (cw[u] & 0xffff) + lane;
      X[u] = 0.0;
      if (po[u] >= 0) {
        X[u] = sigma[(size_t)i * B + t] + (i == t ? ridge : 0.0);
        M0[po[u]] = X[u];
      }
    }
    __syncthreads();
    if (tid == 0) pivot_root(M0[0], dg, B, 0);  // R_00 = 1 is implicit (see below)
    int j = 0;
    for (; j < B; ++j) {
      __syncthreads();  // M after step j-1 and pivot j are visible
      const double rl = dg[B + j];
      if (rl != rl) break;  // pivot j failed (NaN marker): uniform
      const double* Mr = M0 + (j & 1) * T;
      double* Mw = M0 + ((j + 1) & 1) * T;
      const int tj = j * (j + 1) / 2;
      // V_j[t]: t > j -> a_tj = Mr[t (t+1)/2 + j];  t < j -> R_jt = Mr[tj + t];  t == j -> 1
      if (warp == 0) {
        if (tid == 0 && j + 1 < B) {
          // the next pivot: a_{j+1,j+1} after this step, the owner's operands and order
          const double x = Mr[(j + 1) * (j + 2) / 2 + j] * rl;
          pivot_root(__dsub_rn(Mr[(j + 1) * (j + 2) / 2 + j + 1], __dmul_rn(x, x)), dg, B, j + 1);
        }
        for (int i = j + lane; i < B; i += 32)  // column j of L: l_jj, l_ij = a_ij / l_jj
          chol[(size_t)i * B + j] = (i == j) ? dg[j] : Mr[i * (i + 1) / 2 + j] * rl;
        for (int t = lane; t <= j; t += 32)     // row j of W = R_j / l_jj
          Wp[tj + t] = (t == j ? 1.0 : Mr[tj + t]) * rl;
        continue;
      }
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        const int i = cw[u] >> 16;  // warp-uniform
        if (i <= j) break;          // rows descend with u: every later chunk is done (or none)
        const int t = (cw[u] & 0xffff) + lane;
        const double vt = t > j ? Mr[ptt[u] + j] : (t == j ? 1.0 : Mr[tj + t]);
        const double x = vt * rl;                         // l_tj  |  W_jt
        const double lij = Mr[i * (i + 1) / 2 + j] * rl;  // l_ij, a broadcast
        // t > j: a_it -= l_ij l_tj;  t == j: the slot becomes R_ij = 0 - l_ij W_jj;
        // t < j: R_it -= l_ij W_jt.  FMA-free throughout (potrf)
        X[u] = __dsub_rn(t == j ? 0.0 : X[u], __dmul_rn(lij, x));
        if (po[u] >= 0) Mw[po[u]] = X[u];
      }
    }
    ok = (j == B);
    __syncthreads();
  }
  FS_T(2);
  if (!ok) {
    if (tid == 0) {
      status_all[m] = SKYRX_ERR_NOT_PD;
      ridge_all[m] = ridge;
    }
    return;
  }
  // sigma_inv = W^T W (= cho_solve(L, I)): inv_ij = sum_{k >= i} W_ki W_kj over 4 x 4
  // tiles (i in I..I+3 >= j in J..J+3), 8 loads per 16 products
  const int nb = (B + 3) >> 2;
  for (int tile = tid; tile < nb * (nb + 1) / 2; tile += kFsThreads) {
    const int ta = tri_row(tile), tb = tile - ta * (ta + 1) / 2;
    const int I = 4 * ta, J = 4 * tb;
    double acc[4][4];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[p][r] = 0.0;
    for (int k = I; k < B; ++k) {
      const double* row = Wp + k * (k + 1) / 2;
      double wa[4], wb[4];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        wa[p] = (I + p <= k) ? row[I + p] : 0.0;  // W_ki = 0 above the diagonal
        wb[p] = (J + p <= k) ? row[J + p] : 0.0;
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[p][r] += wa[p] * wb[r];
    }
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int i = I + p, jj = J + r;
        if (i < B && jj <= i) {
          inv[(size_t)i * B + jj] = acc[p][r];
          inv[(size_t)jj * B + i] = acc[p][r];
        }
      }
  }
  FS_T(3);
  // W (f64, upper zeros), the factor's upper zeros, the f32 transposed copy for K4
  for (int e = tid; e < (int)BB; e += kFsThreads) {
    const int i = e / B, c = e - i * B;
    w64[e] = c <= i ? Wp[i * (i + 1) / 2 + c] : 0.0;
    if (c > i) chol[e] = 0.0;
  }
  for (int e = tid; e < ld_w * ld_w; e += kFsThreads) {
    const int k = e / ld_w, j = e - k * ld_w;
    wf[e] = (j < B && k < B && k <= j) ? (float)Wp[j * (j + 1) / 2 + k] : 0.0f;
  }
  FS_T(4);
  if (tid == 0) {
    status_all[m] = SKYRX_OK;
    ridge_all[m] = ridge;
  }
}

size_t finalize_small_smem(int B) {
  const size_t T = (size_t)B * (B + 1) / 2;
  return (3 * T + 2 * (size_t)B) * sizeof(double);
}

// launched by skyrx_stats_finalize for 1 <= B <= 128
int launch_finalize_small(const double* moments, const double* shift, const int32_t* flags,
                          int B, int batch, double* mu, double* sigma, double* chol,
                          double* sigma_inv, double* w64, float* wf, int ld_w, float* mhl,
                          double* ridge, int32_t* status, cudaStream_t st) {
  const int per_warp = (fs_chunks(B) + kFsWarps - 2) / (kFsWarps - 1);
  const size_t sm = finalize_small_smem(B);
#define SKYRX_FS(ch)                                                                          \
  if (per_warp <= (ch)) {                                                                     \
    cudaFuncSetAttribute(finalize_small_kernel<ch>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         (int)sm);                                                            \
    finalize_small_kernel<ch><<<batch, kFsThreads, sm, st>>>(                                 \
        moments, shift, flags, B, mu, sigma, chol, sigma_inv, w64, wf, ld_w, mhl, ridge,      \
        status);                                                                              \
    SKYRX_CHECK_LAUNCH("skyrx_stats_finalize/small");                                         \
    return SKYRX_OK;                                                                          \
  }
  SKYRX_FS(2) SKYRX_FS(4) SKYRX_FS(8) SKYRX_FS(10)
#undef SKYRX_FS
  set_error("finalize_small: B = %d too large", B);
  return SKYRX_ERR_ARG;
}

}  // namespace skyrx
