// K3 for B <= 128 — blocked (panel) factorisation of one background per CTA.
//
// Replaces rx.py:56-86 (mu, unbiased symmetric sigma, ridge ladder eps * trace / B over
// RIDGE_EPSILONS rx.py:23, Cholesky, sigma_inv = cho_solve(L, I) symmetrised) and
// produces W = L^-1 (f64 and the f32 transposed copy K4 reads).
//
// finalize_small.cu advances the factor one column per CTA barrier (70 barriers plus a
// pivot chain per step at B = 70).  Here the columns come in panels of fp_panel() columns:
//   phase 1  warp 0 factors panel p in registers (lanes own rows; the pivot is broadcast
//            by a shuffle and every lane takes sqrt / 1 / l itself, so a column costs
//            one shuffle + the pivot chain + one shuffle per later panel column), while
//            warps 1..15 apply W panel p-1 to the rows of R below it;
//   phase 2  warp 0 forms W panel p (rows j of W = R_j / l_jj, lanes own columns), while
//            warps 1..15 apply L panel p to the trailing submatrix of A;
// two CTA barriers per panel instead of one per column.  Every entry sees exactly the
// operations of the right-looking column algorithm in the same order (a_it -= l_ij l_tj,
// R_it -= l_ij W_jt for ascending j, FMA-free like potrf so an exactly rank-deficient
// input meets an exactly zero pivot), so mu, sigma, L and W are bit-identical to
// finalize_small_kernel and finalize_kernel (tests/test_gpu_finalize.py); sigma_inv =
// W^T W runs the same per-entry FMA chain as finalize_small (bit-identical).
#include "common.cuh"

namespace skyrx {

constexpr int kFpThreads = 384;  // 170 registers per thread: the panel warps hold their block without spills
constexpr int kFpWarps = kFpThreads / 32;
// panel width: 8 columns, 6 for 4..6 rows per lane, 4 beyond (the register block fits)
__host__ __device__ constexpr int fp_panel(int rpl) { return rpl >= 7 ? 4 : (rpl >= 4 ? 6 : 8); }
__constant__ double kFpRidgeEps[6] = {0.0, 1e-10, 1e-9, 1e-8, 1e-7, 1e-6};  // rx.py:23

// -DSKYRX_FIN_PROFILE: clock64 at the phase boundaries of matrix 0 plus the cycles warp 0
// spends in its panels and warp 1 in its trailing updates (skyrx_fp_profile)
#ifdef SKYRX_FIN_PROFILE
__device__ long long fp_prof[16];
#define FP_T(k)                                                     \
  do {                                                              \
    __syncthreads();                                                \
    if (blockIdx.x == 0 && threadIdx.x == 0) fp_prof[k] = clock64(); \
  } while (0)
#define FP_ACC(k, ...)                                                          \
  do {                                                                          \
    const long long t0_ = clock64();                                            \
    __VA_ARGS__;                                                                \
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) atomicAdd((unsigned long long*)&fp_prof[k], \
                                                    (unsigned long long)(clock64() - t0_)); \
  } while (0)
extern "C" __attribute__((visibility("default"))) int skyrx_fp_profile(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, fp_prof, sizeof(fp_prof));
}
#else
#define FP_T(k) \
  do {          \
  } while (0)
#define FP_ACC(k, ...) __VA_ARGS__
#endif

#ifdef SKYRX_FP_NO_TRAIL  // profile experiment: warp 0's chain alone (results invalid)
constexpr bool kFpNoTrail = true;
#else
constexpr bool kFpNoTrail = false;
#endif

__device__ __forceinline__ int fp_tri_row(int e) {
  int i = (int)((sqrtf(8.0f * (float)e + 1.0f) - 1.0f) * 0.5f);
  while (i * (i + 1) / 2 > e) --i;
  while ((i + 1) * (i + 2) / 2 <= e) ++i;
  return i;
}
__device__ __forceinline__ int tri(int i) { return i * (i + 1) / 2; }

// where entry (i, t <= i) of a lower-triangular working matrix lives (packed in shared
// memory; a global-memory row-major variant for 128 < B <= 384 was 3x slower than the
// general kernels: its trailing updates serialise on L2 round trips)
struct PackedIx {
  __device__ __forceinline__ int operator()(int i, int t) const { return tri(i) + t; }
};

// warp 0: factor columns [j0, j0 + np) of A (packed lower, already updated by every
// earlier column); the panel's L entries replace them in place, pivots go to dg.
// Returns false (uniformly) on a non-positive or NaN pivot.
template <int RPL, class IX>
__device__ __forceinline__ bool chol_panel(double* Ap, IX ix, double* dg, int B, int j0) {
  constexpr int P = fp_panel(RPL);
  const int lane = threadIdx.x & 31;
  const int np = min(P, B - j0);
  // Every lane holds the panel's P x P diagonal block D (broadcast loads) and factors it
  // itself, so no lane waits on another: its own rows below take l_ic = a_ic / l_cc and
  // a_ic' -= l_ic l_c'c from its registers and D.  No shuffles (each __shfl_sync is a
  // divergence check that splits the scheduling region): the pivot chain sqrt -> 1 / l
  // -> the next a_jj - l^2 (~180 cycles) is the only serial path per column.  The block's
  // rows are also some lane's own rows: same operands, same order, same values.
  double D[P][P];
#pragma unroll
  for (int c2 = 0; c2 < P; ++c2)
#pragma unroll
    for (int c = 0; c <= c2; ++c) D[c2][c] = c2 < np ? Ap[ix(j0 + c2, j0 + c)] : 1.0;
  double a[RPL][P];
#pragma unroll
  for (int r = 0; r < RPL; ++r) {
    const int i = j0 + lane + 32 * r;
#pragma unroll
    for (int c = 0; c < P; ++c)
      a[r][c] = (i < B && c < np && j0 + c <= i) ? Ap[ix(i, j0 + c)] : 0.0;
  }
  bool bad = false;  // a failed pivot is recorded; the panel runs on in NaNs (no early exit)
#pragma unroll
  for (int c = 0; c < P; ++c) {
    const double v = D[c][c];
    bad |= c < np && !(v > 0.0);  // potrf's failure
    const double l = sqrt(v);
    const double rl = 1.0 / l;
    if (lane == 0 && c < np) dg[j0 + c] = l, dg[B + j0 + c] = rl;
#pragma unroll
    for (int c2 = c + 1; c2 < P; ++c2) D[c2][c] = D[c2][c] * rl;  // l_{c2, c}
#pragma unroll
    for (int c2 = c + 1; c2 < P; ++c2)
#pragma unroll
      for (int c3 = c + 1; c3 <= c2; ++c3)
        D[c2][c3] = __dsub_rn(D[c2][c3], __dmul_rn(D[c2][c], D[c3][c]));
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      const int i = j0 + lane + 32 * r;
      if (i > j0 + c && i < B && c < np) {
        a[r][c] = a[r][c] * rl;  // l_ic
        Ap[ix(i, j0 + c)] = a[r][c];
      }
#pragma unroll
      for (int c3 = c + 1; c3 < P; ++c3)
        a[r][c3] = __dsub_rn(a[r][c3], __dmul_rn(a[r][c], D[c3][c]));
    }
  }
  return !bad;
}

// warp 0: rows [j0, j0 + np) of W = L^-1 from R (already holding every earlier row's
// contribution): W_jt = R_jt / l_jj (R_jj = 1), then the panel's later rows take
// R_j2,t -= l_j2,j W_jt.  Lanes own columns t.
template <int RPL, class IX>
__device__ __forceinline__ void w_panel(const double* __restrict__ Ap, double* __restrict__ Rp,
                                        IX ix, const double* __restrict__ dg, int B, int j0) {
  constexpr int P = fp_panel(RPL);
  const int lane = threadIdx.x & 31;
  const int np = min(P, B - j0);
  double rr[RPL][P];
#pragma unroll
  for (int k = 0; k < RPL; ++k) {
    const int t = lane + 32 * k;
#pragma unroll
    for (int c = 0; c < P; ++c) rr[k][c] = (c < np && t < j0 + c) ? Rp[ix(j0 + c, t)] : 0.0;
  }
  // the panel's L block l_{j0+c2, j0+c} (c < c2), loaded up front: the row chain below
  // is then dmul / dsub only
  double lq[P][P];
#pragma unroll
  for (int c2 = 1; c2 < P; ++c2)
#pragma unroll
    for (int c = 0; c < c2; ++c) lq[c2][c] = c2 < np ? Ap[ix(j0 + c2, j0 + c)] : 0.0;
#pragma unroll
  double rlv[P];
#pragma unroll
  for (int c = 0; c < P; ++c) rlv[c] = c < np ? dg[B + j0 + c] : 0.0;
#pragma unroll
  for (int c = 0; c < P; ++c) {
    if (c >= np) break;
    const int j = j0 + c;
    const double rl = rlv[c];
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      const int t = lane + 32 * k;
      if (t <= j) {
        rr[k][c] = (t == j ? 1.0 : rr[k][c]) * rl;
        Rp[ix(j, t)] = rr[k][c];
      }
    }
#pragma unroll
    for (int c2 = c + 1; c2 < P; ++c2) {
      if (c2 >= np) break;
      const double lj = lq[c2][c];  // l_{j2, j}
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        const int t = lane + 32 * k;
        if (t <= j) rr[k][c2] = __dsub_rn(rr[k][c2], __dmul_rn(lj, rr[k][c]));
      }
    }
  }
}

template <int RPL>
__global__ void __launch_bounds__(kFpThreads, 1) finalize_panel_kernel(
    const double* __restrict__ moments_all, const double* __restrict__ shift_all,
    const int32_t* __restrict__ flags_all, int B, double* __restrict__ mu_all,
    double* __restrict__ sigma_all, double* __restrict__ chol_all,
    double* __restrict__ inv_all, double* __restrict__ w64_all, float* __restrict__ wf_all,
    int ld_w, float* __restrict__ mhl_all, double* __restrict__ ridge_all,
    int32_t* __restrict__ status_all) {
  constexpr int P = fp_panel(RPL);
  extern __shared__ __align__(16) double fp[];
  __shared__ double red[kFpWarps];
  __shared__ int fail;
  const int T = B * (B + 1) / 2;
  double* Sp = fp;        // packed lower sigma
  double* Ap = Sp + T;    // packed lower A (+ ridge) -> L, panel by panel, in place
  double* Rp = Ap + T;    // packed lower R -> W = L^-1 (diagonal: W_jj = 1 / l_jj)
  double* dg = Rp + T;    // [l_jj | 1 / l_jj]
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
  FP_T(0);

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
  for (int b = tid; b < B; b += kFpThreads) {  // rx.py:59
    const double mb = shift[b] + s[b] / n;
    mu[b] = mb;
    const float hi = (float)mb;
    mhl[b] = hi;
    mhl[B + b] = (float)(mb - (double)hi);
  }
  // sigma (rx.py:65-66), symmetric by construction, and its trace
  // four entries per thread in flight: their global loads first, then the arithmetic
  for (int e0 = tid; e0 < T; e0 += 4 * kFpThreads) {
    int ii[4], kk[4];
    double qa[4], qb[4], si[4], sk[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * kFpThreads;
      ii[u] = 0, kk[u] = 0, qa[u] = qb[u] = si[u] = sk[u] = 0.0;
      if (e < T) {
        ii[u] = fp_tri_row(e), kk[u] = e - tri(ii[u]);
        qa[u] = q[(size_t)ii[u] * B + kk[u]];
        qb[u] = q[(size_t)kk[u] * B + ii[u]];
        si[u] = s[ii[u]], sk[u] = s[kk[u]];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * kFpThreads;
      if (e < T) {
        const double vik = (qa[u] - si[u] * sk[u] / n) / (n - 1.0);
        const double vki = (qb[u] - sk[u] * si[u] / n) / (n - 1.0);
        const double v = (vik + vki) / 2.0;
        Sp[e] = v;
        sigma[(size_t)ii[u] * B + kk[u]] = v;
        sigma[(size_t)kk[u] * B + ii[u]] = v;
      }
    }
  }
  __syncthreads();
  // the trace in the general kernel's order (ridge = eps * trace / B must match it bitwise)
  double tr = 0.0;
  for (int b = tid; b < B; b += kFpThreads) tr += Sp[tri(b) + b];
  tr = warp_sum(tr);
  if (lane == 0) red[warp] = tr;
  __syncthreads();
  double trace = 0.0;
  for (int w = 0; w < kFpWarps; ++w) trace += red[w];  // fixed order: deterministic
  const double scale = trace > 0.0 ? trace / B : 1.0;
  FP_T(1);

  double ridge = 0.0;
  bool ok = false;
  const int wt = tid - 32, nwt = kFpThreads - 32;  // warps 1..15: the trailing updates
#pragma unroll 1
  for (int a = 0; a < 6 && !ok; ++a) {
    ridge = kFpRidgeEps[a] * scale;
    __syncthreads();  // every read of `fail` from the previous attempt is done
    for (int e = tid; e < T; e += kFpThreads) {
      const int i = fp_tri_row(e), t = e - tri(i);
      Ap[e] = Sp[e] + (i == t ? ridge : 0.0);
      Rp[e] = 0.0;
    }
    if (tid == 0) fail = 0;
    __syncthreads();
    bool failed = false;
    for (int j0 = 0; j0 < B; j0 += P) {
      // ---- phase 1: factor panel p | R rows >= j0 take W panel p-1
      if (warp == 0) {
        bool okp;
        FP_ACC(5, okp = chol_panel<RPL>(Ap, PackedIx{}, dg, B, j0));
        if (!okp && lane == 0) fail = 1;
      } else if (j0 > 0 && !kFpNoTrail) FP_ACC(7, {
        const int p0 = j0 - P;
        const int cnt = (B - j0) * j0;
        for (int e = wt; e < cnt; e += nwt) {
          const int i = j0 + e / j0, t = e - (e / j0) * j0;
          const double* li = Ap + tri(i);
          double x = Rp[tri(i) + t];
          for (int j = max(p0, t); j < j0; ++j) x = __dsub_rn(x, __dmul_rn(li[j], Rp[tri(j) + t]));
          Rp[tri(i) + t] = x;
        }
      });
      __syncthreads();
      if (fail) {
        failed = true;
        break;
      }
      // ---- phase 2: W panel p | the trailing submatrix takes L panel p
      const int j1 = min(j0 + P, B);
      if (warp == 0) {
        FP_ACC(6, w_panel<RPL>(Ap, Rp, PackedIx{}, dg, B, j0));
      } else if (!kFpNoTrail) FP_ACC(8, {
        const int mm = B - j1;
        const int cnt = mm * (mm + 1) / 2;
        for (int e = wt; e < cnt; e += nwt) {
          const int ii = fp_tri_row(e), tt = e - tri(ii);
          const int i = j1 + ii, t = j1 + tt;
          const double* li = Ap + tri(i);
          const double* lt = Ap + tri(t);
          double x = li[t];
          for (int j = j0; j < j1; ++j) x = __dsub_rn(x, __dmul_rn(li[j], lt[j]));
          Ap[tri(i) + t] = x;
        }
      });
      __syncthreads();
    }
    ok = !failed;
  }
  if (!ok) {
    if (tid == 0) {
      status_all[m] = SKYRX_ERR_NOT_PD;
      ridge_all[m] = ridge;
    }
    return;
  }
  FP_T(2);
  const double* Wp = Rp;
  // sigma_inv = W^T W (= cho_solve(L, I)): inv_ij = sum_{k >= i} W_ki W_kj, per entry the
  // same ascending-k FMA chain as finalize_small's 4 x 4 tiles, here over 2 x 2 tiles so
  // every thread holds one (i in I..I+1 >= j in J..J+1)
  const int nb = (B + 1) >> 1;
  for (int tile = tid; tile < nb * (nb + 1) / 2; tile += kFpThreads) {
    const int ta = fp_tri_row(tile), tb = tile - tri(ta);
    const int I = 2 * ta, J = 2 * tb;
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll 4
    for (int k = I; k < B; ++k) {
      const double* row = Wp + tri(k);
      double wa[2], wb[2];
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        wa[p] = (I + p <= k) ? row[I + p] : 0.0;  // W_ki = 0 above the diagonal
        wb[p] = (J + p <= k) ? row[J + p] : 0.0;
      }
#pragma unroll
      for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int r = 0; r < 2; ++r) acc[p][r] += wa[p] * wb[r];
    }
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int i = I + p, jj = J + r;
        if (i < B && jj <= i) {
          inv[(size_t)i * B + jj] = acc[p][r];
          inv[(size_t)jj * B + i] = acc[p][r];
        }
      }
  }
  FP_T(3);
  // L (upper zeros), W (f64, upper zeros), the f32 transposed copy for K4
  for (int i = warp; i < B; i += kFpWarps)
#pragma unroll 4
    for (int c = lane; c < B; c += 32) {
      chol[(size_t)i * B + c] = c < i ? Ap[tri(i) + c] : (c == i ? dg[i] : 0.0);
      w64[(size_t)i * B + c] = c <= i ? Wp[tri(i) + c] : 0.0;
    }
  for (int k = warp; k < ld_w; k += kFpWarps)
    for (int j = lane; j < ld_w; j += 32)
      wf[(size_t)k * ld_w + j] = (j < B && k < B && k <= j) ? (float)Wp[tri(j) + k] : 0.0f;
  FP_T(4);
  if (tid == 0) {
    status_all[m] = SKYRX_OK;
    ridge_all[m] = ridge;
  }
}

size_t finalize_panel_smem(int B) {
  const size_t T = (size_t)B * (B + 1) / 2;
  return (3 * T + 2 * (size_t)B) * sizeof(double);
}

// launched by skyrx_stats_finalize for 1 <= B <= 128
int launch_finalize_panel(const double* moments, const double* shift, const int32_t* flags,
                          int B, int batch, double* mu, double* sigma, double* chol,
                          double* sigma_inv, double* w64, float* wf, int ld_w, float* mhl,
                          double* ridge, int32_t* status, cudaStream_t st) {
  const size_t sm = finalize_panel_smem(B);
#define SKYRX_FP(rpl)                                                                          \
  if (B <= 32 * (rpl)) {                                                                       \
    cudaFuncSetAttribute(finalize_panel_kernel<rpl>,                                           \
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);                \
    finalize_panel_kernel<rpl><<<batch, kFpThreads, sm, st>>>(                                 \
        moments, shift, flags, B, mu, sigma, chol, sigma_inv, w64, wf, ld_w, mhl, ridge,       \
        status);                                                                               \
    SKYRX_CHECK_LAUNCH("skyrx_stats_finalize/panel");                                          \
    return SKYRX_OK;                                                                           \
  }
  SKYRX_FP(1) SKYRX_FP(2) SKYRX_FP(3) SKYRX_FP(4)
#undef SKYRX_FP
  set_error("finalize_panel: B = %d too large", B);
  return SKYRX_ERR_ARG;
}

}  // namespace skyrx
