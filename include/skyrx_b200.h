/*
 * skyrx_b200.h — C ABI of the B200 (sm_100a) calibrate + RX hot path.
 *
 * Drop-in boundary for the reference package `skyrx` (arXiv 2602.13509,
 * /root/reference/pkg/src/skyrx).  The reference is Python; its only native
 * slot on this path is `skyrx._accel` (numba, _accel.py:19-31 / 109-131).  A
 * maintainer binds this library with ctypes exactly as INTEGRATION.md shows;
 * paper_2602_13509_b200/_lib.py is that binding.
 *
 * Conventions
 *   - every pointer argument is a DEVICE pointer unless its name ends in _host;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream);
 *   - cubes are C-order (lines, samples, bands), bands innermost (BIP,
 *     cube.py:80-105); pixel n = line * samples + sample;
 *   - every call is asynchronous on `stream`, re-entrant and thread-safe (no
 *     global scratch: callers pass workspaces), and returns an int status;
 *     skyrx_last_error() gives the calling thread's last message;
 *   - results are deterministic: no floating-point atomics anywhere.
 */
#ifndef SKYRX_B200_H_
#define SKYRX_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* status codes (host return values and per-matrix device status words) */
#define SKYRX_OK 0
#define SKYRX_ERR_ARG 1          /* bad argument; message in skyrx_last_error()  */
#define SKYRX_ERR_CUDA 2         /* CUDA runtime error                           */
#define SKYRX_ERR_INSUFFICIENT 3 /* rx.py:51-52 "insufficient samples"          */
#define SKYRX_ERR_NONFINITE 4    /* rx.py:53-54 "non-finite values"             */
#define SKYRX_ERR_NOT_PD 5       /* rx.py:79-80 "not positive definite ..."     */
#define SKYRX_ERR_RANGE 6        /* tensor-core quantiser overflow: recompute    */

/* pixel source kinds */
#define SKYRX_IN_RAW_U16 0 /* uint16 raw counts + (dark, coeff, gain) calibration */
#define SKYRX_IN_F32 1     /* float32 radiance (RadianceCube.values)             */
#define SKYRX_IN_F64 2     /* float64 pixels (only skyrx_mahalanobis_sq)         */

const char* skyrx_version(void);
const char* skyrx_last_error(void);
int skyrx_device_check(void); /* 0 if a sm_100 device is visible */

/* ---------------------------------------------------------------- K1 calibration
 * Replaces calibrate.py:90-102 (apply_calibration: keep == NULL, factor == 1)
 * and calibrate.py:135-176 (calibrate_bin_rgb).  out[l,s,o] = sum over j<factor,
 * left to right in f32, of max(0, f32(raw[l,s,keep[o*factor+j]]) - dark) * coeff
 * / gain[l]; each op IEEE round-to-nearest (bit-exact vs the reference).
 * rgb (nullable) receives out[..., rgb_idx[c]] for c < 3 (calibrate.py:129-132).
 */
int skyrx_calibrate(const uint16_t* raw, int64_t lines, int32_t samples, int32_t bands,
                    const float* dark, const float* coeff, const float* gain,
                    const int32_t* keep, int32_t kept, int32_t factor,
                    float* out, const int32_t* rgb_idx_host, float* rgb, void* stream);

/* Same band selection / binning / RGB on an f32 radiance cube:
 * discard_oob_bands (calibrate.py:105-114), bin_bands (calibrate.py:117-126),
 * extract_rgb (calibrate.py:129-132). */
int skyrx_bin_radiance(const float* in, int64_t lines, int32_t samples, int32_t bands,
                       const int32_t* keep, int32_t kept, int32_t factor, float* out,
                       const int32_t* rgb_idx_host, float* rgb, void* stream);

/* ---------------------------------------------------------------- K2 background moments
 * Moments block layout (float64): [n, s[B], Q[B*B]] with shift c:
 *   s = sum(x - c), Q = sum((x - c)(x - c)^T)  (Q stored full, symmetric).
 * This is the payload all-reduced across GPUs (SURVEY §8 R-GLOBAL) and folded
 * by forgetting (R-STREAM).  Equivalent to rx.py:56-66's two passes up to FP64
 * rounding once finalized.
 */
size_t skyrx_moments_len(int32_t bands); /* 1 + B + B*B doubles */

/* shift c[b] = f32(mean of a strided sample of <= 4096 pixels), stored as f64 */
int skyrx_stats_shift(int32_t kind, const void* pixels, int64_t lines, int32_t samples,
                      int32_t bands, const float* dark, const float* coeff, const float* gain,
                      double* shift, void* stream);

int skyrx_stats_workspace(int64_t lines, int32_t samples, int32_t bands, size_t* bytes);

/* Accumulate moments of all pixels of the cube (fused calibration for RAW).
 * precise = 0: f32 products, f32 runs of <= 192 products promoted to f64
 *              (fast path; SURVEY §7 precision budget);
 * precise = 1: f64 products and sums throughout (reference-grade, for the
 *              drop-in compute_stats and the reference's 1e-9 suites).
 * flags[0] |= 1 if any calibrated value is non-finite (rx.py:53-54); for RAW
 * input also |= 128 (the clamp check ran) and |= 64 if a raw value was below
 * dark (calibrate.py:99 clamps it).  "No clamp anywhere" = flags 8 without 4
 * (raw-byte pass) or 128 without 64 (this pass): the exact-digit score kernels
 * need it. */
int skyrx_stats_accumulate(int32_t kind, const void* pixels, int64_t lines, int32_t samples,
                           int32_t bands, const float* dark, const float* coeff,
                           const float* gain, const double* shift, int32_t precise,
                           double* moments, int32_t* flags, void* workspace,
                           size_t workspace_bytes, void* stream);

/* Tensor-core (tcgen05 kind::i8) moments for RAW cubes with B <= 79: values
 * quantised to 21-bit fixed point around the sample shift (skyrx_quant_shift
 * gives c_b and 2^e_b), three int8 digits, exact int32 digit Gram.  Writes
 * the same [n, s, Q] moments block; flags |= 2 if a value fell outside the
 * quantiser range (caller then recomputes with skyrx_stats_accumulate). */
int skyrx_stats_tc_supported(int64_t lines, int32_t samples, int32_t bands, const void* raw);
size_t skyrx_stats_tc_workspace(int32_t bands);
int skyrx_quant_shift(int32_t kind, const void* pixels, int64_t lines, int32_t samples,
                      int32_t bands, const float* dark, const float* coeff, const float* gain,
                      double* shift, float* qinv, void* stream);
int skyrx_stats_tc(const uint16_t* raw, int64_t lines, int32_t samples, int32_t bands,
                   const float* dark, const float* coeff, const float* gain, const double* shift,
                   const float* qinv, double* moments, int32_t* flags, void* workspace,
                   size_t workspace_bytes, void* stream);

/* The same quantised-digit tensor-core moments of an already calibrated f32 radiance cube
 * (replaces compute_stats(cube) rx.py:42-66 for mode="fast" on a RadianceCube, B <= 79,
 * samples*bands*4 % 16 == 0); shift / qinv from skyrx_quant_shift(SKYRX_IN_F32, ...).
 * flags |= 1 on a non-finite value, |= 2 if the quantiser range overflowed (then use
 * skyrx_stats_accumulate). */
int skyrx_stats_tc_f32(const float* pixels, int64_t lines, int32_t samples, int32_t bands,
                       const double* shift, const float* qinv, double* moments, int32_t* flags,
                       void* workspace, size_t workspace_bytes, void* stream);

/* Raw-byte tensor-core moments (RAW cubes, one constant line gain, B <= 128,
 * samples*bands*2 % 16 == 0): exact integer byte Grams per sample column
 * (tcgen05 kind::i8, TMA-fed), calibration applied per sample in f64.  Same
 * [n, s, Q] moments about `shift`; flags |= 4 if any value clamps at 0.  For
 * windows <= 256 bytes (B <= 128) the clamped pixels are then corrected exactly
 * in the same call (the moments kernel marks them while their tile is on chip,
 * a sparse kernel adds their corrections) and flags |= 256: the moments are
 * final (finalize accepts 4 with 256).  Wider windows (B > 128) leave 4
 * without 256: the caller recomputes with another path.  workspace >=
 * skyrx_stats_raw_workspace(bands) (>= skyrx_stats_raw_workspace_for(L, S, B) for the
 * clamp correction). */
int skyrx_stats_raw_supported(int64_t lines, int32_t samples, int32_t bands, const void* raw);
size_t skyrx_stats_raw_workspace(int32_t bands);
/* workspace that also holds the clamp correction's pixel bitmap (L * S bits); with only
 * skyrx_stats_raw_workspace(bands) bytes a clamp leaves flags 4 without 256 */
size_t skyrx_stats_raw_workspace_for(int64_t lines, int32_t samples, int32_t bands);
int skyrx_stats_raw(const uint16_t* raw, int64_t lines, int32_t samples, int32_t bands,
                    const float* dark, const float* coeff, double gain, const double* shift,
                    double* moments, int32_t* flags, void* workspace, size_t workspace_bytes,
                    void* stream);
/* The same, with the shift chosen by the call: shift (OUT, B f64) = f32(mean) of
 * the cube from its exact sums, so no separate skyrx_stats_shift pass is needed. */
int skyrx_stats_raw_own_shift(const uint16_t* raw, int64_t lines, int32_t samples, int32_t bands,
                              const float* dark, const float* coeff, double gain, double* shift,
                              double* moments, int32_t* flags, void* workspace,
                              size_t workspace_bytes, void* stream);

/* state = forget * state + chunk (R-STREAM exponential forgetting) */
int skyrx_moments_fold(double* state, const double* chunk, int32_t bands, double forget,
                       void* stream);
/* the same, copying the pre-fold state to prev (StreamingRX's undo point for a chunk whose
 * moments must be redone) in the same launch */
int skyrx_moments_fold_keep(double* state, const double* chunk, int32_t bands, double forget,
                            double* prev, void* stream);

/* ---------------------------------------------------------------- K3 factorisation
 * Replaces rx.py:56-86 finalisation: mu, unbiased symmetric sigma, ridge
 * ladder eps in (0,1e-10,...,1e-6)*trace/B (rx.py:23, 68-80), Cholesky,
 * sigma_inv = cho_solve(L, I) symmetrised (rx.py:82-83), plus the f32 whitening
 * matrix W = L^-1 (padded to ld_w columns) and mu split into f32 hi/lo for K4.
 * Batched over `batch` independent matrices (strips): array i starts at
 * i * (its per-matrix size).  status[i] = SKYRX_OK / ERR_INSUFFICIENT /
 * ERR_NONFINITE / ERR_NOT_PD.  flags may be NULL.
 */
int skyrx_stats_finalize(const double* moments, const double* shift, const int32_t* flags,
                         int32_t bands, int32_t batch, double* mu, double* sigma,
                         double* chol, double* sigma_inv, double* whiten64, float* whiten,
                         int32_t ld_w, float* mu_hilo, double* ridge, int32_t* status,
                         void* stream);

/* W = L^-1 (f64 B*B workspace), its f32 transposed padded copy (ld_w*ld_w)
 * and mu hi/lo, from caller-supplied CubeStats (rx_scores(cube, stats)). */
int skyrx_whiten_prepare(const double* chol, const double* mu, int32_t bands, double* whiten64,
                         float* whiten, int32_t ld_w, float* mu_hilo, void* stream);

/* ---------------------------------------------------------------- K4 RX scores
 * Replaces rx.py:89-97 + _accel.py:75-90 for a whole cube: delta = ||W (x - mu)||^2
 * with x calibrated on the fly (kind RAW) or read (kind F32); f32 out (L,S).
 * max_bits (nullable, device uint32, pre-zeroed) receives atomicMax of the
 * order-preserving key of every score (ScoreMap.max_score, cube.py:174-176);
 * keys: f2ord(x) = bits ^ (sign ? 0xffffffff : 0x80000000).
 */
int skyrx_score(int32_t kind, const void* pixels, int64_t lines, int32_t samples,
                int32_t bands, const float* dark, const float* coeff, const float* gain,
                const float* mu_hilo, const float* whiten, int32_t ld_w, float* scores,
                uint32_t* max_bits, void* stream);

/* Tensor-core (tcgen05) variant of skyrx_score for RAW cubes with B <= 80:
 * f16 hi/lo split of (x - mu) and of W, f32 TMEM accumulation, sum of squares
 * in the epilogue.  wpack = skyrx_pack_whiten(whiten64) (skyrx_wpack_bytes(B)
 * bytes per matrix).  flags (nullable) = the moments-pass flags word: when it
 * reads 8 (raw-byte path ran, no value below dark) the clamp is skipped.
 * gain may be NULL: every line gain is 1 (the transform drops the division).
 * topk_hist0 (nullable) = skyrx_topk_histogram(ws) after skyrx_topk_init: the
 * kernel adds the digit-0 histogram of its scores, so the select continues
 * with skyrx_topk_pick(0) instead of a first skyrx_topk_hist pass.
 * skyrx_score_tc_supported() says whether the shape and
 * alignment allow it (every line segment of a tile must be a 16-B multiple). */
size_t skyrx_wpack_bytes(int32_t bands);
int skyrx_pack_whiten(const double* whiten64, int32_t bands, int32_t batch, void* wpack,
                      void* stream);
int skyrx_score_tc_supported(int64_t lines, int32_t samples, int32_t bands, const void* raw);
int skyrx_score_tc(const uint16_t* raw, int64_t lines, int32_t samples, int32_t bands,
                   const float* dark, const float* coeff, const float* gain,
                   const float* mu_hilo, const void* wpack, const int32_t* flags,
                   float* scores, uint32_t* max_key, uint32_t* topk_hist0, void* stream);

/* Exact-digit tensor-core score (raw-byte moments path ran, no clamp, one gain,
 * B <= 128): per sample column s, z = V_s a + q_s with the integer deviations
 * a = r - R_s (R_s = rint(dark + mu g / coeff)) split into two f16-exact digits
 * and V_s = W diag(coeff_s / g) in f16 hi/lo.  skyrx_score_prep writes one
 * record per sample (skyrx_score_rec_bytes(B) bytes each; batch backgrounds of
 * samples records, background i from whiten64 + i*B*B and mu_hilo + i*2B with the
 * SAME dark/coeff/gain).  Raw counts >= 4096 set flags |= 16 (the digit split
 * assumes 12-bit data): the caller then rescores with skyrx_score_tc. */
size_t skyrx_score_rec_bytes(int32_t bands);
int skyrx_score_prep(const double* whiten64, const float* mu_hilo, int32_t samples,
                     int32_t bands, const float* dark, const float* coeff, double gain,
                     int32_t batch, void* records, void* stream);
int skyrx_score_tcs_supported(int64_t lines, int32_t samples, int32_t bands, const void* raw);
int skyrx_score_tcs(const uint16_t* raw, int64_t lines, int32_t samples, int32_t bands,
                    const void* records, int32_t* flags, float* scores, uint32_t* max_key,
                    uint32_t* topk_hist0, void* stream);

/* The same for wide cubes, 128 < B <= 272 (even B): V_s streamed in N-blocks of
 * 64 rows per tile (records from skyrx_scorew_prep, skyrx_scorew_rec_bytes(B)
 * each).  The kernel scores nothing and sets flags |= 32 unless the moments
 * pass proved "no clamp" (flags 8 w/o 4 or 128 w/o 64); raw >= 4096 sets 16. */
size_t skyrx_scorew_rec_bytes(int32_t bands);
int skyrx_scorew_prep(const double* whiten64, const float* mu_hilo, int32_t samples,
                      int32_t bands, const float* dark, const float* coeff, double gain,
                      int32_t batch, void* records, void* stream);
int skyrx_scorew_supported(int64_t lines, int32_t samples, int32_t bands, const void* raw);
int skyrx_scorew(const uint16_t* raw, int64_t lines, int32_t samples, int32_t bands,
                 const void* records, int32_t* flags, float* scores, uint32_t* max_key,
                 uint32_t* topk_hist0, void* stream);

/* The kernel slot itself: _accel.mahalanobis_sq(pixels, mu, chol_lower)
 * (_accel.py:109-131) with FP64 arithmetic; pixels f32 or f64 (kind F32/F64).
 * whiten64 is a f64 workspace of B*B + BP*BP doubles, BP = 8*ceil(B/8). */
int skyrx_mahalanobis_sq(int32_t kind, const void* pixels, int64_t n, int32_t bands,
                         const double* mu, const double* chol, double* whiten64,
                         double* out, void* stream);

/* ---------------------------------------------------------------- K5 normalise / threshold / top-k
 * rx.py:100-105: out = v / f32(max) unless max <= 0 (then a copy);
 * rx.py:108-112: mask = v > t in f32.  max_bits from skyrx_score or skyrx_max. */
int skyrx_max(const float* v, int64_t n, uint32_t* max_bits, void* stream);
int skyrx_normalize(const float* v, int64_t n, const uint32_t* max_bits, float* out,
                    void* stream);
int skyrx_threshold(const float* v, int64_t n, float t, uint8_t* mask, void* stream);
/* rx.py:115-124: out = sqrt(max(f64(v) / max_score, 0)), zeros if max_score <= 0 */
int skyrx_transmit_domain(const float* v, int64_t n, double max_score, double* out,
                          void* stream);

/* R-TOPK: thr = the (k+1)-th largest value (-inf if k >= n) by a
 * 3-digit radix select; mask = v > thr.  workspace from skyrx_topk_workspace. */
size_t skyrx_topk_workspace(void);
int skyrx_topk_threshold(const float* v, int64_t n, int64_t k, float* thr, void* workspace,
                         void* stream);
int skyrx_mask_gt(const float* v, int64_t n, const float* thr, uint8_t* mask, void* stream);

/* The same select split into its steps, for a threshold over values spread
 * across ranks (R-GLOBAL): init with the GLOBAL n and k, then
 * for digit 0..2: skyrx_topk_hist on the local values, SUM all-reduce of the
 * skyrx_topk_hist_len() uint32 bins at skyrx_topk_histogram(workspace), and
 * skyrx_topk_pick (identical on every rank, since the bins are identical).
 * skyrx_topk_threshold == init + 3 x (hist + pick) on one rank. */
int skyrx_topk_init(int64_t n_total, int64_t k, void* workspace, void* stream);
int skyrx_topk_hist(const float* v, int64_t n, int32_t digit, void* workspace, void* stream);
int skyrx_topk_pick(int32_t digit, void* workspace, float* thr, void* stream);
uint32_t* skyrx_topk_histogram(void* workspace);
int32_t skyrx_topk_hist_len(void);

/* R-TOPK threshold AND mask in one pass over the scores (single rank): after
 * skyrx_topk_init(n, k, ws) and — if hist0_done — the digit-0 histogram fused
 * into a score kernel (topk_hist0 = skyrx_topk_histogram(ws)), writes
 * thr = the (k+1)-th largest value and mask = v > thr, identical to
 * skyrx_topk_threshold + skyrx_mask_gt.  cand: cand_cap 8-byte slots for the
 * values inside the threshold's top-11-bit bin (overflow or n >= 2^32 falls
 * back to a rescan, still exact).  v 16-B aligned, mask 4-B aligned. */
int skyrx_topk_mask(const float* v, int64_t n, int32_t hist0_done, float* thr, uint8_t* mask,
                    void* workspace, void* cand, int64_t cand_cap, void* stream);

/* ---------------------------------------------------------------- link payload (next to the path)
 * datalink.py:141-177: per pixel [RGB565 | half(sqrt(score / max))] little-endian u16
 * words.  skyrx_link_maxima: keys[0..3] = order-preserving u32 keys of the cube's max
 * score and max R, G, B (rgb is (n, 3) f32); skyrx_link_payload encodes with them,
 * or (keys == NULL) with max_host_host[0..3] = max_score, max_r, max_g, max_b. */
int skyrx_link_maxima(const float* scores, const float* rgb, int64_t n, uint32_t* keys,
                      void* stream);
int skyrx_link_payload(const float* scores, const float* rgb, int64_t n, const uint32_t* keys,
                       const double* max_host, uint16_t* payload, void* stream);
/* Whole line packets (datalink.py:176-189, 205-240): row l of `packets` (lines x (128 + 4S)
 * bytes) = headers[l] (128 bytes, host-built, its four f32 maxima at bytes 32..47 replaced by
 * the device keys) followed by the S payload words of line l. */
int skyrx_link_packets(const float* scores, const float* rgb, int lines, int samples,
                       const uint32_t* keys, const uint8_t* headers, uint8_t* packets,
                       void* stream);
/* The cube's whole frame stream in one matrix (datalink.py:243-285): lines / group_k groups of
 * group_k data frames then group_r parity frames, each row 8 + 128 + 4S bytes = frame head
 * (u32 group id = gid0 + g, u8 index, u8 kind, u16 length) + packet. Data rows are filled
 * here; parity payloads are left to skyrx_gf_matmul over the data rows (their heads are
 * written here). */
int skyrx_link_frames(const float* scores, const float* rgb, int lines, int samples,
                      const uint32_t* keys, const uint8_t* headers, int group_k, int group_r,
                      int gid0, uint8_t* frames, void* stream);

/* ---- GF(256) Reed-Solomon erasure code (fec.py:101-195) ----------------
 * skyrx_gf_matmul: for g < groups, out_g (r x n, row pitch opitch) = M_g (r x k, row-major)
 * times D_g (k x n, row pitch dpitch) over GF(2^8) with polynomial 0x11D; M_g = mat +
 * g * mat_gstride (0: one matrix for all), D_g = data + g * d_gstride, out_g likewise.
 * Replaces _accel.gf256_matmul (_accel.py:50-70, 92-107): parity = E[k:] @ group payloads
 * (fec.py:140-155), recovered = inv(E[rows])[absent] @ received (fec.py:182-191). */
int skyrx_gf_matmul(const uint8_t* mat, int64_t mat_gstride, int r, int k, const uint8_t* data,
                    int64_t dpitch, int64_t d_gstride, int64_t n, uint8_t* out, int64_t opitch,
                    int64_t o_gstride, int groups, void* stream);
/* skyrx_gf_invert: per problem g, invert the k x k matrix whose row i is row rows[g*k + i] of
 * `mat` (row length ld) by Gauss-Jordan (fec.py:82-98) and write its rows sel[g*k + 0 ..
 * nsel[g]-1] to out + g*k*k, zero rows after them; status[g] = 1 if singular, else 0. */
int skyrx_gf_invert(const uint8_t* mat, int ld, const int32_t* rows, int k, const int32_t* sel,
                    const int32_t* nsel, int groups, uint8_t* out, int32_t* status, void* stream);

/* ---------------------------------------------------------------- synthetic sensor (bench/test inputs)
 * Bit-identical to oracle/synth.py generate_lines(): raw counts for lines
 * [line0, line0 + nlines) of the seeded scene.  Tables as in SceneTables. */
int skyrx_synth_raw(uint32_t seedkey, uint32_t cellkey, int32_t samples, int32_t bands,
                    int32_t components, const uint32_t* cw24, const float* mean,
                    const float* factor, const float* sd, const float* aspec,
                    const float* asd, const float* xbar, const float* dark,
                    const float* coeff, int64_t line0, int64_t nlines, uint16_t* out,
                    void* stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* SKYRX_B200_H_ */
