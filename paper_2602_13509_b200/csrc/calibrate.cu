// K1 — radiometric calibration (+ optional band discard / binning / RGB).
//
// Reference semantics: calibrate.py:90-102 (apply_calibration) and
// calibrate.py:135-176 (calibrate_bin_rgb).  Bit-exact: every op is a
// separately rounded f32 intrinsic and binned bands are summed left to right
// (the order the reference's band-major boolean-indexed block produces; see
// oracle/skyrx_oracle.py:sequential_sum_f32).
//
// HBM-bound elementwise map: 2 B read + 4 B write per element; the plain path
// moves 16 B of raw per thread per iteration (uint4) with float4 table loads.
#include <algorithm>
#include <type_traits>

#include "common.cuh"

namespace skyrx {

// plain apply_calibration, 8 elements (one uint4 of raw) per step
__global__ void __launch_bounds__(256) calibrate_vec8_kernel(
    const uint4* __restrict__ raw, int64_t n8, int64_t sb8, const float4* __restrict__ dark,
    const float4* __restrict__ coeff, const float* __restrict__ gain, float4* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t line = i / sb8;
    const int64_t t = i - line * sb8;  // index of the 8-group inside the line
    const uint4 r = __ldcs(raw + i);   // streamed once
    const float g = __ldg(gain + line);
    const float4 d0 = __ldg(dark + 2 * t), d1 = __ldg(dark + 2 * t + 1);
    const float4 c0 = __ldg(coeff + 2 * t), c1 = __ldg(coeff + 2 * t + 1);
    float4 o0, o1;
    o0.x = calib((float)(r.x & 0xffffu), d0.x, c0.x, g);
    o0.y = calib((float)(r.x >> 16), d0.y, c0.y, g);
    o0.z = calib((float)(r.y & 0xffffu), d0.z, c0.z, g);
    o0.w = calib((float)(r.y >> 16), d0.w, c0.w, g);
    o1.x = calib((float)(r.z & 0xffffu), d1.x, c1.x, g);
    o1.y = calib((float)(r.z >> 16), d1.y, c1.y, g);
    o1.z = calib((float)(r.w & 0xffffu), d1.z, c1.z, g);
    o1.w = calib((float)(r.w >> 16), d1.w, c1.w, g);
    __stcs(out + 2 * i, o0);
    __stcs(out + 2 * i + 1, o1);
  }
}

__global__ void __launch_bounds__(256) calibrate_scalar_kernel(
    const uint16_t* __restrict__ raw, int64_t n, int64_t sb, const float* __restrict__ dark,
    const float* __restrict__ coeff, const float* __restrict__ gain, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t line = i / sb;
    const int64_t t = i - line * sb;
    out[i] = calib((float)raw[i], __ldg(dark + t), __ldg(coeff + t), __ldg(gain + line));
  }
}

struct Rgb3 {
  int c[3];
};

// general path: one thread per output (line, sample, out_band); RAW calibrates,
// F32 re-bins an existing radiance cube
template <int KIND>
__global__ void __launch_bounds__(256) calibrate_bin_kernel(
    const void* __restrict__ src, int64_t lines, int32_t samples, int32_t bands,
    const float* __restrict__ dark, const float* __restrict__ coeff,
    const float* __restrict__ gain, const int32_t* __restrict__ keep, int32_t nout,
    int32_t factor, float* __restrict__ out, Rgb3 rgb_idx, float* __restrict__ rgb) {
  const int64_t total = lines * (int64_t)samples * nout;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pix = i / nout;
    const int32_t o = (int32_t)(i - pix * nout);
    const int64_t line = pix / samples;
    const int32_t s = (int32_t)(pix - line * samples);
    const float g = (KIND == SKYRX_IN_RAW_U16) ? __ldg(gain + line) : 1.0f;
    float acc = 0.0f;
    for (int j = 0; j < factor; ++j) {
      const int b = keep ? __ldg(keep + o * factor + j) : o * factor + j;
      float x;
      if constexpr (KIND == SKYRX_IN_RAW_U16) {
        const int64_t tb = (int64_t)s * bands + b;
        x = calib((float)reinterpret_cast<const uint16_t*>(src)[pix * bands + b],
                  __ldg(dark + tb), __ldg(coeff + tb), g);
      } else {
        x = reinterpret_cast<const float*>(src)[pix * bands + b];
      }
      acc = (j == 0) ? x : __fadd_rn(acc, x);
    }
    out[i] = acc;
    if (rgb) {
#pragma unroll
      for (int c = 0; c < 3; ++c)
        if (rgb_idx.c[c] == o) rgb[pix * 3 + c] = acc;
    }
  }
}

// tiled general path (R-FUSED at paper geometry, 1000 x 900 x 300 -> 70).  A CTA owns
// a block of SB consecutive samples over a range of lines, and every thread owns up to
// PO fixed (sample, output band) pairs of the block: their kept band indices and dark /
// coeff words sit in registers for the whole line range (the one-thread-per-output
// kernel above re-reads 2 * factor table words per output, four times the raw bytes it
// calibrates, and spends most of its issue on index divisions).  Per line, the block's
// SB x bands raw words are one contiguous range (16-byte loads into shared memory) and
// its SB x nout outputs another (coalesced stores).  Same ops, same order as calib()
// and the left-to-right band sum, so bit-identical.
// kBinBufs line buffers per CTA, kBinBufs - 1 lines in flight: at 2 CTAs per SM (121
// registers) one line in flight per CTA kept ~17 KB per SM outstanding, 0.28 of the HBM
// bandwidth at paper geometry (Little's law wants ~45 KB per SM)
#ifndef SKYRX_BIN_BUFS
#define SKYRX_BIN_BUFS 3
#endif
constexpr int kBinBufs = SKYRX_BIN_BUFS;
#ifndef SKYRX_BIN_LPS
#define SKYRX_BIN_LPS 4
#endif
constexpr int kBinLps = SKYRX_BIN_LPS;  // lines per ring slot

template <int KIND, int PO, int FMAX>
__global__ void __launch_bounds__(256) calibrate_bin_tiled_kernel(
    const void* __restrict__ src, int64_t lines, int32_t samples, int32_t bands,
    const float* __restrict__ dark, const float* __restrict__ coeff,
    const float* __restrict__ gain, const int32_t* __restrict__ keep, int32_t nout,
    int32_t factor, int32_t sb, int64_t lines_per_cta, float* __restrict__ out, Rgb3 rgb_idx,
    float* __restrict__ rgb) {
  using T = typename std::conditional<KIND == SKYRX_IN_RAW_U16, uint16_t, float>::type;
  constexpr bool kRaw = KIND == SKYRX_IN_RAW_U16;
  extern __shared__ __align__(16) unsigned char cb_smem[];
  T* tile = reinterpret_cast<T*>(cb_smem);  // [sb * bands] raw words of one line
  const int s0 = blockIdx.x * sb;
  const int ns = min(sb, samples - s0);
  const int nrow = ns * bands;
  const int nouts = ns * nout;
  // this thread's fixed (sample, output) pairs e = tid + 256 q and their tables
  int rowoff[PO], kbv[PO][FMAX];
  float dkv[PO][FMAX], ckv[PO][FMAX];
  int rgbm[PO];  // the RGB channels this output band feeds (several when targets share a band)
  bool tab_ok = true;  // every table word of this thread admits calib_fast
  // the output's FMAX bands are consecutive from an even word (discard_oob_bands keeps one
  // contiguous range): its raw counts come as FMAX/2 32-bit words
  bool pairs[PO];
  uint32_t soff[PO];  // byte offset of the output's first band word in a line buffer
#pragma unroll
  for (int q = 0; q < PO; ++q) {
    const int e = threadIdx.x + 256 * q;
    const int sl = e < nouts ? e / nout : 0, o = e < nouts ? e - sl * nout : 0;
    rowoff[q] = sl * bands;
    rgbm[q] = 0;
#pragma unroll
    for (int c = 0; c < 3; ++c)
      if (rgb_idx.c[c] == o) rgbm[q] |= 1 << c;
    pairs[q] = kRaw && factor == FMAX && FMAX % 2 == 0;
    soff[q] = 0;
#pragma unroll
    for (int j = 0; j < FMAX; ++j) {
      const int k = o * factor + (j < factor ? j : 0);
      const int b = keep ? __ldg(keep + k) : k;
      kbv[q][j] = b;
      pairs[q] = pairs[q] && b == kbv[q][0] + j && ((rowoff[q] + kbv[q][0]) & 1) == 0;
      if (j == 0) soff[q] = (uint32_t)(rowoff[q] + b) * (uint32_t)sizeof(T);
      if (kRaw) {
        const int64_t tb = (int64_t)(s0 + sl) * bands + b;
        dkv[q][j] = __ldg(dark + tb);
        ckv[q][j] = __ldg(coeff + tb);
        tab_ok = tab_ok && (dkv[q][j] == 0.0f || calib_fast_range(dkv[q][j])) &&
                 calib_fast_range(ckv[q][j]);
      }
    }
  }
  // CTA-uniform path choices (every thread's tables / band layout admit them)
  bool vec_all = kRaw;
#pragma unroll
  for (int q = 0; q < PO; ++q) vec_all = vec_all && (pairs[q] || threadIdx.x + 256 * q >= nouts);
  const bool vec_cta = __syncthreads_and(vec_all) != 0;
  const bool fast_cta = kRaw && __syncthreads_and(tab_ok) != 0;
  if (!rgb)
#pragma unroll
    for (int q = 0; q < PO; ++q) rgbm[q] = 0;
  const T* in = reinterpret_cast<const T*>(src);
  const int64_t l0 = blockIdx.y * lines_per_cta;
  const int64_t l1 = min(lines, l0 + lines_per_cta);
  const int nbytes = nrow * (int)sizeof(T);
  const int bufw = (nrow + 15) & ~15;  // words per buffer (16-byte aligned)
  const bool vec = ((((uintptr_t)in) | ((uintptr_t)samples * bands * sizeof(T)) |
                     ((uintptr_t)s0 * bands * sizeof(T))) & 15) == 0 && (nbytes & 15) == 0;
  // a ring slot holds kBinLps consecutive lines: one barrier, one wait and one fetch round
  // per kBinLps lines (the per-line control work was half the kernel's instructions)
  const int64_t nsteps = (l1 - l0 + kBinLps - 1) / kBinLps;
  auto fetch = [&](int64_t step, T* dst) {
#pragma unroll
    for (int h = 0; h < kBinLps; ++h) {
      const int64_t line = l0 + step * kBinLps + h;
      if (line >= l1) break;
      const T* g = in + (line * samples + s0) * (int64_t)bands;
      if (vec) {
        const uint32_t d0 = (uint32_t)__cvta_generic_to_shared(dst + h * bufw);
        for (int v = threadIdx.x; v < nbytes / 16; v += blockDim.x)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d0 + 16 * v),
                       "l"(reinterpret_cast<const char*>(g) + 16 * (size_t)v));
      } else {
        for (int e = threadIdx.x; e < nrow; e += blockDim.x) dst[h * bufw + e] = g[e];
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  // kBinBufs slots: steps s+1 .. s+kBinBufs-1 are in flight while step s is calibrated
  for (int b = 0; b < kBinBufs - 1; ++b) {
    if (b < nsteps) fetch(b, tile + b * kBinLps * bufw);
    else asm volatile("cp.async.commit_group;\n" ::);
  }
  for (int64_t step = 0; step < nsteps; ++step) {
    const int cur = (int)(step % kBinBufs);
    asm volatile("cp.async.wait_group %0;\n" ::"n"(kBinBufs - 2));
    __syncthreads();  // step `step` is in slot cur; the slot fetched next is free
    const int64_t nxt = step + kBinBufs - 1;
    if (nxt < nsteps) fetch(nxt, tile + (int)(nxt % kBinBufs) * kBinLps * bufw);
    else asm volatile("cp.async.commit_group;\n" ::);
#pragma unroll
    for (int h = 0; h < kBinLps; ++h) {
    const int64_t line = l0 + step * kBinLps + h;
    if (line >= l1) break;
    const T* tl = tile + (cur * kBinLps + h) * bufw;
    const float gl = kRaw ? __ldg(gain + line) : 1.0f;
    const float gi = __frcp_rn(gl);
    float* o_line = out + (line * samples + s0) * (int64_t)nout;
    float* rgb_line = rgb ? rgb + (line * samples + s0) * 3 : nullptr;
    // CTA-uniform variants: whole-word raw loads (VEC), calib_fast (FAST); the band loop is
    // fully unrolled over FMAX == factor bands with no per-element branching
    const uint32_t tl32 = (uint32_t)__cvta_generic_to_shared(tl);
    auto body = [&](auto vec_c, auto fast_c, auto one_c) {
      constexpr bool VEC = decltype(vec_c)::value, FAST = decltype(fast_c)::value;
      constexpr bool ONE = decltype(one_c)::value;  // gain 1: x / 1 == x, no division
#pragma unroll
      for (int q = 0; q < PO; ++q) {
        const int e = threadIdx.x + 256 * q;
        if (e < nouts) {
          const T* row = tl + rowoff[q];
          float rv[FMAX];
          if constexpr (VEC) {  // exact u16 -> f32: (2^23 + r) - 2^23
#pragma unroll
            for (int j = 0; j < FMAX; j += 2) {
              uint32_t v;
              asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(tl32 + soff[q] + 2 * j));
              rv[j] = __uint_as_float(__byte_perm(v, 0x4B000000u, 0x7610)) - 8388608.0f;
              rv[j + 1] = __uint_as_float(__byte_perm(v, 0x4B000000u, 0x7632)) - 8388608.0f;
            }
          } else {
#pragma unroll
            for (int j = 0; j < FMAX; ++j) rv[j] = j < factor ? (float)row[kbv[q][j]] : 0.0f;
          }
          float acc = 0.0f;
          if constexpr (kRaw && VEC && FAST && FMAX % 2 == 0) {
            // band pairs in f32x2 (same per-lane rounding), then the left-to-right sum
#pragma unroll
            for (int j = 0; j < FMAX; j += 2) {
              const float2 rr = make_float2(rv[j], rv[j + 1]);
              const float2 dd = make_float2(dkv[q][j], dkv[q][j + 1]);
              const float2 cc = make_float2(ckv[q][j], ckv[q][j + 1]);
              float2 x2;
              if constexpr (ONE) {
                const float2 t = fsub2(rr, dd);
                x2 = fmul2(make_float2(fmaxf(t.x, 0.0f), fmaxf(t.y, 0.0f)), cc);
              } else {
                x2 = calib_fast2(rr, dd, cc, gl, gi);
              }
              acc = (j == 0) ? __fadd_rn(x2.x, x2.y) : __fadd_rn(__fadd_rn(acc, x2.x), x2.y);
            }
          } else {
#pragma unroll
          for (int j = 0; j < FMAX; ++j) {
            if (VEC || j < factor) {
              float x;
              if constexpr (kRaw) {
                x = ONE ? __fmul_rn(fmaxf(__fsub_rn(rv[j], dkv[q][j]), 0.0f), ckv[q][j])
                    : FAST ? calib_fast(rv[j], dkv[q][j], ckv[q][j], gl, gi)
                           : calib(rv[j], dkv[q][j], ckv[q][j], gl);
              } else {
                x = rv[j];
              }
              acc = (j == 0) ? x : __fadd_rn(acc, x);
            }
          }
          }
          __stcs(o_line + e, acc);
          if (rgbm[q]) {
            float* px = rgb_line + (rowoff[q] / bands) * 3;
#pragma unroll
            for (int c = 0; c < 3; ++c)
              if (rgbm[q] & (1 << c)) px[c] = acc;
          }
        }
      }
    };
    using T_ = std::true_type;
    using F_ = std::false_type;
    const bool fast = fast_cta && calib_fast_range(gl);
    if (vec_cta && fast && gl == 1.0f) body(T_{}, T_{}, T_{});
    else if (vec_cta && fast) body(T_{}, T_{}, F_{});
    else if (fast) body(F_{}, T_{}, F_{});
    else body(F_{}, F_{}, F_{});
    }
  }
}

template <int KIND>
static bool launch_bin_tiled(const void* src, int64_t lines, int32_t samples, int32_t bands,
                             const float* dark, const float* coeff, const float* gain,
                             const int32_t* keep, int32_t nout, int32_t factor, float* out,
                             Rgb3 r, float* rgb, cudaStream_t st) {
  constexpr int PO = 4, FMAX = 4;  // up to 1024 outputs per CTA, bin factors up to 4
  if (factor > FMAX || nout > 256 * PO || lines < 1 || samples < 1) return false;
  const int sb = std::min(samples, (256 * PO) / nout);
  const size_t elem = KIND == SKYRX_IN_RAW_U16 ? 2 : 4;
  const size_t sm = kBinBufs * kBinLps * (((size_t)sb * bands + 15) / 16 * 16) * elem;
  if (sm > 200 * 1024) return false;
  auto k = calibrate_bin_tiled_kernel<KIND, PO, FMAX>;
  if (sm > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const int sblocks = (samples + sb - 1) / sb;
  // about 6 CTAs per SM, each over a contiguous range of lines
  int64_t ychunks = std::max<int64_t>(1, (int64_t)kSMs * 6 / sblocks);
  ychunks = std::min<int64_t>(ychunks, lines);
  const int64_t per = (lines + ychunks - 1) / ychunks;
  ychunks = (lines + per - 1) / per;
  k<<<dim3(sblocks, (unsigned)ychunks), 256, sm, st>>>(src, lines, samples, bands, dark, coeff,
                                                       gain, keep, nout, factor, sb, per, out,
                                                       r, rgb);
  return true;
}

static int grid_for(int64_t work, int threads) {
  int64_t blocks = ceil_div<int64_t>(work, threads);
  const int64_t cap = (int64_t)kSMs * 16;
  return (int)(blocks < cap ? (blocks < 1 ? 1 : blocks) : cap);
}

}  // namespace skyrx

using namespace skyrx;

extern "C" int skyrx_calibrate(const uint16_t* raw, int64_t lines, int32_t samples,
                               int32_t bands, const float* dark, const float* coeff,
                               const float* gain, const int32_t* keep, int32_t kept,
                               int32_t factor, float* out, const int32_t* rgb_idx_host,
                               float* rgb, void* stream) {
  SKYRX_REQUIRE(lines >= 0 && samples >= 0 && bands >= 0, "negative cube shape");
  SKYRX_REQUIRE(factor >= 1, "band count %d not divisible by factor %d", kept, factor);
  if (keep == nullptr) kept = bands;
  SKYRX_REQUIRE(kept % factor == 0, "band count %d not divisible by factor %d", kept, factor);
  const int64_t pixels = lines * (int64_t)samples;
  const int32_t nout = kept / factor;
  cudaStream_t st = as_stream(stream);
  if (pixels == 0 || nout == 0) return SKYRX_OK;
  const bool plain = keep == nullptr && factor == 1 && rgb == nullptr;
  if (plain) {
    const int64_t n = pixels * bands;
    const int64_t sb = (int64_t)samples * bands;
    const bool aligned = (sb % 8 == 0) && ((uintptr_t)raw % 16 == 0) &&
                         ((uintptr_t)out % 16 == 0) && ((uintptr_t)dark % 16 == 0) &&
                         ((uintptr_t)coeff % 16 == 0);
    if (aligned) {
      calibrate_vec8_kernel<<<grid_for(n / 8, 256), 256, 0, st>>>(
          (const uint4*)raw, n / 8, sb / 8, (const float4*)dark, (const float4*)coeff, gain,
          (float4*)out);
    } else {
      calibrate_scalar_kernel<<<grid_for(n, 256), 256, 0, st>>>(raw, n, sb, dark, coeff, gain,
                                                                 out);
    }
  } else {
    Rgb3 r{{-1, -1, -1}};
    if (rgb && rgb_idx_host)
      for (int c = 0; c < 3; ++c) r.c[c] = rgb_idx_host[c];
    const int64_t total = pixels * nout;
    if (!launch_bin_tiled<SKYRX_IN_RAW_U16>(raw, lines, samples, bands, dark, coeff, gain, keep,
                                            nout, factor, out, r, rgb, st))
      calibrate_bin_kernel<SKYRX_IN_RAW_U16><<<grid_for(total, 256), 256, 0, st>>>(
          raw, lines, samples, bands, dark, coeff, gain, keep, nout, factor, out, r, rgb);
  }
  SKYRX_CHECK_LAUNCH("skyrx_calibrate");
  return SKYRX_OK;
}

extern "C" int skyrx_bin_radiance(const float* in, int64_t lines, int32_t samples,
                                  int32_t bands, const int32_t* keep, int32_t kept,
                                  int32_t factor, float* out, const int32_t* rgb_idx_host,
                                  float* rgb, void* stream) {
  SKYRX_REQUIRE(lines >= 0 && samples >= 0 && bands >= 0, "negative cube shape");
  if (keep == nullptr) kept = bands;
  SKYRX_REQUIRE(factor >= 1 && kept % factor == 0, "band count %d not divisible by factor %d",
                kept, factor);
  const int64_t pixels = lines * (int64_t)samples;
  const int32_t nout = kept / factor;
  if (pixels == 0 || nout == 0) return SKYRX_OK;
  Rgb3 r{{-1, -1, -1}};
  if (rgb && rgb_idx_host)
    for (int c = 0; c < 3; ++c) r.c[c] = rgb_idx_host[c];
  if (!launch_bin_tiled<SKYRX_IN_F32>(in, lines, samples, bands, nullptr, nullptr, nullptr, keep,
                                      nout, factor, out, r, rgb, as_stream(stream)))
    calibrate_bin_kernel<SKYRX_IN_F32><<<grid_for(pixels * nout, 256), 256, 0,
                                         as_stream(stream)>>>(in, lines, samples, bands,
                                                              nullptr, nullptr, nullptr, keep,
                                                              nout, factor, out, r, rgb);
  SKYRX_CHECK_LAUNCH("skyrx_bin_radiance");
  return SKYRX_OK;
}
