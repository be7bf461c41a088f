// Pixel-tile loader shared by the Gram (K2) and score (K4) kernels.
//
// A tile is P consecutive pixels of a BIP cube; its bytes are contiguous
// (P * B * elem).  Each element is calibrated on the fly (RAW kind, bit-exact
// calibrate.py:98-101) or read (F32/F64 kinds), centred, and stored to shared
// memory as d[p * ld + b] in the arithmetic type T:
//   T = float : v = (x - sub_hi[b]) - sub_lo[b]   (two-term f32 centring)
//   T = double: v = double(x) - sub64[b]           (precise mode)
// Padding bands/pixels are written as 0 so they contribute nothing.
#pragma once
#include "common.cuh"

namespace skyrx {

struct CubeRef {
  const void* pixels;   // uint16 raw, float32 radiance or float64 pixels
  const float* dark;    // (S, B)  RAW only
  const float* coeff;   // (S, B)  RAW only
  const float* gain;    // (L,)    RAW only
  int64_t npix;         // L * S
  int32_t samples;
  int32_t bands;
};

// Returns false if any input/calibrated value is non-finite.
template <int KIND, typename T>
__device__ __forceinline__ bool load_tile(const CubeRef& c, int64_t p0, int P, int ld, int bp,
                                          const float* __restrict__ sub_hi,
                                          const float* __restrict__ sub_lo,
                                          const double* __restrict__ sub64, T* __restrict__ d,
                                          int32_t* s_line, int32_t* s_samp,
                                          bool* clamped = nullptr) {
  const int B = c.bands;
  const int NT = blockDim.x;
  if constexpr (KIND == SKYRX_IN_RAW_U16) {
    // per-pixel (line, sample) once per tile
    for (int p = threadIdx.x; p < P; p += NT) {
      const int64_t pix = p0 + p;
      if (pix < c.npix) {
        const int64_t line = pix / c.samples;
        s_line[p] = (int32_t)line;
        s_samp[p] = (int32_t)(pix - line * c.samples);
      } else {
        s_line[p] = -1;
        s_samp[p] = 0;
      }
    }
    __syncthreads();
  }
  bool ok = true;
  const int total = P * bp;
  for (int e = threadIdx.x; e < total; e += NT) {
    const int p = e / bp;
    const int b = e - p * bp;
    T v = T(0);
    const int64_t pix = p0 + p;
    if (b < B && pix < c.npix) {
      const int64_t gi = pix * (int64_t)B + b;
      if constexpr (KIND == SKYRX_IN_F64) {
        const double x = __ldg(reinterpret_cast<const double*>(c.pixels) + gi);
        ok &= (bool)isfinite(x);
        v = (T)(x - sub64[b]);
      } else {
        float x;
        if constexpr (KIND == SKYRX_IN_RAW_U16) {
          const int64_t tb = (int64_t)s_samp[p] * B + b;
          const float r = (float)__ldg(reinterpret_cast<const uint16_t*>(c.pixels) + gi);
          const float dk = __ldg(c.dark + tb);
          if (clamped && r < dk) *clamped = true;  // calibrate.py:99 clamps this value
          x = calib(r, dk, __ldg(c.coeff + tb), __ldg(c.gain + s_line[p]));
        } else {
          x = __ldg(reinterpret_cast<const float*>(c.pixels) + gi);
        }
        ok &= finite_f(x);
        if constexpr (sizeof(T) == 4) {
          float t = __fsub_rn(x, sub_hi[b]);
          if (sub_lo) t = __fsub_rn(t, sub_lo[b]);
          v = t;
        } else {
          v = (double)x - sub64[b];
        }
      }
    }
    d[p * ld + b] = v;
  }
  return ok;
}

}  // namespace skyrx
