// Shared device helpers for the skyrx B200 hot path (sm_100a).
//
// Numerics contract: calibration is reproduced bit for
// bit, so every f32 op on that path is an explicitly rounded intrinsic
// (__fsub_rn/__fmul_rn/__fdiv_rn): no FMA contraction, no fast-math, and
// subnormals are kept (a 1e-40 gain must still overflow to inf,
// test_pipeline.py:84-102).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <cstdarg>

#include "../../include/skyrx_b200.h"

namespace skyrx {

constexpr int kSMs = 148;
constexpr size_t kSmemMax = 232448;  // 227 KB opt-in dynamic shared memory per CTA

// ------------------------------------------------------------------ errors
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);

#define SKYRX_CHECK_LAUNCH(what)                                         \
  do {                                                                    \
    cudaError_t _e = cudaGetLastError();                                  \
    if (_e != cudaSuccess) return ::skyrx::cuda_status(_e, what);         \
  } while (0)

#define SKYRX_REQUIRE(cond, ...)                                          \
  do {                                                                    \
    if (!(cond)) {                                                        \
      ::skyrx::set_error(__VA_ARGS__);                                    \
      return SKYRX_ERR_ARG;                                               \
    }                                                                     \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ------------------------------------------------------------------ math
// calibrate.py:98-101: out = max(0, f32(raw) - dark) * coeff / gain, each op RN.
__device__ __forceinline__ float calib(float raw, float dark, float coeff, float gain) {
  float t = __fsub_rn(raw, dark);
  t = t < 0.0f ? 0.0f : t;  // np.maximum keeps NaN (a NaN dark must stay non-finite)
  t = __fmul_rn(t, coeff);
  return __fdiv_rn(t, gain);
}

// calib() with the division by the line gain as a multiplication by y = RN(1/g) plus one
// FMA correction (Markstein: y within half an ulp of 1/g and q within one ulp of t/g give
// RN(q + (t - q g) y) = RN(t/g)), 4 instructions instead of the __fdiv_rn sequence.  Only
// for operands that keep every intermediate normal and finite: the caller checks g, dark and
// coeff (calib_fast_ok); tools/fastdiv_probe.cu compares it with __fdiv_rn bit for bit.
__device__ __forceinline__ float calib_fast(float raw, float dark, float coeff, float gain,
                                            float ginv) {
  // finite operands (calib_fast_range): no NaN to keep, so max(t, 0) is one FMNMX
  const float t = __fmul_rn(fmaxf(__fsub_rn(raw, dark), 0.0f), coeff);
  const float q = __fmul_rn(t, ginv);
  const float r = __fmaf_rn(-q, gain, t);
  return __fmaf_rn(r, ginv, q);
}
// |x| in [2^-60, 2^60] (normal, finite); dark may also be 0
__device__ __forceinline__ bool calib_fast_range(float x) {
  const float a = fabsf(x);
  return a >= 8.6736174e-19f && a <= 1.1529215e18f;
}

__device__ __forceinline__ bool finite_f(float x) { return isfinite(x); }

template <typename T>
__host__ __device__ __forceinline__ T ceil_div(T a, T b) { return (a + b - 1) / b; }

// order-preserving float <-> uint32 map (total order, -0 < +0 collapsed)
__device__ __forceinline__ uint32_t f2ord(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// packed f32x2 arithmetic (FFMA2 / FADD2 on sm_100): two lanes per instruction,
// each lane rounded exactly like the scalar fmaf / __fadd_rn
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 r;
  asm("{\n\t.reg .b64 a, b, c, d;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\tmov.b64 c, {%6, %7};\n\t"
      "fma.rn.f32x2 d, a, b, c;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 a, b, d;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "add.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 a, b, d;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "mul.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 a, b, d;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "sub.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}

// calib_fast on two values at once (f32x2 ops, each lane rounded like the scalar form)
__device__ __forceinline__ float2 calib_fast2(float2 raw, float2 dark, float2 coeff, float gain,
                                              float ginv) {
  float2 t = fsub2(raw, dark);
  t = fmul2(make_float2(fmaxf(t.x, 0.0f), fmaxf(t.y, 0.0f)), coeff);
  const float2 gi2 = make_float2(ginv, ginv);
  const float2 q = fmul2(t, gi2);
  const float2 r = ffma2(make_float2(-q.x, -q.y), make_float2(gain, gain), t);
  return ffma2(r, gi2, q);
}

// moments that must be recomputed: the int8 quantiser overflowed (2), or a value clamped
// at 0 (4) on a raw-byte path that did not correct it (256: clamp_fix_kernel did)
__host__ __device__ __forceinline__ bool flags_range(int32_t f) {
  return (f & 2) || ((f & 4) && !(f & 256));
}

// moments-pass flags word (include/skyrx_b200.h): proven "no raw value below dark"
// either by the raw-byte tensor-core pass (8 without 4) or the general pass (128 without 64)
__device__ __forceinline__ bool flags_noclamp(int32_t f) {
  return (f & 12) == 8 || (f & 192) == 128;
}

// 16-byte vectors for shared-memory operand loads
template <typename T>
struct Vec16;
template <>
struct Vec16<float> {
  using type = float4;
  static constexpr int n = 4;
};
template <>
struct Vec16<double> {
  using type = double2;
  static constexpr int n = 2;
};
__device__ __forceinline__ void unpack(const float4& v, float* o) {
  o[0] = v.x, o[1] = v.y, o[2] = v.z, o[3] = v.w;
}
__device__ __forceinline__ void unpack(const double2& v, double* o) { o[0] = v.x, o[1] = v.y; }

// load 8 consecutive T from 16-B aligned shared memory
template <typename T>
__device__ __forceinline__ void load8(const T* p, T* o) {
  using V = typename Vec16<T>::type;
  constexpr int VN = Vec16<T>::n;
#pragma unroll
  for (int q = 0; q < 8; q += VN) unpack(*reinterpret_cast<const V*>(p + q), o + q);
}

// Warp reductions
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace skyrx
