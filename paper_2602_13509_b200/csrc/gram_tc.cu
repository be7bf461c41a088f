// K2-TC — fused calibrate + background moments on the tensor cores, exact in int32.
//
// Reference: rx.py:56-66 (f64 mean, then f64 Gram of centred pixels).  Here
// every calibrated value is centred by the sample shift c_b and quantised to a
// fixed point D = floor((x - c_b) / q_b + u) with a per-element dither u in [0, 1)
// (unbiased even for lattice-valued data), |D| < 2^22 (q_b a power of two from 4.2x the
// largest sampled deviation).  E = D + 2^22 is split into three unsigned bytes
// E = e2*2^16 + e1*2^8 + e0 (e2 < 128) and the Gram of the digits is accumulated EXACTLY
// in int32 by tcgen05.mma kind::i8 (unsigned; digit products < 2^16, TMEM drained every
// 255 tiles of 128 pixels):
//     G_E = sum_a 2^16a Pa,a + sum_{a>b} 2^8(a+b) (Pa,b + Pa,b^T),  Pa,b = Ea^T Eb
// One constant band (index B, E = 1 on valid pixels) makes the same products carry n and
// sum(E); the reduce removes the offset exactly: G_D = G_E - 2^22 (S_i + S_j) + n 2^44.
// The only approximation left is the quantisation (noise ~q/sqrt(12) per element,
// averaged over the cube).  Values outside the quantiser range (or non-finite) set
// flags |= 2 and the host recomputes that cube with the FFMA kernel.
//
// Per element the workers spend ~12 instructions: raw words as u32 pairs (exact u16 ->
// f32 by the 2^23 trick), calibration with the per-line 1/g as a multiply (the moments
// are not a bit-exact calibration anyway: rx.py's f32 rounding is the reference's own
// ~1e-8), quantisation by the 1.5 * 2^23 magic add (round to nearest of tq + u - 1/2 =
// floor(tq + u)), a Weyl-sequence dither over a per-pixel hash, and byte digits moved
// into the three operand planes with PRMT (no per-digit shifts or masks).
//
// Operands are MN-major (bands contiguous) so each pixel row writes 16-byte
// chunks: smem address of (digit a, band b, pixel p) =
//     (p/8)*LBO + (a*NG + b/16)*128 + (p%8)*16 + b%16,  LBO = 3*NG*128.
// Per 32-pixel K step three MMAs cover the six products:
//     A = E2 (M=128), B = [E0|E1|E2] (N = 3*BPg) -> P20 P21 P22
//     A = E1,         B = [E0|E1]    (N = 2*BPg) -> P10 P11
//     A = E0,         B = E0         (N =   BPg) -> P00          (6*BPg <= 480 TMEM cols)
#include "common.cuh"
#include "tc_common.cuh"
#include "umma.cuh"

namespace skyrx {
using namespace umma;

// worker warps: kGtH threads per pixel row (each a contiguous run of 16-band groups), then the
// TMA and MMA warps.  What bounds the kernel is shared memory, not issue: per 128-pixel tile
// the MMAs read ~108 KB of digit planes, the workers' per-pixel calibration rows ~80 KB, plus
// the plane writes and the raw ring (4 workers per row, 4 operand stages, or 40 % fewer
// instructions, measured: none faster than 3.67 ms per c4 strip, profiles/r02_ablation.md)
#ifndef GTC_H
#define GTC_H 2
#endif
constexpr int kGtH = GTC_H;
constexpr int kGtWorkers = 128 * kGtH;
constexpr int kGtThreads = kGtWorkers + 64;
constexpr int kGtTmaWarp = kGtWorkers / 32, kGtMmaWarp = kGtTmaWarp + 1;
constexpr int kGtRawStages = 3;
constexpr int kGtOpStages = 2;
constexpr int kGtWmax = 32;
constexpr int kGtFlushTiles = 255;  // 255 tiles * 128 px * 255^2 < 2^31
constexpr int kGtOff = 1 << 22;     // E = D + kGtOff >= 0

// idesc for kind::i8 with unsigned 8-bit operands, MN-major A and B, S32 accumulators
__host__ __device__ constexpr uint32_t idesc_gt_u8(int M, int N) {
  return (2u << 4) | (0u << 7) | (0u << 10) | (1u << 15) | (1u << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

struct GramTcParams {
  const uint16_t* raw;
  const float* dark;
  const float* coeff;
  const float* gain;
  const double* shift;   // c_b (f32-representable)
  const float* qinv;     // 2^e_b
  double* part;          // per CTA: Y[BPg*BPg] then X[BPg*BPg], column-major [j][i]
  int32_t* flags;
  TileSched ts;
  int64_t per_cta;
  uint32_t raw_stage_bytes;
};

// KIND: SKYRX_IN_RAW_U16 (calibrate on the fly, the fused path) or SKYRX_IN_F32 (an
// already calibrated radiance cube: compute_stats(mode="fast") on a RadianceCube)
template <int BPG, int KIND = SKYRX_IN_RAW_U16>
__global__ void __launch_bounds__(kGtThreads, 1) gram_tc_kernel(GramTcParams p) {
  constexpr bool kF32 = KIND == SKYRX_IN_F32;
  constexpr uint32_t ESZ = kF32 ? 4u : 2u;  // bytes per band value in the ring
  constexpr int NG = BPG / 16;
  constexpr uint32_t LBO = 3u * NG * 128u;
  // 16 pixel groups (128 px) + pad for the M=128 A reads past the last group
  constexpr uint32_t OP_BYTES = 16u * LBO + 1024u;
  constexpr uint32_t N2 = 3 * BPG, N1 = 2 * BPG, N0 = BPG;
  static_assert(6 * BPG <= 512, "TMEM holds six BPG-wide products");
  extern __shared__ __align__(1024) uint8_t sm[];
  const int B = p.ts.B;
  uint8_t* raw_ring = sm;
  uint8_t* op_ring = raw_ring + kGtRawStages * p.raw_stage_bytes;
  // per (sample of the block, band pair): {c q, -(d c) q} x 2, the quantiser scale folded in
  float4* tab4 = reinterpret_cast<float4*>(op_ring + kGtOpStages * OP_BYTES);  // [Wmax][BPG/2]
  float* cs = reinterpret_cast<float*>(tab4 + kGtWmax * (BPG / 2));  // [BPG] -c_b q_b
  float* qs = cs + BPG;
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(qs + BPG) + 7) & ~uintptr_t(7));
  uint64_t* raw_full = bars;
  uint64_t* raw_empty = raw_full + kGtRawStages;
  uint64_t* op_full = raw_empty + kGtRawStages;
  uint64_t* op_empty = op_full + kGtOpStages;
  uint64_t* acc_full = op_empty + kGtOpStages;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  // balanced contiguous item ranges: every CTA owns >= 1 tile (grid <= items),
  // so every per-CTA partial below is written
  const int64_t it0 = (int64_t)blockIdx.x * p.ts.items / gridDim.x;
  int64_t it1 = (int64_t)(blockIdx.x + 1) * p.ts.items / gridDim.x;
  if (it1 > p.ts.items) it1 = p.ts.items;
  const int n = it0 < it1 ? (int)(it1 - it0) : 0;
  const int nflush = (n + kGtFlushTiles - 1) / kGtFlushTiles;

  if (tid == 0) {
    for (int s = 0; s < kGtRawStages; ++s) mbar_init(&raw_full[s], 1), mbar_init(&raw_empty[s], kGtWorkers);
    for (int s = 0; s < kGtOpStages; ++s) mbar_init(&op_full[s], kGtWorkers), mbar_init(&op_empty[s], 1);
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, kGtWorkers);
    fence_mbar_init();
  }
  if (warp == kGtMmaWarp) tmem_alloc(tmem_slot, 512);
  for (int b = tid; b < BPG; b += blockDim.x) {
    // tq = (x - c_b) q_b as one FFMA: x q_b - c_b q_b (q_b a power of two: exact scaling)
    cs[b] = b < B ? -((float)p.shift[b] * p.qinv[b]) : 0.0f;
    qs[b] = b < B ? p.qinv[b] : 0.0f;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kGtTmaWarp) {
    if ((tid & 31) == 0) {  // ------------------------------------------- TMA producer
      for (int t = 0; t < n; ++t) {
        const int s = t % kGtRawStages;
        mbar_wait(&raw_empty[s], ((t / kGtRawStages) & 1) ^ 1);
        const TileInfo ti = tile_info(p.ts, it0 + t);
        const uint32_t seg = (uint32_t)ti.w * B * ESZ;
        mbar_arrive_expect_tx(&raw_full[s], seg * (uint32_t)ti.nlines);
        uint8_t* dst = raw_ring + s * p.raw_stage_bytes;
        for (int li = 0; li < ti.nlines; ++li) {
          const uint8_t* src = reinterpret_cast<const uint8_t*>(p.raw) +
                               ((ti.line0 + li) * (int64_t)p.ts.S + ti.s0) * B * ESZ;
          bulk_g2s(dst + li * seg, src, seg, &raw_full[s]);
        }
      }
    }
  } else if (warp == kGtMmaWarp) {
    {  // --------------------------------- MMA issuer (whole warp, one elected lane issues)
      constexpr uint32_t id2 = idesc_gt_u8(128, N2);
      constexpr uint32_t id1 = idesc_gt_u8(128, N1);
      constexpr uint32_t id0 = idesc_gt_u8(128, N0);
      for (int t = 0; t < n; ++t) {
        const int os = t % kGtOpStages;
        const bool first = (t % kGtFlushTiles) == 0;
        if (first && t > 0) mbar_wait(acc_empty, ((t / kGtFlushTiles) - 1) & 1);
        mbar_wait(&op_full[os], (t / kGtOpStages) & 1);
        tc_fence_after();
        const uint8_t* base = op_ring + os * OP_BYTES;
        if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {  // 4 x 32 pixels
          const uint8_t* kb = base + ks * 4 * LBO;
          const uint32_t acc = (first && ks == 0) ? 0u : 1u;
          const uint64_t b = smem_desc(kb, LBO, 128);
          mma_i8(tmem + 0, smem_desc(kb + 2 * NG * 128, LBO, 128), b, id2, acc);
          mma_i8(tmem + N2, smem_desc(kb + NG * 128, LBO, 128), b, id1, acc);
          mma_i8(tmem + N2 + N1, smem_desc(kb, LBO, 128), b, id0, acc);
        }
        mma_commit(&op_empty[os]);
        if ((t % kGtFlushTiles) == kGtFlushTiles - 1 || t == n - 1) mma_commit(acc_full);
        }
        __syncwarp();
      }
    }
  } else {  // ------------------------------------------------------------ workers
    const int r = tid & 127;          // pixel row
    const int h = tid >> 7;           // which band groups this thread packs
    const int g_lo = h * NG / kGtH, g_hi = (h + 1) * NG / kGtH;  // this thread's groups
    int cur_block = -1;
    bool range_ok = true;
    int flushes = 0;
    auto flush = [&]() {
      mbar_wait(acc_full, flushes & 1);
      tc_fence_after();
      // warp w reads TMEM lanes 32*(w%4).., columns split by h
      const int lane_row = 32 * (warp & 3) + (tid & 31);  // band row i
      const uint32_t tl = warp_uniform(tmem + ((uint32_t)(32 * (warp & 3)) << 16));
      double* Y = p.part + (size_t)blockIdx.x * 2 * BPG * BPG;
      double* X = Y + BPG * BPG;
      for (int jc = h; jc < NG; jc += kGtH) {
#pragma unroll 1
        for (int hc = 0; hc < 2; ++hc) {  // 8 columns at a time (registers)
          const uint32_t col = jc * 16 + hc * 8;
          uint32_t p20[8], p21[8], p22[8], p10[8], p11[8], p00[8];
          tmem_ld8(tl + 0 * BPG + col, p20);
          tmem_ld8(tl + 1 * BPG + col, p21);
          tmem_ld8(tl + 2 * BPG + col, p22);
          tmem_ld8(tl + N2 + 0 * BPG + col, p10);
          tmem_ld8(tl + N2 + 1 * BPG + col, p11);
          tmem_ld8(tl + N2 + N1 + col, p00);
          tmem_ld_wait();
          if (lane_row < BPG) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int j = (int)col + q;
              const double y = 4294967296.0 * (double)(int32_t)p22[q] +
                               65536.0 * (double)(int32_t)p11[q] + (double)(int32_t)p00[q];
              const double x = 16777216.0 * (double)(int32_t)p21[q] +
                               65536.0 * (double)(int32_t)p20[q] + 256.0 * (double)(int32_t)p10[q];
              const size_t o = (size_t)j * BPG + lane_row;
              if (flushes == 0) {
                Y[o] = y;
                X[o] = x;
              } else {
                Y[o] += y;
                X[o] += x;
              }
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(acc_empty);
      ++flushes;
    };
    for (int t = 0; t < n; ++t) {
      const TileInfo ti = tile_info(p.ts, it0 + t);
      if (!kF32 && ti.block != cur_block) {
        asm volatile("bar.sync 1, %0;" ::"n"(kGtWorkers) : "memory");
        for (int e = tid; e < ti.w * (BPG / 2); e += kGtWorkers) {
          const int j = e / (BPG / 2), pr = e - j * (BPG / 2);
          float v[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int b = 2 * pr + h;
            if (b < B) {
              const int64_t g = (int64_t)(ti.s0 + j) * B + b;
              const float c = __ldg(p.coeff + g);
              v[2 * h] = c * qs[b];
              v[2 * h + 1] = -(__fmul_rn(__ldg(p.dark + g), c) * qs[b]);  // -(d c) q
            }
          }
          tab4[e] = make_float4(v[0], v[1], v[2], v[3]);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kGtWorkers) : "memory");
        cur_block = ti.block;
      }
      const int s = t % kGtRawStages;
      const int os = t % kGtOpStages;
      mbar_wait(&raw_full[s], (t / kGtRawStages) & 1);
      mbar_wait(&op_empty[os], ((t / kGtOpStages) & 1) ^ 1);
      const bool valid = r < ti.rows;
      int j = 0;
      float gi = 1.0f;
      uint32_t pixkey = 0;
      if (valid) {
        const int li = r / ti.w;
        j = r - li * ti.w;
        if (!kF32) gi = 1.0f / __ldg(p.gain + ti.line0 + li);
        const uint64_t pix = (uint64_t)(ti.line0 + li) * (uint64_t)p.ts.S + (uint64_t)(ti.s0 + j);
        pixkey = (uint32_t)(pix * 0x9E3779B97F4A7C15ull >> 32) * 0x85EBCA6Bu;
      }
      const uint8_t* rowb = raw_ring + s * p.raw_stage_bytes + (size_t)r * B * ESZ;
      const float4* tj = tab4 + j * (BPG / 2);
      uint8_t* ob = op_ring + os * OP_BYTES + (uint32_t)(r >> 3) * LBO + (uint32_t)(r & 7) * 16u;
      // band k's value -> E = D + 2^22 (as a u32), D = floor(tq + u)
      // x: the calibrated value already in quantiser units (RAW) or the radiance (F32)
      auto quant = [&](float x, int k) -> uint32_t {
        const float tq = kF32 ? __fmaf_rn(x, qs[k], cs[k]) : __fmaf_rn(x, gi, cs[k]);
        // dither: Weyl step over the band on a per-pixel hash, u - 1/2 in [-1/2, 1/2)
        const uint32_t h = pixkey + (uint32_t)k * 0x9E3779B9u;
        const float um = __uint_as_float(0x3F800000u | (h >> 9)) - 1.5f;
        const float sv = __fadd_rn(tq, um);
        range_ok &= fabsf(sv) < 4190000.0f;  // |D| < 2^22 (and false for NaN)
        // RN(sv + 1.5 * 2^23) has ulp 1: its low mantissa bits are RN(sv) = floor(tq + u)
        const float t = __fadd_rn(sv, 12582912.0f);
        return (uint32_t)(__float_as_int(t) - 0x4B400000 + kGtOff);
      };
      for (int gq = g_lo; gq < g_hi; ++gq) {
        uint32_t w0[4], w1[4], w2[4];
        if (!kF32 && (B & 1) == 0 && valid && gq * 16 + 16 <= B) {
          // a full group of 16 bands: no per-element conditions, band pairs in f32x2
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint32_t e[4];
#pragma unroll
            for (int q = 0; q < 4; q += 2) {
              const int k = gq * 16 + q4 * 4 + q;
              const uint32_t v = *reinterpret_cast<const uint32_t*>(rowb + 2 * k);
              const float2 rf = fadd2(make_float2(__uint_as_float(__byte_perm(v, 0x4B000000u, 0x7610)),
                                                  __uint_as_float(__byte_perm(v, 0x4B000000u, 0x7632))),
                                      make_float2(-8388608.0f, -8388608.0f));
              const float4 tb4 = tj[k >> 1];
              const float2 c2 = *reinterpret_cast<const float2*>(cs + k);
              float2 x = ffma2(rf, make_float2(tb4.x, tb4.z), make_float2(tb4.y, tb4.w));
              x.x = x.x < 0.0f ? 0.0f : x.x;  // keeps NaN
              x.y = x.y < 0.0f ? 0.0f : x.y;
              const float2 tq = ffma2(x, make_float2(gi, gi), c2);
              const uint32_t h0 = pixkey + (uint32_t)k * 0x9E3779B9u, h1 = h0 + 0x9E3779B9u;
              const float2 sv = fadd2(tq, fadd2(make_float2(__uint_as_float(0x3F800000u | (h0 >> 9)),
                                                            __uint_as_float(0x3F800000u | (h1 >> 9))),
                                                make_float2(-1.5f, -1.5f)));
              range_ok &= fabsf(sv.x) < 4190000.0f && fabsf(sv.y) < 4190000.0f;
              const float2 tt = fadd2(sv, make_float2(12582912.0f, 12582912.0f));
              e[q] = (uint32_t)(__float_as_int(tt.x) - 0x4B400000 + kGtOff);
              e[q + 1] = (uint32_t)(__float_as_int(tt.y) - 0x4B400000 + kGtOff);
            }
            const uint32_t p01 = __byte_perm(e[0], e[1], 0x5140);
            const uint32_t p23 = __byte_perm(e[2], e[3], 0x5140);
            w0[q4] = __byte_perm(p01, p23, 0x5410);
            w1[q4] = __byte_perm(p01, p23, 0x7632);
            w2[q4] = __byte_perm(__byte_perm(e[0], e[1], 0x0062), __byte_perm(e[2], e[3], 0x0062), 0x5410);
          }
        } else {
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          uint32_t e[4];
#pragma unroll
          for (int q = 0; q < 4; q += 2) {
            const int k = gq * 16 + q4 * 4 + q;
            float xa = 0.0f, xb = 0.0f;
            bool ina = valid && k < B, inb = valid && k + 1 < B;
            if constexpr (kF32) {
              const float* fp = reinterpret_cast<const float*>(rowb);
              if (ina) xa = fp[k];
              if (inb) xb = fp[k + 1];
            } else {
              float ra, rb;
              if ((B & 1) == 0 && inb) {  // one u32 = bands k, k+1 (rows are 4-byte aligned)
                const uint32_t v = *reinterpret_cast<const uint32_t*>(rowb + 2 * k);
                ra = __uint_as_float(__byte_perm(v, 0x4B000000u, 0x7610)) - 8388608.0f;
                rb = __uint_as_float(__byte_perm(v, 0x4B000000u, 0x7632)) - 8388608.0f;
              } else {
                const uint16_t* rp = reinterpret_cast<const uint16_t*>(rowb);
                ra = ina ? (float)rp[k] : 0.0f;
                rb = inb ? (float)rp[k + 1] : 0.0f;
              }
              // max(., 0) that keeps NaN (np.maximum, calibrate.py:99): a NaN dark or coeff
              // must reach the range check below (flags |= 2 -> the f64 redo reports it)
              const float4 tb4 = tj[k >> 1];  // k even
              if (ina) {
                const float ta = __fmaf_rn(ra, tb4.x, tb4.y);
                xa = ta < 0.0f ? 0.0f : ta;
              }
              if (inb) {
                const float tb = __fmaf_rn(rb, tb4.z, tb4.w);
                xb = tb < 0.0f ? 0.0f : tb;
              }
            }
            // padding bands (k >= B, not the constant band) quantise to E = 2^22 with
            // q_b = c_b = 0: they only add the known offset, removed with the others
            e[q] = ina ? quant(xa, k) : (valid && k == B ? 1u : (uint32_t)kGtOff);
            e[q + 1] = inb ? quant(xb, k + 1) : (valid && k + 1 == B ? 1u : (uint32_t)kGtOff);
            if (!valid) e[q] = e[q + 1] = 0u;
          }
          // bytes 0, 1, 2 of the four E words -> the three digit planes
          const uint32_t p01 = __byte_perm(e[0], e[1], 0x5140);
          const uint32_t p23 = __byte_perm(e[2], e[3], 0x5140);
          w0[q4] = __byte_perm(p01, p23, 0x5410);
          w1[q4] = __byte_perm(p01, p23, 0x7632);
          w2[q4] = __byte_perm(__byte_perm(e[0], e[1], 0x0062), __byte_perm(e[2], e[3], 0x0062), 0x5410);
        }
        }
        *reinterpret_cast<uint4*>(ob + (0 * NG + gq) * 128) = make_uint4(w0[0], w0[1], w0[2], w0[3]);
        *reinterpret_cast<uint4*>(ob + (1 * NG + gq) * 128) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
        *reinterpret_cast<uint4*>(ob + (2 * NG + gq) * 128) = make_uint4(w2[0], w2[1], w2[2], w2[3]);
      }
      fence_async_smem();
      mbar_arrive(&op_full[os]);
      mbar_arrive(&raw_empty[s]);
      if ((t % kGtFlushTiles) == kGtFlushTiles - 1 && t != n - 1) flush();
    }
    if (n > 0) flush();
    if (!range_ok) atomicOr(p.flags, 2);  // incl. non-finite values: the f64 redo reports them
  }
  (void)nflush;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kGtMmaWarp) tmem_dealloc(tmem, 512);
}

// Gram (units) = sum over CTAs of Y + X + X^T, then scale to moments [n, s, Q]
template <int BPG>
__global__ void gram_tc_reduce_kernel(const double* __restrict__ part, int nparts, int B,
                                      const float* __restrict__ qinv, double* __restrict__ moments) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;  // e = i * BPG + j
  if (e >= BPG * BPG) return;
  const int i = e / BPG, j = e - i * BPG;
  if (i > B || j > B || j > i) return;  // lower triangle incl. the constant band B
  // G_E(a, b), a >= b: the digit Gram of E = D + 2^22 (constant band B: E = 1)
  auto G = [&](int a, int b) {
    double v = 0.0;
    for (int c = 0; c < nparts; ++c) {
      const double* Y = part + (size_t)c * 2 * BPG * BPG;
      const double* X = Y + BPG * BPG;
      v += Y[(size_t)b * BPG + a] + X[(size_t)b * BPG + a] + X[(size_t)a * BPG + b];
    }
    return v;
  };
  constexpr double off = (double)kGtOff;
  const double n = G(B, B);  // pixel count (exact)
  double* s_out = moments + 1;
  double* q_out = moments + 1 + B;
  const double qi = i < B ? 1.0 / (double)qinv[i] : 1.0;
  const double qj = j < B ? 1.0 / (double)qinv[j] : 1.0;
  if (i == B && j == B) {
    moments[0] = n;
  } else if (i == B) {
    s_out[j] = (G(B, j) - n * off) * qj;  // sum over pixels of (x_j - c_j), quantised
  } else {
    const double v = G(i, j) - off * (G(B, i) + G(B, j)) + n * off * off;
    q_out[(size_t)i * B + j] = v * qi * qj;
    q_out[(size_t)j * B + i] = v * qi * qj;
  }
}

// c_b = f32(mean of a strided sample), q_b from 8x the largest sampled deviation
template <int KIND>
__global__ void quant_shift_kernel(const void* pixels, int64_t npix, int32_t samples, int32_t B,
                                   const float* dark, const float* coeff, const float* gain,
                                   double* shift, float* qinv) {
  // one CTA per band (grid = B), 256 threads over the sample, fixed-order reductions
  __shared__ double part[8];
  __shared__ float partf[8];
  __shared__ float c_sh;
  const int64_t step = npix > 4096 ? npix / 4096 : 1;
  const int64_t m = npix > 0 ? (npix + step - 1) / step : 0;
  const int b = blockIdx.x;
  auto val = [&](int64_t i) {
    const int64_t pix = i * step;
    const int64_t gi = pix * B + b;
    if constexpr (KIND == SKYRX_IN_RAW_U16) {
      const int64_t line = pix / samples;
      const int64_t tb = (pix - line * samples) * B + b;
      return calib((float)reinterpret_cast<const uint16_t*>(pixels)[gi], dark[tb], coeff[tb],
                   gain[line]);
    } else {
      return reinterpret_cast<const float*>(pixels)[gi];
    }
  };
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) acc += (double)val(i);
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += part[w];
    c_sh = m > 0 ? (float)(s / (double)m) : 0.0f;
  }
  __syncthreads();
  const float c = c_sh;
  float amax = 0.0f;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x)
    amax = fmaxf(amax, fabsf(__fsub_rn(val(i), c)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if ((threadIdx.x & 31) == 0) partf[threadIdx.x >> 5] = amax;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 0; w < 8; ++w) amax = fmaxf(amax, partf[w]);
    const float bound = fmaxf(4.2f * amax, 1e-30f);
    int e = 0;
    frexpf(bound, &e);                 // bound < 2^e
    int ex = 22 - e;                   // |x - c| <= 4 amax  =>  |D| < 2^22 * 4/4.2
    ex = ex > 120 ? 120 : (ex < -120 ? -120 : ex);
    shift[b] = (double)c;
    qinv[b] = ldexpf(1.0f, ex);
  }
}

static int bpg_for(int B) { return ((B + 1 + 15) / 16) * 16; }

template <int BPG, int KIND = SKYRX_IN_RAW_U16>
static int launch_gram_tc(GramTcParams p, double* moments, cudaStream_t st) {
  constexpr uint32_t ESZ = KIND == SKYRX_IN_F32 ? 4u : 2u;
  p.raw_stage_bytes = (uint32_t)(((128u * p.ts.B * ESZ) + 127u) & ~127u);
  constexpr uint32_t LBO = 3u * (BPG / 16) * 128u;
  const size_t smem = kGtRawStages * (size_t)p.raw_stage_bytes + kGtOpStages * (16u * LBO + 1024u) +
                      (size_t)kGtWmax * (BPG / 2) * 16 + 2 * BPG * 4 + 16 * 8 + 64;
  int grid = kSMs;
  if (p.ts.items < grid) grid = (int)p.ts.items;
  if (grid < 1) grid = 1;
  p.per_cta = (p.ts.items + grid - 1) / grid;
  cudaFuncSetAttribute(gram_tc_kernel<BPG, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  gram_tc_kernel<BPG, KIND><<<grid, kGtThreads, smem, st>>>(p);
  SKYRX_CHECK_LAUNCH("gram_tc_kernel");
  gram_tc_reduce_kernel<BPG><<<ceil_div(BPG * BPG, 256), 256, 0, st>>>(p.part, grid, p.ts.B, p.qinv,
                                                                        moments);
  SKYRX_CHECK_LAUNCH("gram_tc_reduce_kernel");
  return SKYRX_OK;
}

}  // namespace skyrx

using namespace skyrx;

extern "C" int skyrx_stats_tc_supported(int64_t lines, int32_t samples, int32_t bands,
                                        const void* raw) {
  TileSched ts;
  if (bands < 1 || bands > 79) return 0;
  if (((uintptr_t)raw & 15) != 0) return 0;
  return tc_sched(lines, samples, bands, kGtWmax, ts) ? 1 : 0;
}

extern "C" size_t skyrx_stats_tc_workspace(int32_t bands) {
  const size_t bpg = (size_t)bpg_for(bands);
  return (size_t)kSMs * 2 * bpg * bpg * sizeof(double) + 256 * sizeof(float);
}

extern "C" int skyrx_quant_shift(int32_t kind, const void* pixels, int64_t lines, int32_t samples,
                                 int32_t bands, const float* dark, const float* coeff,
                                 const float* gain, double* shift, float* qinv, void* stream) {
  SKYRX_REQUIRE(bands > 0 && lines >= 0 && samples >= 0, "bad cube shape");
  const int64_t npix = lines * (int64_t)samples;
  if (kind == SKYRX_IN_RAW_U16)
    quant_shift_kernel<SKYRX_IN_RAW_U16><<<bands, 256, 0, as_stream(stream)>>>(
        pixels, npix, samples, bands, dark, coeff, gain, shift, qinv);
  else
    quant_shift_kernel<SKYRX_IN_F32><<<bands, 256, 0, as_stream(stream)>>>(
        pixels, npix, samples, bands, dark, coeff, gain, shift, qinv);
  SKYRX_CHECK_LAUNCH("skyrx_quant_shift");
  return SKYRX_OK;
}

extern "C" int skyrx_stats_tc(const uint16_t* raw, int64_t lines, int32_t samples, int32_t bands,
                              const float* dark, const float* coeff, const float* gain,
                              const double* shift, const float* qinv, double* moments,
                              int32_t* flags, void* workspace, size_t workspace_bytes,
                              void* stream) {
  SKYRX_REQUIRE(skyrx_stats_tc_supported(lines, samples, bands, raw),
                "tensor-core moments path unsupported for this shape/alignment");
  SKYRX_REQUIRE(workspace_bytes >= skyrx_stats_tc_workspace(bands), "workspace too small");
  GramTcParams p{};
  p.raw = raw;
  p.dark = dark;
  p.coeff = coeff;
  p.gain = gain;
  p.shift = shift;
  p.qinv = qinv;
  p.part = reinterpret_cast<double*>(workspace);
  p.flags = flags;
  tc_sched(lines, samples, bands, kGtWmax, p.ts);
  cudaStream_t st = as_stream(stream);
  switch (bpg_for(bands)) {
    case 16: return launch_gram_tc<16>(p, moments, st);
    case 32: return launch_gram_tc<32>(p, moments, st);
    case 48: return launch_gram_tc<48>(p, moments, st);
    case 64: return launch_gram_tc<64>(p, moments, st);
    case 80: return launch_gram_tc<80>(p, moments, st);
  }
  set_error("unsupported band count %d", bands);
  return SKYRX_ERR_ARG;
}

// compute_stats(mode="fast") on an f32 radiance cube (rx.py:42-66 on a RadianceCube): the
// same quantised-digit tensor-core Gram, the values read as they are.  shift / qinv from
// skyrx_quant_shift(SKYRX_IN_F32, ...).
extern "C" int skyrx_stats_tc_f32(const float* pixels, int64_t lines, int32_t samples,
                                  int32_t bands, const double* shift, const float* qinv,
                                  double* moments, int32_t* flags, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  SKYRX_REQUIRE(skyrx_stats_tc_supported(lines, samples, bands, pixels),
                "tensor-core moments path unsupported for this shape/alignment");
  SKYRX_REQUIRE(workspace_bytes >= skyrx_stats_tc_workspace(bands), "workspace too small");
  SKYRX_REQUIRE(((int64_t)samples * bands * 4) % 16 == 0, "f32 lines must be 16-byte multiples");
  GramTcParams p{};
  p.raw = reinterpret_cast<const uint16_t*>(pixels);  // byte address; the kernel reads f32
  p.shift = shift;
  p.qinv = qinv;
  p.part = reinterpret_cast<double*>(workspace);
  p.flags = flags;
  tc_sched(lines, samples, bands, kGtWmax, p.ts);
  cudaStream_t st = as_stream(stream);
  switch (bpg_for(bands)) {
    case 16: return launch_gram_tc<16, SKYRX_IN_F32>(p, moments, st);
    case 32: return launch_gram_tc<32, SKYRX_IN_F32>(p, moments, st);
    case 48: return launch_gram_tc<48, SKYRX_IN_F32>(p, moments, st);
    case 64: return launch_gram_tc<64, SKYRX_IN_F32>(p, moments, st);
    case 80: return launch_gram_tc<80, SKYRX_IN_F32>(p, moments, st);
  }
  set_error("unsupported band count %d", bands);
  return SKYRX_ERR_ARG;
}
