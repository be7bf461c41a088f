// K4-TC — fused calibrate + RX score on the 5th-gen tensor cores (tcgen05).
//
// delta(p) = sum_j z_pj^2,  z = D W^T,  D = x - mu (128 pixels x KP bands),
// W = L^-1 (KP x KP, lower).  Precision: D and W are
// split into f16 hi + lo (W per output row scaled by a power of two so lo
// stays normal); z accumulates Dhi*Whi + Dhi*Wlo + Dlo*Whi in the f32 TMEM
// accumulator (which truncates, tools/umma_probe.cu); emulated worst-case
// score error 1.6e-6 against the f64 reference (tolerance 1e-4), measured
// 1.4e-6 on B200 (tools/debug_score.py).
//
// Warp roles (persistent CTA, one per SM, 448 threads):
//   warp 12      TMA producer : raw line segments of each tile -> smem ring (cp.async.bulk)
//   warp 13      MMA issuer   : 3*KP/16 tcgen05.mma per tile into a 3-deep TMEM
//                               accumulator ring (128 lanes = pixels, KP columns)
//   warps 0-7    transform    : two threads per pixel row (each half of the bands):
//                               calibrate + centre + f16 split into the K-major A operand
//   warps 8-11   epilogue     : tcgen05.ld, sum of squares (FFMA2), unscale, store, max
// Tiles are 128 pixels (one line x 128 samples) dealt round-robin to the CTAs.
// Each worker keeps its row's per-sample calibration constants in registers.
#include <cuda_fp16.h>

#include <type_traits>

#include "common.cuh"
#include "tc_common.cuh"
#include "tma.cuh"
#include "umma.cuh"

namespace skyrx {
using namespace umma;

// Warp roles (persistent CTA, one per SM):
//   warps 0..4G-1  transform : G threads per pixel row, each owning a contiguous
//                              run of the row's 8-band chunks (G = 3 for KP >= 48)
//   next 4 warps   epilogue  : one thread per pixel row (TMEM lane quarter = warp % 4)
//   last 2 warps   TMA producer, MMA issuer (one elected lane each)
__host__ __device__ constexpr int sc_groups(int kp) { return kp >= 48 ? 3 : 2; }
__host__ __device__ constexpr int sc_threads(int kp) { return 128 * sc_groups(kp) + 128 + 64; }
// registers per thread such that the busiest SM sub-partition (ceil(warps / 4)
// warps) fits its 16K-register file
__host__ __device__ constexpr int sc_maxreg(int kp) {
  return (16384 / (32 * ((sc_threads(kp) / 32 + 3) / 4))) / 8 * 8;
}
constexpr int kTcEpilogue = 128;
constexpr int kScoreRawStagesMax = 8;
constexpr int kScoreAStages = 2;
// NCAT: the two products that read D_hi run as ONE MMA against B = [W_hi | W_lo]
// (N = 2 KP - 16 ks): each accumulator holds z_hi-part (columns [0, KP)) and the
// D_hi W_lo part (columns [KP, 2 KP)), summed by the epilogue.  10 instead of 15
// MMAs per tile: every tcgen05.mma re-reads its 4 KB A slice from TMEM, and those
// reads bound the tensor side (profiles/r01_ablation.md).
#ifndef SCX_NO_NCAT
constexpr bool kScoreNcat = true;
constexpr int kScoreAcc = 2;      // TMEM accumulator ring: columns [0, 2 * 2 KP)
constexpr int kScoreABase = 320;  // A ring (f16 hi/lo, from the transform warps): [320, 320 + 2 KP)
#else
constexpr bool kScoreNcat = false;
constexpr int kScoreAcc = 3;      // TMEM accumulator ring: columns [0, 3 KP)
constexpr int kScoreABase = 256;  // A ring (f16 hi/lo, from the transform warps): [256, 256 + 2 KP)
#endif
constexpr int kScoreWmax = 128;
constexpr int kTopkBins = 2048;  // digit 0 of the top-k radix select (select.cu)

// -DSKYRX_SC_PROFILE builds accumulate per-CTA wait cycles of each role
// (tools/sc_profile.py reads them through skyrx_sc_profile); compiled out otherwise
#ifdef SKYRX_SC_PROFILE
__device__ unsigned long long sc_prof[160][10];
#define SC_PW(idx, ...)                                                   \
  do {                                                                    \
    const unsigned long long t0_ = clock64();                             \
    __VA_ARGS__;                                                          \
    if ((threadIdx.x & 31) == 0) atomicAdd(&sc_prof[blockIdx.x][idx], clock64() - t0_); \
  } while (0)
#else
#define SC_PW(idx, ...) __VA_ARGS__
#endif

struct ScoreTcParams {
  const uint16_t* raw;
  const float* dark;
  const float* coeff;
  const float* gain;
  const float* mu_hilo;
  const uint8_t* wpack;
  float* scores;
  uint32_t* max_key;
  uint32_t* hist0;       // nullable: + digit-0 (top 11 key bits) histogram of the scores
  const int32_t* flags;  // moments-pass flags: (flags & 12) == 8 -> no value below dark
  TileSched ts;
  CtaPlan plan;  // block-pinned schedule (tc_common.cuh)
  uint32_t raw_stage_bytes;
  int map_last;  // 1: multi-line tiles (last, narrow block) come in ONE 2-D TMA (tmap)
  int nraw;   // raw ring depth (as many stages as shared memory allows, <= kScoreRawStagesMax)
};

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__host__ __device__ constexpr uint32_t wpack_bytes_for(int kp) {
  return 2u * kp * kp * 2u + kp * 4u;
}

// 8 centred values -> f16 hi (round to nearest) + f16 lo (the exact f32 residual,
// rounded), written to this thread's TMEM lane: 4 columns of hi, 4 of lo
__device__ __forceinline__ void store_split8(const float2 (&dv)[4], uint32_t thi, uint32_t tlo) {
  uint32_t hw[4], lw[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const __half2 h = __floats2half2_rn(dv[q].x, dv[q].y);
    const float2 res = fsub2(dv[q], __half22float2(h));
    const __half2 l = __floats2half2_rn(res.x, res.y);
    hw[q] = *reinterpret_cast<const uint32_t*>(&h);
    lw[q] = *reinterpret_cast<const uint32_t*>(&l);
  }
  tmem_st4(thi, hw[0], hw[1], hw[2], hw[3]);
  tmem_st4(tlo, lw[0], lw[1], lw[2], lw[3]);
}

// MODE 0 with exactly CHT chunks per thread, batched: every raw word of the row
// is loaded first, then all the arithmetic (12 independent band-pair chains at
// CHT = 3 instead of 4 between two tcgen05.st), then all the TMEM stores.  The
// tcgen05.st asm is a compiler barrier, so the chunk-by-chunk form serialises
// each chunk's dependency chain (profiles/r01_ablation.md: the transform warps
// were latency-bound at ~0.45 issue/cycle).
template <int CHT>
__device__ __forceinline__ void transform_row_batched(uint32_t rr32, const float2 (&tco)[CHT * 4],
                                                      const float2 (&tnof)[CHT * 4], uint32_t thi,
                                                      uint32_t tlo) {
  const float2 bias = make_float2(-8388608.0f, -8388608.0f);
  uint32_t wv[CHT * 4];
#pragma unroll
  for (int i = 0; i < CHT * 4; ++i) wv[i] = ld_shared_u32(rr32 + 4 * i);
  uint32_t hw[CHT * 4], lw[CHT * 4];
#pragma unroll
  for (int i = 0; i < CHT * 4; ++i) {
    const uint32_t v = wv[i];
    const float2 rf = fadd2(make_float2(__uint_as_float(__byte_perm(v, 0x4B000000u, 0x7610)),
                                        __uint_as_float(__byte_perm(v, 0x4B000000u, 0x7632))),
                            bias);
    const float2 d = ffma2(rf, tco[i], tnof[i]);
    const __half2 h = __floats2half2_rn(d.x, d.y);
    const float2 res = fsub2(d, __half22float2(h));
    const __half2 l = __floats2half2_rn(res.x, res.y);
    hw[i] = *reinterpret_cast<const uint32_t*>(&h);
    lw[i] = *reinterpret_cast<const uint32_t*>(&l);
  }
#pragma unroll
  for (int cc = 0; cc < CHT; ++cc) {
    tmem_st4(thi + 4 * cc, hw[4 * cc], hw[4 * cc + 1], hw[4 * cc + 2], hw[4 * cc + 3]);
    tmem_st4(tlo + 4 * cc, lw[4 * cc], lw[4 * cc + 1], lw[4 * cc + 2], lw[4 * cc + 3]);
  }
}

// One pixel row's share (CHT 8-band chunks) of the A operand.  Per band pair
// (tco = coeff, tnof = -(dark*coeff + mu) in registers, nm = -mu broadcast):
//   MODE 0: gain 1, no value below dark  d = fma(r, c, nof)
//   MODE 1: gain 1, clamp                d = max(fma(r, c, nof), -mu)
//   MODE 2: per-line gain g              d = max(r c - dark c, 0) / g - mu
//   MODE 3: odd B (2-byte aligned rows), general formula
template <int MODE, int CHT>
__device__ __forceinline__ void transform_row(const uint8_t* rr, uint32_t rr32,
                                              const float2 (&tco)[CHT * 4],
                                              const float2 (&tnof)[CHT * 4], const float2* nm,
                                              float g, uint32_t thi, uint32_t tlo, int cnt) {
  const float gi = 1.0f / g;
  const float2 bias = make_float2(-8388608.0f, -8388608.0f);
#pragma unroll
  for (int cc = 0; cc < CHT; ++cc) {
    if (cc >= cnt) break;  // warp-uniform
    float2 rf[4];
    if (MODE != 3) {  // 4-byte aligned rows: two counts per LDS.32
      uint32_t wv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) wv[q] = ld_shared_u32(rr32 + 16 * cc + 4 * q);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t v = wv[q];
        // exact u16 -> f32 on the ALU pipes: (2^23 + r) - 2^23
        rf[q] = fadd2(make_float2(__uint_as_float(__byte_perm(v, 0x4B000000u, 0x7610)),
                                  __uint_as_float(__byte_perm(v, 0x4B000000u, 0x7632))),
                      bias);
      }
    } else {
      const uint16_t* r16 = reinterpret_cast<const uint16_t*>(rr) + 8 * cc;
#pragma unroll
      for (int q = 0; q < 4; ++q) rf[q] = make_float2((float)r16[2 * q], (float)r16[2 * q + 1]);
    }
    float2 dv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 co = tco[cc * 4 + q], nof = tnof[cc * 4 + q];
      if (MODE == 0) {
        dv[q] = ffma2(rf[q], co, nof);
      } else if (MODE == 1) {
        const float2 d = ffma2(rf[q], co, nof);
        dv[q] = make_float2(fmaxf(d.x, nm[8 * cc + 2 * q].x), fmaxf(d.y, nm[8 * cc + 2 * q + 1].x));
      } else {
        const float m0 = nm[8 * cc + 2 * q].x, m1 = nm[8 * cc + 2 * q + 1].x;
        const float2 d = ffma2(rf[q], co, make_float2(nof.x - m0, nof.y - m1));
        dv[q] = ffma2(make_float2(fmaxf(d.x, 0.0f), fmaxf(d.y, 0.0f)), make_float2(gi, gi),
                      make_float2(m0, m1));
      }
    }
    store_split8(dv, thi + cc * 4, tlo + cc * 4);
  }
}

// Transform warps: calibrate + centre + f16-split every tile of this CTA into
// the A ring.  MODE is uniform over the launch (see transform_row).
template <int KP, int MODE, int CHT, bool BATCHED = false>
__device__ __forceinline__ void transform_loop(const ScoreTcParams& p, int n, int blk, int64_t g0,
                                               int64_t gstep, uint8_t* raw_ring, uint32_t tmem,
                                               const float2* mu, uint64_t* raw_full,
                                               uint64_t* raw_empty, uint64_t* a_full,
                                               uint64_t* a_empty) {
  constexpr int NCH = KP / 8;
  constexpr int NG = sc_groups(KP);  // CHT = chunks per thread (compile time)
  const int tid = threadIdx.x;
  const int r = tid & 127;  // pixel row of the tile
  const int h = tid >> 7;   // band group
  const int lane = tid & 31;
  const int B = p.ts.B;
  // real chunks only (8*c < B); the all-padding chunks of A are zeroed once
  const int nchr = (B + 7) / 8;
  const int cpg = (nchr + NG - 1) / NG;
  const int c_lo = cpg * h;
  const int cnt = min(cpg, nchr - c_lo);
  const int NR = p.nraw;
  // this row's calibration in registers; a tile row maps to the same sample of
  // the current block on every tile, so the tables change only with the block
  float2 tco[CHT * 4], tnof[CHT * 4];
  auto load_row_tables = [&](const TileInfo& tb) {
    const int64_t srow = (int64_t)(tb.s0 + r % tb.w) * B;
#pragma unroll
    for (int cc = 0; cc < CHT; ++cc)
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int k = 8 * (c_lo + cc) + q;
        float co = 0.0f, nof = 0.0f;
        if (k < B) {
          const double mu_k = (double)p.mu_hilo[k] + (double)p.mu_hilo[B + k];
          co = __ldg(p.coeff + srow + k);
          nof = -(float)((double)__ldg(p.dark + srow + k) * (double)co + mu_k);
        }
        float* c2 = reinterpret_cast<float*>(&tco[cc * 4 + q / 2]);
        float* o2 = reinterpret_cast<float*>(&tnof[cc * 4 + q / 2]);
        c2[q & 1] = co;
        o2[q & 1] = nof;
      }
  };
  TileInfo ti = tile_at(p.ts, blk, g0);
  if (n > 0) load_row_tables(ti);  // the CTA never leaves this block
  // A stage `as` lives in TMEM columns [kScoreABase + as*KP, + KP): hi in the first
  // KP/2 (two f16 per column), lo in the next KP/2; this thread's lane = its row
  const uint32_t tl =
      warp_uniform(tmem + ((uint32_t)(32 * ((tid >> 5) & 3)) << 16) + kScoreABase + 4 * c_lo);
  if (h == 0) {  // zero the all-padding chunks of both A stages (never rewritten)
    const uint32_t tz = warp_uniform(tmem + ((uint32_t)(32 * ((tid >> 5) & 3)) << 16) + kScoreABase);
    for (int st = 0; st < kScoreAStages; ++st)
      for (int c = nchr; c < NCH; ++c) {
        tmem_st4(tz + st * KP + 4 * c, 0u, 0u, 0u, 0u);
        tmem_st4(tz + st * KP + KP / 2 + 4 * c, 0u, 0u, 0u, 0u);
      }
    tmem_st_wait();
  }
  const float2* nm0 = mu + 8 * c_lo;
  const uint32_t ring32 = smem_u32(raw_ring), raw_full32 = smem_u32(raw_full);
  const uint32_t raw_empty32 = smem_u32(raw_empty), a_full32 = smem_u32(a_full);
  const uint32_t a_empty32 = smem_u32(a_empty);
  int s = 0;
  uint32_t ph = 0, aph = 0;
  // the tile loop is unrolled over the two A stages: with the stage a compile-time constant
  // every tcgen05.st address is the loop-invariant uniform base plus an immediate (one R2UR
  // per warp for the whole loop instead of ~5 R2UR + NOPs per tile)
  static_assert(kScoreAStages == 2, "the transform loop is unrolled over two A stages");
  auto tile = [&](int t, auto as_c) {
    constexpr int AS = decltype(as_c)::value;
    if (t > 0) tile_next_in_block(p.ts, ti, gstep);
    // rows past the tile's end transform stale ring bytes (finite u16 counts): the
    // TMEM stores are warp-collective, and the epilogue drops those rows
    float g = 1.0f;
    if (MODE >= 2 && p.gain) {
      const int64_t line = ti.line0 + r / ti.w;
      g = __ldg(p.gain + (line < p.ts.L ? line : p.ts.L - 1));
    }
    SC_PW(0, mbar_wait(raw_full32 + 8 * s, ph));
    SC_PW(1, mbar_wait(a_empty32 + 8 * AS, aph ^ 1));
    tc_fence_after();
    const uint32_t roff = s * p.raw_stage_bytes + r * B * 2 + 16 * c_lo;
    const uint32_t thi = tl + AS * KP;
#ifndef SCX_NO_XFORM  // ablation switches (tools/build_sc_var.sh), off in the product
    if constexpr (BATCHED) {
      SC_PW(2, transform_row_batched<CHT>(ring32 + roff, tco, tnof, thi, thi + KP / 2));
    } else {
      SC_PW(2, transform_row<MODE, CHT>(raw_ring + roff, ring32 + roff, tco, tnof, nm0, g, thi,
                                        thi + KP / 2, cnt));
    }
#endif
    SC_PW(3, tmem_st_wait());
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {  // one arrival per warp
      mbar_arrive(a_full32 + 8 * AS);
      mbar_arrive(raw_empty32 + 8 * s);
    }
    if (++s == NR) s = 0, ph ^= 1;
    if (AS == kScoreAStages - 1) aph ^= 1;
  };
  for (int t = 0; t < n; t += 2) {
    tile(t, std::integral_constant<int, 0>{});
    if (t + 1 < n) tile(t + 1, std::integral_constant<int, 1>{});
  }
}

template <int KP>
__global__ void __maxnreg__(sc_maxreg(KP)) score_tc_kernel(
    const __grid_constant__ CUtensorMap tmap, const __grid_constant__ ScoreTcParams p) {
  constexpr int kTcTransform = 128 * sc_groups(KP);
  constexpr int kEpiWarp0 = kTcTransform / 32;
  constexpr int kTmaWarp = (kTcTransform + kTcEpilogue) / 32;
  constexpr int kMmaWarp = kTmaWarp + 1;
  constexpr int NP = KP;
  constexpr int NCH = KP / 8;            // 8-band chunks per row
  static_assert(KP % 16 == 0, "KP is a multiple of 16: both row halves own NCH/2 chunks");
  constexpr uint32_t W_BYTES = NP * KP * 2u;
  constexpr uint32_t SBO_B = (KP / 8) * 128u;
  constexpr uint32_t TMEM_COLS = 512;
  constexpr int AW = kScoreNcat ? 2 * NP : NP;  // TMEM columns per accumulator
  static_assert(kScoreAcc * AW <= kScoreABase, "accumulators below the A ring");
  static_assert(!kScoreNcat || 2 * NP <= 256, "N = 2 KP fits one MMA");
  static_assert(kScoreABase + kScoreAStages * KP <= 512, "A ring fits TMEM");
  extern __shared__ __align__(1024) uint8_t sm[];
  const int B = p.ts.B;
  uint8_t* raw_ring = sm;
  const int NR = p.nraw;
  uint8_t* wsm = raw_ring + NR * p.raw_stage_bytes;
  float* colscale = reinterpret_cast<float*>(wsm + 2 * W_BYTES);
  float2* mu = reinterpret_cast<float2*>(colscale + NP);   // [KP] {-mu, 0}
  uint32_t* shist = reinterpret_cast<uint32_t*>(mu + KP);  // [2048] digit-0 histogram
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(shist + kTopkBins) + 7) & ~uintptr_t(7));
  uint64_t* raw_full = bars;
  uint64_t* raw_empty = raw_full + kScoreRawStagesMax;
  uint64_t* a_full = raw_empty + kScoreRawStagesMax;
  uint64_t* a_empty = a_full + kScoreAStages;
  uint64_t* acc_full = a_empty + kScoreAStages;
  uint64_t* acc_empty = acc_full + kScoreAcc;
  uint64_t* w_bar = acc_empty + kScoreAcc;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(w_bar + 1);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
#ifdef SKYRX_SC_PROFILE
  const unsigned long long sc_t0 = clock64();
#endif
  // block-pinned schedule: this CTA walks line groups g0, g0 + gstep, ... of block blk
  const int blk = p.plan.block[blockIdx.x];
  const int64_t g0 = p.plan.rank[blockIdx.x];
  const int64_t gstep = p.plan.count[blockIdx.x];
  const int64_t ngb = block_groups(p.ts, blk);
  const int n = g0 < ngb ? (int)((ngb - 1 - g0) / gstep + 1) : 0;

  if (tid == 0) {
    for (int s = 0; s < NR; ++s)
      mbar_init(&raw_full[s], 1), mbar_init(&raw_empty[s], kTcTransform / 32);
    for (int s = 0; s < kScoreAStages; ++s)
      mbar_init(&a_full[s], kTcTransform / 32), mbar_init(&a_empty[s], 1);
    for (int s = 0; s < kScoreAcc; ++s)
      mbar_init(&acc_full[s], 1), mbar_init(&acc_empty[s], kTcEpilogue / 32);
    mbar_init(w_bar, 1);
    fence_mbar_init();
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_slot, TMEM_COLS);
  // mu[k].x = f32(-mu_k): clamp floor of the centred value, read as a warp broadcast
  for (int i = tid; i < kTopkBins; i += blockDim.x) shist[i] = 0;
  for (int k = tid; k < KP; k += blockDim.x)
    mu[k] = k < B ? make_float2((float)(-((double)p.mu_hilo[k] + (double)p.mu_hilo[B + k])), 0.0f)
                  : make_float2(0.0f, 0.0f);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kTmaWarp) {
    if ((tid & 31) == 0) {  // ------------------------------------------- TMA producer
      const uint32_t wb = wpack_bytes_for(KP);
      mbar_arrive_expect_tx(w_bar, wb);
      bulk_g2s(wsm, p.wpack, wb, w_bar);
      int s = 0;
      uint32_t ph = 0;
      TileInfo ti = tile_at(p.ts, blk, g0);
      for (int t = 0; t < n; ++t) {
        if (t > 0) tile_next_in_block(p.ts, ti, gstep);
        mbar_wait(&raw_empty[s], ph ^ 1);
        const uint32_t seg = (uint32_t)ti.w * B * 2u;
        const bool by_map = ti.r > 1 && p.map_last;
        // a tensor copy always lands the full box (lines past L are zero-filled)
        mbar_arrive_expect_tx(&raw_full[s], seg * (uint32_t)(by_map ? ti.r : ti.nlines));
        uint8_t* dst = raw_ring + s * p.raw_stage_bytes;
        if (by_map) {
          // narrow block: nlines x seg bytes, one tensor copy (box = full tile)
          tma_load_2d(dst, &tmap, (int)((int64_t)ti.s0 * B / 2), (int)ti.line0, &raw_full[s]);
        } else {
          for (int li = 0; li < ti.nlines; ++li) {
            const uint16_t* src = p.raw + ((ti.line0 + li) * (int64_t)p.ts.S + ti.s0) * B;
            bulk_g2s(dst + li * seg, src, seg, &raw_full[s]);
          }
        }
        if (++s == NR) s = 0, ph ^= 1;
      }
    }
  } else if (warp == kMmaWarp) {
#ifdef SCX_LANE0_ISSUE  // experiment: the issuing loop on lane 0 alone
    if ((tid & 31) == 0) {
#else
    {  // ------------------------------- MMA issuer (whole warp, the elected lane issues)
#endif
      mbar_wait(w_bar, 0);
      int as = 0, acs = 0;
      uint32_t aph = 0, cph = 0;
      for (int t = 0; t < n; ++t) {
        SC_PW(4, mbar_wait(&a_full[as], aph));
        SC_PW(5, mbar_wait(&acc_empty[acs], cph ^ 1));
        tc_fence_after();
        const uint32_t abase = tmem + kScoreABase + as * KP;  // A from TMEM
        const uint32_t d = tmem + acs * AW;
#ifdef SCX_LANE0_ISSUE
        if (true) {
#else
        if (elect_one()) {
#endif
        // W = L^-1 is lower triangular: k-step ks (k in [16ks, 16ks+16)) only feeds
        // outputs j >= 16ks, so its MMAs cover N = KP - 16ks columns from column 16ks
        // (40 % fewer tensor cycles at KP = 80); k-step 0 spans every column and
        // initialises the accumulator.
#pragma unroll
        for (int ks = 0; ks < KP / 16; ++ks) {
          const uint32_t ahi = abase + ks * 8;
          const uint32_t alo = abase + KP / 2 + ks * 8;
          const uint32_t off_b = (uint32_t)(2 * ks) * SBO_B + ks * 256;  // rows j >= 16ks
          const uint64_t bhi = smem_desc(wsm + off_b, 128, SBO_B);
          const uint64_t blo = smem_desc(wsm + W_BYTES + off_b, 128, SBO_B);
          const uint32_t idk = idesc_f16_f32(128, NP - 16 * ks, 0, 0);
          const uint32_t dk = d + 16 * ks;
#ifndef SCX_NO_MMA
          if constexpr (kScoreNcat) {
            // B rows: W_hi rows 16ks.. then (contiguous in shared memory) all of W_lo
            (void)blo;
            mma_f16_ts(dk, ahi, bhi, idesc_f16_f32(128, 2 * NP - 16 * ks, 0, 0), ks > 0);
            mma_f16_ts(dk, alo, bhi, idk, 1);
          } else {
            mma_f16_ts(dk, ahi, bhi, idk, ks > 0);
#ifndef SCX_ONE_PRODUCT
            mma_f16_ts(dk, ahi, blo, idk, 1);
            mma_f16_ts(dk, alo, bhi, idk, 1);
#endif
          }
#endif
        }
        mma_commit(&a_empty[as]);
        mma_commit(&acc_full[acs]);
        }
#ifndef SCX_LANE0_ISSUE
        __syncwarp();
#endif
        if (++as == kScoreAStages) as = 0, aph ^= 1;
        if (++acs == kScoreAcc) acs = 0, cph ^= 1;
      }
    }
  } else if (warp >= kEpiWarp0) {  // ------------------------------------ epilogue
    const int r = tid & 127;  // pixel row = TMEM lane
    const int lane = tid & 31;
    mbar_wait(w_bar, 0);
    const float ws2 = colscale[0] * colscale[0];  // one power-of-two scale for all of W
    const uint32_t tbase = warp_uniform(tmem + ((uint32_t)(32 * (warp & 3)) << 16));
    uint32_t local_max = 0;
    TileInfo ti = tile_at(p.ts, blk, g0);
    // the CTA never leaves its block, so a row's (line, sample) offsets are fixed
    const int li = n > 0 ? r / ti.w : 0;
    const int sc = r - li * ti.w;
    const uint32_t acc_full32 = smem_u32(acc_full), acc_empty32 = smem_u32(acc_empty);
    uint32_t cph = 0;
    // unrolled over the two accumulators (constant TMEM addresses, as in the transform)
    static_assert(kScoreAcc == 2, "the epilogue loop is unrolled over two accumulators");
    auto tile = [&](int t, auto acs_c) {
      constexpr int acs = decltype(acs_c)::value;
      if (t > 0) tile_next_in_block(p.ts, ti, gstep);
      SC_PW(6, mbar_wait(acc_full32 + 8 * acs, cph));
      tc_fence_after();
      float2 acc = make_float2(0.0f, 0.0f);
      const uint32_t tacc = tbase + acs * AW;
#ifdef SCX_NO_EPI
      if (false)
#endif
#pragma unroll
      for (int c = 0; c < NCH; c += 2) {
        uint32_t v[16];
        tmem_ld16(tacc + c * 8, v);
        if constexpr (kScoreNcat) {
          uint32_t w[16];
          tmem_ld16(tacc + NP + c * 8, w);
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 16; q += 2) {
            const float2 z = fadd2(make_float2(__uint_as_float(v[q]), __uint_as_float(v[q + 1])),
                                   make_float2(__uint_as_float(w[q]), __uint_as_float(w[q + 1])));
            acc = ffma2(z, z, acc);
          }
        } else {
          tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 16; q += 2) {
            const float2 z = make_float2(__uint_as_float(v[q]), __uint_as_float(v[q + 1]));
            acc = ffma2(z, z, acc);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty32 + 8 * acs);  // one arrival per warp
      const bool valid = r < ti.rows;
      uint32_t key = 0;
      if (valid) {
        const float sum = (acc.x + acc.y) * ws2;
        p.scores[(ti.line0 + li) * (int64_t)p.ts.S + ti.s0 + sc] = sum;
        key = f2ord(sum);
        local_max = max(local_max, key);
      }
      if (p.hist0 && valid)  // shared-memory histogram of the top 11 key bits
        atomicAdd(&shist[key >> 21], 1u);  // plain: __match_any_sync cost ~10 % of the kernel
      if (acs == kScoreAcc - 1) cph ^= 1;
    };
    for (int t = 0; t < n; t += 2) {
      tile(t, std::integral_constant<int, 0>{});
      if (t + 1 < n) tile(t + 1, std::integral_constant<int, 1>{});
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
      local_max = max(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
    if (lane == 0 && local_max && p.max_key) atomicMax(p.max_key, local_max);
  } else {  // ------------------------------------------------------------ transform
    mbar_wait(w_bar, 0);
    // one arithmetic mode for the whole launch (uniform branch):
    //   odd B -> 3; per-line gains given -> 2; moments pass proved raw >= dark -> 0; else 1
    const bool noclamp = p.flags != nullptr && flags_noclamp(__ldg(p.flags));
    // chunks per thread: sized for B = KP; a smaller B runs fewer (cnt, runtime)
    constexpr int NG = sc_groups(KP), NCH = KP / 8;
    constexpr int CHT = (NCH + NG - 1) / NG;
    if (B & 1)
      transform_loop<KP, 3, CHT>(p, n, blk, g0, gstep, raw_ring, tmem, mu, raw_full, raw_empty,
                                 a_full, a_empty);
    else if (p.gain != nullptr)
      transform_loop<KP, 2, CHT>(p, n, blk, g0, gstep, raw_ring, tmem, mu, raw_full, raw_empty,
                                 a_full, a_empty);
#ifndef SCX_NO_BATCHED
    else if (noclamp && KP == 80 && (B + 7) / 8 == 9) {
      // B = 65..72 (c1-c4): exactly three chunks per thread, batched
      if constexpr (KP == 80)
        transform_loop<KP, 0, 3, true>(p, n, blk, g0, gstep, raw_ring, tmem, mu, raw_full,
                                       raw_empty, a_full, a_empty);
    }
#endif
    else if (noclamp)
      transform_loop<KP, 0, CHT>(p, n, blk, g0, gstep, raw_ring, tmem, mu, raw_full, raw_empty,
                                 a_full, a_empty);
    else
      transform_loop<KP, 1, CHT>(p, n, blk, g0, gstep, raw_ring, tmem, mu, raw_full, raw_empty,
                                 a_full, a_empty);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc(tmem, TMEM_COLS);
#ifdef SKYRX_SC_PROFILE
  if (tid == 0) sc_prof[blockIdx.x][9] += clock64() - sc_t0;
#endif
  if (p.hist0)
    for (int i = tid; i < kTopkBins; i += blockDim.x)
      if (shist[i]) atomicAdd(&p.hist0[i], shist[i]);
}

// W (f64, row-major B x B, lower) -> f16 hi/lo K-major B operand + column scales
template <int KP>
__global__ void pack_whiten_kernel(const double* __restrict__ w64, int B, uint8_t* __restrict__ out) {
  constexpr uint32_t SBO_B = (KP / 8) * 128u;
  constexpr uint32_t W_BYTES = KP * KP * 2u;
  const double* W = w64 + (size_t)blockIdx.x * B * B;
  uint8_t* o = out + (size_t)blockIdx.x * wpack_bytes_for(KP);
  float* colscale = reinterpret_cast<float*>(o + 2 * W_BYTES);
  // one power-of-two scale for the whole matrix (the epilogue then squares raw
  // accumulators and multiplies once); tiny rows stay accurate in absolute terms,
  // which is what delta = sum_j z_j^2 needs
  __shared__ double smx[32];
  double m0 = 0.0;
  for (int e = threadIdx.x; e < B * B; e += blockDim.x) m0 = fmax(m0, fabs(W[e]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m0 = fmax(m0, __shfl_xor_sync(0xffffffffu, m0, o));
  if ((threadIdx.x & 31) == 0) smx[threadIdx.x >> 5] = m0;
  __syncthreads();
  double mx = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) mx = fmax(mx, smx[i]);
  int e = 0;
  if (mx > 0.0) frexp(mx, &e);           // mx in [2^(e-1), 2^e)
  const double sc = ldexp(1.0, 14 - e);  // max scaled value in [2^13, 2^14)
  for (int jn = threadIdx.x; jn < KP; jn += blockDim.x) colscale[jn] = (float)ldexp(1.0, e - 14);
  // one thread per (jn, k) entry, k fastest: neighbouring threads write neighbouring halves
  for (int t = threadIdx.x; t < KP * KP; t += blockDim.x) {
    const int jn = t / KP, k = t - jn * KP;
    const double v = (jn < B && k < B && k <= jn) ? W[(size_t)jn * B + k] * sc : 0.0;
    const __half hh = __double2half(v);
    const __half l = __double2half(v - (double)__half2float(hh));
    const uint32_t off = (jn >> 3) * SBO_B + (k >> 3) * 128u + (jn & 7) * 16u + (k & 7) * 2u;
    *reinterpret_cast<__half*>(o + off) = hh;
    *reinterpret_cast<__half*>(o + W_BYTES + off) = l;
  }
}

static int kp_for(int B) { return ((B + 15) / 16) * 16; }

template <int KP>
static int launch_score_tc(ScoreTcParams p, cudaStream_t st) {
  p.raw_stage_bytes = (uint32_t)(((128u * p.ts.B * 2u) + 127u) & ~127u);
  const size_t fixed = wpack_bytes_for(KP) + KP * 8 + kTopkBins * 4 +
                       (2 * kScoreRawStagesMax + 2 * kScoreAStages + 5) * 8 + 16 + 64;
  int nraw = (int)((kSmemMax - fixed) / p.raw_stage_bytes);
  if (nraw > kScoreRawStagesMax) nraw = kScoreRawStagesMax;
  if (nraw < 2) {
    set_error("score_tc: shared memory too small for B = %d", p.ts.B);
    return SKYRX_ERR_ARG;
  }
  p.nraw = nraw;
  const size_t smem = fixed + (size_t)nraw * p.raw_stage_bytes;
  if (p.ts.items < 1) return SKYRX_OK;
  if (p.ts.nb > kMaxPlanCtas) {
    set_error("score_tc: %d sample blocks exceed the schedule table", p.ts.nb);
    return SKYRX_ERR_ARG;
  }
#ifndef SCX_GRID_ENV
  const int grid = plan_ctas(p.ts, p.ts.items < kSMs ? (int)p.ts.items : kSMs, p.plan);
#else  // experiment: fewer CTAs than SMs (run beside another kernel)
  int g0 = kSMs;
  if (const char* e = getenv("SKYRX_SC_GRID")) g0 = atoi(e) > 0 ? atoi(e) : g0;
  const int grid = plan_ctas(p.ts, p.ts.items < g0 ? (int)p.ts.items : g0, p.plan);
#endif
  // the narrow last block packs rl lines per tile: fetch each tile with ONE 2-D
  // TMA (u32 elements; box = wl*B/2 x rl) instead of rl tiny line copies
  CUtensorMap map;
  memset(&map, 0, sizeof(map));
  p.map_last = 0;
  const int64_t box0 = (int64_t)p.ts.wl * p.ts.B / 2;
  if (p.ts.rl > 1 && box0 <= 256 && p.ts.rl <= 256 && tensor_map_encoder() != nullptr) {
    const cuuint64_t line_bytes = (cuuint64_t)p.ts.S * p.ts.B * 2;
    cuuint64_t dims[2] = {line_bytes / 4, (cuuint64_t)p.ts.L};
    cuuint64_t strides[1] = {line_bytes};
    cuuint32_t box[2] = {(cuuint32_t)box0, (cuuint32_t)p.ts.rl};
    cuuint32_t estr[2] = {1, 1};
    const CUresult r = tensor_map_encoder()(
        &map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, (void*)p.raw, dims, strides, box, estr,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    p.map_last = r == CUDA_SUCCESS ? 1 : 0;
  }
  cudaFuncSetAttribute(score_tc_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  score_tc_kernel<KP><<<grid, sc_threads(KP), smem, st>>>(map, p);
  SKYRX_CHECK_LAUNCH("score_tc_kernel");
  return SKYRX_OK;
}

}  // namespace skyrx

using namespace skyrx;

extern "C" size_t skyrx_wpack_bytes(int32_t bands) {
  return wpack_bytes_for(kp_for(bands));
}

extern "C" int skyrx_pack_whiten(const double* whiten64, int32_t bands, int32_t batch,
                                 void* wpack, void* stream) {
  SKYRX_REQUIRE(bands > 0 && bands <= 80 && batch >= 1, "pack_whiten supports 1 <= B <= 80");
  cudaStream_t st = as_stream(stream);
  switch (kp_for(bands)) {
#define SKYRX_KP(k) \
  case k:           \
    pack_whiten_kernel<k><<<batch, 512, 0, st>>>(whiten64, bands, (uint8_t*)wpack); break;
    SKYRX_KP(16) SKYRX_KP(32) SKYRX_KP(48) SKYRX_KP(64) SKYRX_KP(80)
#undef SKYRX_KP
  }
  SKYRX_CHECK_LAUNCH("skyrx_pack_whiten");
  return SKYRX_OK;
}

extern "C" int skyrx_score_tc_supported(int64_t lines, int32_t samples, int32_t bands,
                                        const void* raw) {
  TileSched ts;
  if (bands < 1 || bands > 80) return 0;  // KP = 96 would need > 227 KB of shared memory
  if (((uintptr_t)raw & 15) != 0) return 0;
  return tc_sched(lines, samples, bands, kScoreWmax, ts) ? 1 : 0;
}

extern "C" int skyrx_score_tc(const uint16_t* raw, int64_t lines, int32_t samples, int32_t bands,
                              const float* dark, const float* coeff, const float* gain,
                              const float* mu_hilo, const void* wpack, const int32_t* flags,
                              float* scores, uint32_t* max_key, uint32_t* topk_hist0,
                              void* stream) {
  SKYRX_REQUIRE(skyrx_score_tc_supported(lines, samples, bands, raw),
                "tensor-core score path unsupported for this shape/alignment");
  ScoreTcParams p{};
  p.raw = raw;
  p.dark = dark;
  p.coeff = coeff;
  p.gain = gain;
  p.mu_hilo = mu_hilo;
  p.wpack = (const uint8_t*)wpack;
  p.scores = scores;
  p.max_key = max_key;
  p.hist0 = topk_hist0;
  p.flags = flags;
  tc_sched(lines, samples, bands, kScoreWmax, p.ts);
  if (lines * (int64_t)samples == 0) return SKYRX_OK;
  cudaStream_t st = as_stream(stream);
  switch (kp_for(bands)) {
    case 16: return launch_score_tc<16>(p, st);
    case 32: return launch_score_tc<32>(p, st);
    case 48: return launch_score_tc<48>(p, st);
    case 64: return launch_score_tc<64>(p, st);
    case 80: return launch_score_tc<80>(p, st);
  }
  set_error("unsupported band count %d", bands);
  return SKYRX_ERR_ARG;
}

#ifdef SKYRX_SC_PROFILE
extern "C" __attribute__((visibility("default"))) int skyrx_sc_profile(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, skyrx::sc_prof, sizeof(skyrx::sc_prof)) == cudaSuccess ? 0 : 1;
}
#endif
