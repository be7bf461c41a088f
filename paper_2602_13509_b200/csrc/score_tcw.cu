// K4-TCW — the exact-digit tensor-core score (score_tcs.cu) for WIDE cubes,
// 128 < B <= 272 (BASELINE config 3, B = 270).
//
// Same arithmetic as K4-TCS: per sample column s, z = V_s a + q_s with a = r - R_s
// split into two f16-exact digits and V_s = W diag(c_s / g) in f16 hi + lo, four
// tcgen05 products, f32 in TMEM.  What changes at this width:
//   * V_s (KP x KP, hi + lo = 296 KB at KP = 272) does not fit shared memory, so it
//     is streamed per tile in N-blocks of 64 output rows through a two-stage ring
//     (1-D bulk copies from the L2-resident per-sample record); block nb only needs
//     K < 64 (nb + 1) because V_s is lower triangular;
//   * TMEM holds the digit operands of one tile (KP columns) and a double-buffered
//     64-column accumulator, so the epilogue squares block nb while the tensor core
//     runs block nb + 1; A is single-buffered (the next tile's transform waits for
//     the current tile's last block);
//   * the raw window of a line is fetched as u32 elements (a box <= 256 elements).
// Warps: 4 transform groups (16 warps), 4 epilogue warps, TMA, MMA.
#include <cuda_fp16.h>

#include "common.cuh"
#include "tma.cuh"
#include "umma.cuh"

namespace skyrx {
using namespace umma;

namespace tcw {

constexpr int kLines = 128;
constexpr int kNB = 64;           // output rows per N-block
constexpr int kAccBase = 0;       // TMEM: 2 x 64 accumulator columns
constexpr int kABase = 128;       // TMEM: A hi [128, 128 + KP/2), A lo [.., 128 + KP)
constexpr int kHist = 2048;
constexpr int kGroups = 4;
constexpr int kThreads = 128 * kGroups + 128 + 64;
constexpr int kMaxReg = (16384 / (32 * ((kThreads / 32 + 3) / 4))) / 8 * 8;
constexpr int64_t kMaxUnitLines = 16384;

__host__ __device__ constexpr int nblocks(int kp) { return (kp + kNB - 1) / kNB; }
__host__ __device__ constexpr int nb_rows(int kp, int nb) {
  return kp - kNB * nb < kNB ? kp - kNB * nb : kNB;
}
__host__ __device__ constexpr int nb_kend(int kp, int nb) { return kNB * nb + nb_rows(kp, nb); }
// bytes of one N-block's operand (hi, then lo): rows x kend f16 each
__host__ __device__ constexpr uint32_t nb_bytes(int kp, int nb) {
  return 2u * 2u * (uint32_t)nb_rows(kp, nb) * (uint32_t)nb_kend(kp, nb);
}
__host__ __device__ constexpr uint32_t nb_offset(int kp, int nb) {
  uint32_t o = 0;
  for (int m = 0; m < nb; ++m) o += nb_bytes(kp, m);
  return o;
}
__host__ __device__ constexpr uint32_t max_nb_bytes(int kp) {
  uint32_t m = 0;
  for (int nb = 0; nb < nblocks(kp); ++nb) m = m > nb_bytes(kp, nb) ? m : nb_bytes(kp, nb);
  return m;
}
// per-sample record: N-block operands | tail: T (KP u16) | q' (KP f32) | inv_scale (f32)
__host__ __device__ constexpr uint32_t tail_bytes(int kp) {
  return ((2u * kp + 4u * kp + 4u) + 15u) & ~15u;
}
__host__ __device__ constexpr uint32_t rec_bytes(int kp) {
  return ((nb_offset(kp, nblocks(kp)) + tail_bytes(kp)) + 127u) & ~127u;
}

struct Params {
  const uint8_t* rec;
  float* scores;
  uint32_t* max_key;
  uint32_t* hist0;
  int32_t* flags;
  int64_t L;
  int32_t S, B;
  int64_t split_lines;
  int64_t units;
  int32_t nw;          // u32 words per line in the tile box (odd number of 16-B chunks x 4)
  uint32_t stage_bytes;
};

__device__ __forceinline__ void unit_geom(const Params& p, int64_t u, int& s, int64_t& l0,
                                          int64_t& nl) {
  s = (int)(u % p.S);
  l0 = (u / p.S) * p.split_lines;
  nl = p.L - l0 < p.split_lines ? p.L - l0 : p.split_lines;
}

__device__ __forceinline__ void digits4(const uint32_t (&w)[4], const uint32_t* t,
                                        uint32_t (&hw)[4], uint32_t (&lw)[4], uint32_t& chk) {
  const __half2 bias_hi = __floats2half2_rn(-36864.0f, -36864.0f);
  const __half2 bias_lo = __floats2half2_rn(-1024.0f, -1024.0f);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    chk |= w[i];
    const uint32_t u = w[i] + t[i];
    const uint32_t hb = ((u >> 5) & 0x00FE00FEu) | 0x78007800u;
    const uint32_t lb = (u & 0x003F003Fu) | 0x64006400u;
    __half2 hh = __hadd2(*reinterpret_cast<const __half2*>(&hb), bias_hi);
    __half2 ll = __hadd2(*reinterpret_cast<const __half2*>(&lb), bias_lo);
    hw[i] = *reinterpret_cast<uint32_t*>(&hh);
    lw[i] = *reinterpret_cast<uint32_t*>(&ll);
  }
}

template <int KP, int CHT, int OFFW>
__device__ __forceinline__ void transform_tile(const uint8_t* stage, uint32_t rowb, uint32_t tl,
                                               const uint32_t* tt, int c_lo, int cnt,
                                               uint32_t& chk) {
  const int r = threadIdx.x & 127;
  const uint4* row = reinterpret_cast<const uint4*>(stage + r * rowb);
  uint4 cur = cnt > 0 ? row[c_lo] : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
  for (int cc = 0; cc < CHT; ++cc) {
    if (cc >= cnt) break;  // warp-uniform
    const uint4 nxt = row[c_lo + cc + 1];
    const uint32_t c8[8] = {cur.x, cur.y, cur.z, cur.w, nxt.x, nxt.y, nxt.z, nxt.w};
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = c8[OFFW + i];
    uint32_t hw[4], lw[4];
    digits4(w, tt + 4 * cc, hw, lw, chk);
    const uint32_t col = tl + 4 * (c_lo + cc);
    tmem_st4(col, hw[0], hw[1], hw[2], hw[3]);
    tmem_st4(col + KP / 2, lw[0], lw[1], lw[2], lw[3]);
    cur = nxt;
  }
}

template <int KP>
__global__ void __maxnreg__(kMaxReg) score_tcw_kernel(const __grid_constant__ CUtensorMap tmap,
                                                      const __grid_constant__ Params p) {
  constexpr int NT = 128 * kGroups;
  constexpr int EPI0 = NT / 32, TMAW = EPI0 + 4, MMAW = TMAW + 1;
  constexpr int NCH = KP / 8;
  constexpr int CHT = (NCH + kGroups - 1) / kGroups;
  constexpr int NNB = nblocks(KP);
  constexpr uint32_t TB = tail_bytes(KP);
  constexpr uint32_t RB = rec_bytes(KP);
  constexpr uint32_t BSTAGE = max_nb_bytes(KP);
  constexpr uint32_t TAIL_OFF = nb_offset(KP, NNB);
  static_assert(kABase + KP <= 512, "TMEM budget");
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* bring = sm;                               // [2][BSTAGE]
  uint8_t* raw = bring + 2 * BSTAGE;                 // one raw stage
  uint8_t* tails = raw + p.stage_bytes;              // [2][TB]
  uint32_t* shist = reinterpret_cast<uint32_t*>(tails + 2 * TB);
  uint64_t* bars = reinterpret_cast<uint64_t*>(shist + kHist);
  uint64_t* raw_full = bars;
  uint64_t* raw_empty = bars + 1;
  uint64_t* a_full = bars + 2;
  uint64_t* a_empty = bars + 3;
  uint64_t* b_full = bars + 4;       // [2]
  uint64_t* b_empty = bars + 6;      // [2]
  uint64_t* acc_full = bars + 8;     // [2]
  uint64_t* acc_empty = bars + 10;   // [2]
  uint64_t* tail_full = bars + 12;   // [2]
  uint64_t* tail_empty = bars + 14;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int B = p.B;
  const int64_t u0 = blockIdx.x, ustep = gridDim.x;
  // the exact-digit form needs "no raw value below dark" from the moments pass;
  // without that proof nothing is scored and flags |= 32 asks for a general rescore
  if (!flags_noclamp(__ldg(p.flags))) {
    if (blockIdx.x == 0 && tid == 0) atomicOr(p.flags, 32);
    return;
  }

  if (tid == 0) {
    mbar_init(raw_full, 1), mbar_init(raw_empty, NT / 32);
    mbar_init(a_full, NT / 32), mbar_init(a_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&b_full[i], 1), mbar_init(&b_empty[i], 1);
      mbar_init(&acc_full[i], 1), mbar_init(&acc_empty[i], 4);
      mbar_init(&tail_full[i], 1), mbar_init(&tail_empty[i], NT / 32 + 4);
    }
    fence_mbar_init();
  }
  for (int i = tid; i < kHist; i += blockDim.x) shist[i] = 0;
  if (warp == MMAW) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == TMAW) {
    if (lane == 0) {  // ------------------------------------------------- TMA producer
      int ui = 0, bs = 0;
      uint32_t rph = 0, bph = 0;
      for (int64_t u = u0; u < p.units; u += ustep, ++ui) {
        int smp;
        int64_t l0, nl;
        unit_geom(p, u, smp, l0, nl);
        const uint8_t* rec = p.rec + (size_t)smp * RB;
        const int tb = ui & 1;
        mbar_wait(&tail_empty[tb], ((ui >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&tail_full[tb], TB);
        bulk_g2s(tails + tb * TB, rec + TAIL_OFF, TB, &tail_full[tb]);
        const int c0 = (int)((((int64_t)smp * B * 2) & ~(int64_t)15) >> 2);
        const int ntile = (int)((nl + kLines - 1) / kLines);
        for (int k = 0; k < ntile; ++k) {
          mbar_wait(raw_empty, rph ^ 1);
          mbar_arrive_expect_tx(raw_full, p.stage_bytes);
          tma_load_2d(raw, &tmap, c0, (int)(l0 + (int64_t)k * kLines), raw_full);
          rph ^= 1;
#pragma unroll 1
          for (int nb = 0; nb < NNB; ++nb) {
            mbar_wait(&b_empty[bs], bph ^ 1);
            const uint32_t nbb = nb_bytes(KP, nb);
            mbar_arrive_expect_tx(&b_full[bs], nbb);
            bulk_g2s(bring + bs * BSTAGE, rec + nb_offset(KP, nb), nbb, &b_full[bs]);
            if (++bs == 2) bs = 0, bph ^= 1;
          }
        }
      }
    }
  } else if (warp == MMAW) {
    {  // ------------------------------- MMA issuer (whole warp, the elected lane issues)
      int ui = 0, bs = 0, acs = 0;
      uint32_t aph = 0, bph = 0, cph = 0;
      const uint32_t ahi = tmem + kABase, alo = tmem + kABase + KP / 2;
      for (int64_t u = u0; u < p.units; u += ustep, ++ui) {
        int smp;
        int64_t l0, nl;
        unit_geom(p, u, smp, l0, nl);
        const int ntile = (int)((nl + kLines - 1) / kLines);
        for (int k = 0; k < ntile; ++k) {
          mbar_wait(a_full, aph);
          aph ^= 1;
#pragma unroll 1
          for (int nb = 0; nb < NNB; ++nb) {
            const int rows = nb_rows(KP, nb), kend = nb_kend(KP, nb);
            const uint32_t sbo = (uint32_t)(kend / 8) * 128u;
            const uint32_t half = (uint32_t)rows * kend * 2u;
            mbar_wait(&b_full[bs], bph);
            mbar_wait(&acc_empty[acs], cph ^ 1);
            tc_fence_after();
            const uint8_t* bh = bring + bs * BSTAGE;
            const uint32_t id = idesc_f16_f32(128, rows, 0, 0);
            const uint32_t d = tmem + kAccBase + acs * kNB;
            if (elect_one()) {
            for (int ks = 0; ks < kend / 16; ++ks) {
              const uint64_t bhi = smem_desc(bh + ks * 256, 128, sbo);
              const uint64_t blo = smem_desc(bh + half + ks * 256, 128, sbo);
              mma_f16_ts(d, ahi + ks * 8, bhi, id, ks > 0);
              mma_f16_ts(d, ahi + ks * 8, blo, id, 1);
              mma_f16_ts(d, alo + ks * 8, bhi, id, 1);
              mma_f16_ts(d, alo + ks * 8, blo, id, 1);
            }
            mma_commit(&b_empty[bs]);
            mma_commit(&acc_full[acs]);
            if (nb == NNB - 1) mma_commit(a_empty);  // the tile's digits are consumed
            }
            __syncwarp();
            if (++bs == 2) bs = 0, bph ^= 1;
            if (++acs == 2) acs = 0, cph ^= 1;
          }
        }
      }
    }
  } else if (warp >= EPI0) {  // --------------------------------------- epilogue
    const int r = tid & 127;
    const uint32_t tbase = warp_uniform(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + kAccBase);
    uint32_t local_max = 0;
    int ui = 0, acs = 0;
    uint32_t cph = 0;
    for (int64_t u = u0; u < p.units; u += ustep, ++ui) {
      int smp;
      int64_t l0, nl;
      unit_geom(p, u, smp, l0, nl);
      const int tb = ui & 1;
      mbar_wait(&tail_full[tb], (ui >> 1) & 1);
      const float* qv = reinterpret_cast<const float*>(tails + tb * TB + 2 * KP);
      const float inv = qv[KP];
      const int ntile = (int)((nl + kLines - 1) / kLines);
      for (int k = 0; k < ntile; ++k) {
        float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll 1
        for (int nb = 0; nb < NNB; ++nb) {
          const int rows = nb_rows(KP, nb);
          mbar_wait(&acc_full[acs], cph);
          tc_fence_after();
          for (int c = 0; c < rows; c += 16) {
            uint32_t v[16];
            tmem_ld16(tbase + acs * kNB + c, v);
            tmem_ld_wait();
            const float* qb = qv + kNB * nb + c;
#pragma unroll
            for (int q = 0; q < 16; q += 4) {
              const float4 qq = *reinterpret_cast<const float4*>(qb + q);
              const float2 z0 = fadd2(make_float2(__uint_as_float(v[q]), __uint_as_float(v[q + 1])),
                                      make_float2(qq.x, qq.y));
              const float2 z1 = fadd2(
                  make_float2(__uint_as_float(v[q + 2]), __uint_as_float(v[q + 3])),
                  make_float2(qq.z, qq.w));
              acc = ffma2(z0, z0, acc);
              acc = ffma2(z1, z1, acc);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[acs]);
          if (++acs == 2) acs = 0, cph ^= 1;
        }
        const int64_t line = l0 + (int64_t)k * kLines + r;
        const bool valid = line < l0 + nl;
        uint32_t key = 0;
        if (valid) {
          const float sum = (acc.x + acc.y) * (inv * inv);
          p.scores[line * p.S + smp] = sum;
          key = f2ord(sum);
          local_max = max(local_max, key);
        }
        // plain shared atomics: __match_any_sync aggregation cost ~10 % of score_tc
        if (p.hist0 && valid) atomicAdd(&shist[key >> 21], 1u);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&tail_empty[tb]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
      local_max = max(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
    if (lane == 0 && local_max && p.max_key) atomicMax(p.max_key, local_max);
  } else {  // ------------------------------------------------------------ transform
    const int g = tid >> 7;
    const int nchr = (B + 7) / 8;
    const int cpg = (nchr + kGroups - 1) / kGroups;
    const int c_lo = cpg * g;
    const int cnt = min(cpg, nchr - c_lo);
    const uint32_t tl = warp_uniform(tmem + ((uint32_t)(32 * ((tid >> 5) & 3)) << 16) + kABase);
    if (g == 0) {  // all-padding chunks of A: zero once
      for (int c = nchr; c < NCH; ++c) {
        tmem_st4(tl + 4 * c, 0u, 0u, 0u, 0u);
        tmem_st4(tl + KP / 2 + 4 * c, 0u, 0u, 0u, 0u);
      }
      tmem_st_wait();
    }
    const uint32_t rowb = (uint32_t)p.nw * 4u;
    uint32_t chk = 0, rph = 0, aph = 0;
    int ui = 0;
    for (int64_t u = u0; u < p.units; u += ustep, ++ui) {
      int smp;
      int64_t l0, nl;
      unit_geom(p, u, smp, l0, nl);
      const int tb = ui & 1;
      mbar_wait(&tail_full[tb], (ui >> 1) & 1);
      uint32_t tt[CHT * 4];
      const uint32_t* tw = reinterpret_cast<const uint32_t*>(tails + tb * TB);
#pragma unroll
      for (int i = 0; i < CHT * 4; ++i) tt[i] = i < cnt * 4 ? tw[4 * c_lo + i] : 0u;
      __syncwarp();
      if (lane == 0) mbar_arrive(&tail_empty[tb]);
      const int offw = (int)((((int64_t)smp * B * 2) & 15) >> 2);
      const int ntile = (int)((nl + kLines - 1) / kLines);
      for (int k = 0; k < ntile; ++k) {
        mbar_wait(raw_full, rph);
        mbar_wait(a_empty, aph ^ 1);
        tc_fence_after();
        if (offw == 0) transform_tile<KP, CHT, 0>(raw, rowb, tl, tt, c_lo, cnt, chk);
        else if (offw == 1) transform_tile<KP, CHT, 1>(raw, rowb, tl, tt, c_lo, cnt, chk);
        else if (offw == 2) transform_tile<KP, CHT, 2>(raw, rowb, tl, tt, c_lo, cnt, chk);
        else transform_tile<KP, CHT, 3>(raw, rowb, tl, tt, c_lo, cnt, chk);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(a_full);
          mbar_arrive(raw_empty);
        }
        rph ^= 1;
        aph ^= 1;
      }
    }
    if (__any_sync(0xffffffffu, (chk & 0xF000F000u) != 0) && lane == 0) atomicOr(p.flags, 16);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == MMAW) tmem_dealloc(tmem, 512);
  if (p.hist0)
    for (int i = tid; i < kHist; i += blockDim.x)
      if (shist[i]) atomicAdd(&p.hist0[i], shist[i]);
}

// one CTA per (kPackS consecutive samples, background): the wide records (N-blocked V_s,
// T, q', inv).  Every element of W is read once per CTA and serves all its samples (the
// per-sample form read the 0.6 MB W four times per sample: 0.43 ms per c3 cube).  Per
// sample the arithmetic and its order are unchanged.
#ifndef TCW_PACK_S
#define TCW_PACK_S 8
#endif
constexpr int kPackS = TCW_PACK_S;

template <int KP>
__global__ void __launch_bounds__(256, 1) tcw_pack_kernel(const double* __restrict__ w64,
                                                       const float* __restrict__ mu_hilo, int B,
                                                       int S, const float* __restrict__ dark,
                                                       const float* __restrict__ coeff, double gain,
                                                       uint8_t* __restrict__ out) {
  constexpr int NNB = nblocks(KP);
  const int s0 = blockIdx.x * kPackS;
  const int ns = min(kPackS, S - s0);
  const int bg = blockIdx.y;
  const double* W = w64 + (size_t)bg * B * B;
  const float* mh = mu_hilo + (size_t)bg * 2 * B;
  __shared__ double cs[kPackS][KP], es[kPackS][KP], red[kPackS][8], scs[kPackS];
  __shared__ int exs[kPackS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < kPackS * KP; e += blockDim.x) {
    const int q = e / KP, k = e - q * KP;
    double c = 0.0, ev = 0.0;
    uint16_t t = 0;
    if (k < B && q < ns) {
      const int s = s0 + q;
      const double mu = (double)mh[k] + (double)mh[B + k];
      const double cg = (double)coeff[(size_t)s * B + k] / gain;
      const double d = (double)dark[(size_t)s * B + k];
      double R = rint(d + mu / cg);
      R = R < 0.0 ? 0.0 : (R > 4095.0 ? 4095.0 : R);
      c = cg;
      ev = cg * (R - d) - mu;
      t = (uint16_t)(4096.0 - R);
    }
    cs[q][k] = c;
    es[q][k] = ev;
    if (q < ns)
      reinterpret_cast<uint16_t*>(out + ((size_t)bg * S + s0 + q) * rec_bytes(KP) +
                                  nb_offset(KP, NNB))[k] = t;
  }
  __syncthreads();
  // per sample: the largest |W_jk c_k| -> one power-of-two scale for V_s
  double m0[kPackS];
#pragma unroll
  for (int q = 0; q < kPackS; ++q) m0[q] = 0.0;
  for (int j = warp; j < B; j += 8)
    for (int k = lane; k <= j; k += 32) {
      const double w = W[(size_t)j * B + k];
#pragma unroll
      for (int q = 0; q < kPackS; ++q) m0[q] = fmax(m0[q], fabs(w * cs[q][k]));
    }
#pragma unroll
  for (int q = 0; q < kPackS; ++q) {
    double m = m0[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) red[q][warp] = m;
  }
  __syncthreads();
  if (tid < kPackS) {
    double mx = 0.0;
    for (int w = 0; w < 8; ++w) mx = fmax(mx, red[tid][w]);
    int ex = 0;
    if (mx > 0.0) frexp(mx, &ex);
    exs[tid] = ex;
    scs[tid] = ldexp(1.0, 14 - ex);
  }
  __syncthreads();
  // q'_j = sum_k W_jk e_k (ascending k, as before), scaled
  for (int j = tid; j < KP; j += blockDim.x) {
    double qj[kPackS];
#pragma unroll
    for (int q = 0; q < kPackS; ++q) qj[q] = 0.0;
    if (j < B) {
      // the row's loads eight at a time ahead of the (ascending, serial) sums
      const double* wr = W + (size_t)j * B;
      int k = 0;
      for (; k + 8 <= j + 1; k += 8) {
        double w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = wr[k + i];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int q = 0; q < kPackS; ++q) qj[q] += w[i] * es[q][k + i];
      }
      for (; k <= j; ++k) {
        const double w = wr[k];
#pragma unroll
        for (int q = 0; q < kPackS; ++q) qj[q] += w * es[q][k];
      }
    }
#pragma unroll
    for (int q = 0; q < kPackS; ++q)
      if (q < ns) {
        float* qo = reinterpret_cast<float*>(out + ((size_t)bg * S + s0 + q) * rec_bytes(KP) +
                                             nb_offset(KP, NNB) + 2 * KP);
        qo[j] = (float)(qj[q] * scs[q]);
        if (j == 0) qo[KP] = (float)ldexp(1.0, exs[q] - 14);
      }
  }
  // N-block operands: block nb = rows [64 nb, 64 nb + rows) x K [0, kend), K-major
  // a thread takes one 16-byte core-matrix row (output row jj, k = 8 k8 .. 8 k8 + 7) for every
  // sample of the CTA; consecutive threads write consecutive 16-byte rows (the canonical
  // layout's (jj & 7) then k8 order), so each warp stores 512 contiguous bytes per sample
  for (int nb = 0; nb < NNB; ++nb) {
    const int rows = nb_rows(KP, nb), kend = nb_kend(KP, nb);
    const int nk8 = kend / 8;
    const uint32_t sbo = (uint32_t)nk8 * 128u;
    for (int g = tid; g < rows * nk8; g += blockDim.x) {
      const int jb = (g >> 3) / nk8, k8 = (g >> 3) - jb * nk8;
      const int jj = 8 * jb + (g & 7), j = kNB * nb + jj, k0 = 8 * k8;
      double w[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int k = k0 + i;
        w[i] = (j < B && k < B && k <= j) ? W[(size_t)j * B + k] : 0.0;
      }
      const uint32_t off = (uint32_t)jb * sbo + (uint32_t)k8 * 128u + (uint32_t)(g & 7) * 16u;
#pragma unroll
      for (int q = 0; q < kPackS; ++q) {
        if (q >= ns) break;
        uint32_t hw[4], lw[4];
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          const double v0 = w[i] * cs[q][k0 + i] * scs[q];
          const double v1 = w[i + 1] * cs[q][k0 + i + 1] * scs[q];
          const __half h0 = __double2half(v0), h1 = __double2half(v1);
          const __half l0 = __double2half(v0 - (double)__half2float(h0));
          const __half l1 = __double2half(v1 - (double)__half2float(h1));
          hw[i / 2] = (uint32_t)__half_as_ushort(h0) | ((uint32_t)__half_as_ushort(h1) << 16);
          lw[i / 2] = (uint32_t)__half_as_ushort(l0) | ((uint32_t)__half_as_ushort(l1) << 16);
        }
        uint8_t* hi = out + ((size_t)bg * S + s0 + q) * rec_bytes(KP) + nb_offset(KP, nb);
        *reinterpret_cast<uint4*>(hi + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(hi + (size_t)rows * kend * 2 + off) =
            make_uint4(lw[0], lw[1], lw[2], lw[3]);
      }
    }
  }
}

}  // namespace tcw

static int tcw_kp(int B) { return ((B + 15) / 16) * 16; }

// u32 words per line in the tile box: the 16-B aligned window of a sample plus one
// chunk, as an odd number of 16-B chunks (conflict-free LDS.128 across lines)
static int tcw_nw(int S, int B) {
  int maxoff = 0;
  for (int s = 0; s < 8 && s < S; ++s) maxoff = maxoff > ((s * B * 2) & 15) ? maxoff : ((s * B * 2) & 15);
  int chunks = (maxoff + 2 * B + 15) / 16 + 1;
  if ((chunks & 1) == 0) ++chunks;
  return chunks * 4;
}

template <int KP>
static int launch_tcw(const uint16_t* raw, tcw::Params p, cudaStream_t st) {
  using namespace tcw;
  p.nw = tcw_nw(p.S, p.B);
  p.stage_bytes = (uint32_t)p.nw * 4u * kLines;
  const size_t smem = 2 * (size_t)max_nb_bytes(KP) + p.stage_bytes + 2 * (size_t)tail_bytes(KP) +
                      kHist * 4 + 16 * 8 + 64;
  SKYRX_REQUIRE(smem <= kSmemMax, "score_tcw: shared memory too small for B = %d", p.B);
  const cuuint64_t line_words = (cuuint64_t)p.S * p.B / 2;
  cuuint64_t dims[2] = {line_words, (cuuint64_t)p.L};
  cuuint64_t strides[1] = {line_words * 4};
  cuuint32_t box[2] = {(cuuint32_t)p.nw, (cuuint32_t)kLines};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMap map;
  const CUresult r = tensor_map_encoder()(
      &map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, (void*)raw, dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SKYRX_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  int64_t nsplit = (p.L + kMaxUnitLines - 1) / kMaxUnitLines;
  while ((int64_t)p.S * nsplit < 8 * kSMs && p.L / (nsplit + 1) >= 4 * kLines) ++nsplit;
  p.split_lines = (p.L + nsplit - 1) / nsplit;
  p.split_lines = (p.split_lines + kLines - 1) / kLines * kLines;
  nsplit = (p.L + p.split_lines - 1) / p.split_lines;
  p.units = (int64_t)p.S * nsplit;
  int grid = kSMs;
  if (p.units < grid) grid = (int)p.units;
  cudaFuncSetAttribute(score_tcw_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  score_tcw_kernel<KP><<<grid, kThreads, smem, st>>>(map, p);
  SKYRX_CHECK_LAUNCH("score_tcw_kernel");
  return SKYRX_OK;
}

}  // namespace skyrx

using namespace skyrx;

#define SKYRX_TCW_KPS(X) X(144) X(160) X(176) X(192) X(208) X(224) X(240) X(256) X(272)

extern "C" size_t skyrx_scorew_rec_bytes(int32_t bands) {
  return (bands <= 128 || bands > 272) ? 0 : tcw::rec_bytes(tcw_kp(bands));
}

extern "C" int skyrx_scorew_prep(const double* whiten64, const float* mu_hilo, int32_t samples,
                                 int32_t bands, const float* dark, const float* coeff,
                                 double gain, int32_t batch, void* records, void* stream) {
  SKYRX_REQUIRE(bands > 128 && bands <= 272 && samples >= 1 && batch >= 1,
                "scorew_prep supports 128 < B <= 272");
  SKYRX_REQUIRE(gain > 0.0, "every line gain must be positive");
  cudaStream_t st = as_stream(stream);
  const dim3 grid((samples + tcw::kPackS - 1) / tcw::kPackS, batch);
  switch (tcw_kp(bands)) {
#define SKYRX_KP(k)                                                                        \
  case k:                                                                                  \
    tcw::tcw_pack_kernel<k><<<grid, 256, 0, st>>>(whiten64, mu_hilo, bands, samples, dark, \
                                                  coeff, gain, (uint8_t*)records);         \
    break;
    SKYRX_TCW_KPS(SKYRX_KP)
#undef SKYRX_KP
  }
  SKYRX_CHECK_LAUNCH("skyrx_scorew_prep");
  return SKYRX_OK;
}

extern "C" int skyrx_scorew_supported(int64_t lines, int32_t samples, int32_t bands,
                                      const void* raw) {
  if (bands <= 128 || bands > 272 || lines < 1 || samples < 1) return 0;
  if (bands & 1) return 0;
  if (((uintptr_t)raw & 15) != 0) return 0;
  if (((int64_t)samples * bands * 2) % 16 != 0) return 0;
  if (tcw_nw(samples, bands) > 256) return 0;
  if (lines > ((int64_t)1 << 31) - 1) return 0;
  return tensor_map_encoder() != nullptr ? 1 : 0;
}

extern "C" int skyrx_scorew(const uint16_t* raw, int64_t lines, int32_t samples, int32_t bands,
                            const void* records, int32_t* flags, float* scores, uint32_t* max_key,
                            uint32_t* topk_hist0, void* stream) {
  SKYRX_REQUIRE(skyrx_scorew_supported(lines, samples, bands, raw),
                "wide exact-digit score path unsupported for this shape/alignment");
  SKYRX_REQUIRE(flags != nullptr, "scorew needs the flags word");
  tcw::Params p{};
  p.rec = (const uint8_t*)records;
  p.scores = scores;
  p.max_key = max_key;
  p.hist0 = topk_hist0;
  p.flags = flags;
  p.L = lines;
  p.S = samples;
  p.B = bands;
  cudaStream_t st = as_stream(stream);
  switch (tcw_kp(bands)) {
#define SKYRX_KP(k) \
  case k:           \
    return launch_tcw<k>(raw, p, st);
    SKYRX_TCW_KPS(SKYRX_KP)
#undef SKYRX_KP
  }
  set_error("unsupported band count %d", bands);
  return SKYRX_ERR_ARG;
}
