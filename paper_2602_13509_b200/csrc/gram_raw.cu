// K2-RAW — background moments straight from the raw uint16 bytes on the tensor cores.
//
// For one sample column s the calibrated pixel is x = C_s (r - d_s) with
// C_s = diag(coeff[s,:]) / gain and d_s = dark[s,:] (calibrate.py:98-101,
// valid whenever no value clamps at 0 and the gain is one constant).  So
//     sum_l x x^T = C_s (G_s - d_s m_s^T - m_s d_s^T + L d_s d_s^T) C_s,
//     G_s = sum_l r r^T,  m_s = sum_l r
// and G_s is an exact integer Gram of 12..16-bit counts.  Reading a line's
// bands as their 2B little-endian bytes, G_s = 65536 HH + 256 (HL + LH) + LL
// comes from ONE byte Gram D = sum_l b b^T (b = the 2B bytes), which the
// tensor cores compute exactly (tcgen05.mma kind::i8, unsigned, s32 TMEM
// accumulators; 255^2 * 32768 lines < 2^31).  TMA loads each tile's bytes
// (128-byte x 128-line boxes, 128B-swizzled by the TMA engine) directly in the
// canonical MN-major SWIZZLE_128B UMMA layout, so no thread touches the data on its way to
// the tensor core.  The CUDA cores only scan each tile for m_s and for the
// per-band minimum (a value below dark would clamp: the cube is then redone by
// the generic path, flags |= 4); for 129..160-byte windows (B = 57..72, the c4 shape)
// m_s comes from the tensor core too (a ones atom appended to the small MMAs' B operand)
// and the scan is the minimum alone.  The scan reads conflict-free: a quarter-warp takes
// 128 contiguous bytes of a tile.  Everything after the integer Gram is f64;
// the result is the exact Gram up to f64 rounding (~1e-13 after centring).
//
// Work unit = (sample s, line range of <= 32768 lines); units are dealt to
// CTAs round-robin (static), so the summation order is fixed.
// Roles: warps 0-3 scan (per-band min for the clamp check and the column sums
// m_s, CUDA cores), warps 4-7 epilogue (TMEM byte Gram -> f64, one unit behind
// the tensor core thanks to a double-buffered accumulator), warp 8 TMA
// producer, warp 9 MMA issuer.  Only the lower triangle of the byte Gram is
// needed: windows wider than 128 bytes add one M=128 x N=(NW-128) MMA for the
// bottom-right block instead of a second full-width one.
#include <algorithm>
#include <type_traits>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tma.cuh"
#include "umma.cuh"

namespace skyrx {
using namespace umma;

// -DSKYRX_GR_PROFILE builds accumulate per-CTA wait cycles of each role
// (tools/gr_profile.py reads them through skyrx_gr_profile); compiled out otherwise
#ifdef SKYRX_GR_PROFILE
__device__ unsigned long long gr_prof[160][12];
#define GR_PW(idx, stmt)                                        \
  do {                                                          \
    const unsigned long long t0_ = clock64();                   \
    stmt;                                                       \
    gr_prof[blockIdx.x][idx] += clock64() - t0_;                \
  } while (0)
#else
#define GR_PW(idx, stmt) stmt
#endif

#ifndef GRX_L2PROMO  // experiment switch: the TMA boxes' L2 promotion
#define GRX_L2PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
// warps: 4 scan, 4 x kGrEpiGroups epilogue (group g takes every kGrEpiGroups-th pair of
// 16-column chunks of a unit's byte Gram), TMA, MMA.  Short units (a 249-line c2 chunk: two
// tiles per unit) are epilogue-bound (84 % of the kernel, tools/gr_profile.py), so the
// epilogue is split over three groups (1 / 2 / 3 / 4 groups: 124 / 101 / 97 / 103 us per chunk)
#ifndef GRX_EPI_GROUPS
#define GRX_EPI_GROUPS 3
#endif
constexpr int kGrEpiGroups = GRX_EPI_GROUPS;  // default; long units of the c4 shape take 2
constexpr int kGrWorkers = 128;   // scan threads (warps 0-3)
// EG epilogue groups: epilogue threads (warps 4..), then the TMA and MMA warps
constexpr int gr_epi(int eg) { return 128 * eg; }
constexpr int gr_threads(int eg) { return kGrWorkers + gr_epi(eg) + 64; }
// MMA issue form: -1 = per window class (below), 0 = lane 0 alone, 1 = whole warp + elected lane
#ifndef GRX_ELECT_MODE
#define GRX_ELECT_MODE -1
#endif
constexpr int kGrLb = 128;        // lines per tile (4 x K=32)
// TMA ring depth (stage = 128 lines x (128 + second-box) bytes) within the shared memory
// left beside the f64 accumulator: 8 stages, 5 for windows > 160 B, 2 for > 192 B
template <int NCH>
#ifndef GRX_STAGES
__host__ __device__ constexpr int gr_stages() { return NCH >= 13 ? 2 : (NCH >= 11 ? 5 : 8); }
#else  // experiment: ring depth for NCH <= 10 (with -DGRX_NO_QACC: TMA-stream tests only)
__host__ __device__ constexpr int gr_stages() { return NCH >= 13 ? 2 : (NCH >= 11 ? 5 : GRX_STAGES); }
#endif
constexpr int64_t kGrMaxUnitLines = 32768;

struct GramRawParams {
  const float* dark;
  const float* coeff;
  double ginv;
  double* part;       // per CTA: Sxx[B*B], Sx[B], n
  int32_t* flags;
  int64_t L;
  int32_t S, B;
  int64_t split_lines;  // lines per unit
  int32_t nsplit;
  int64_t units;        // all work items: regular units, then the tail's pieces
  // tail balancing: the S * nsplit regular units are dealt round-robin; the last,
  // partial round (rem units) is cut into tail_k pieces each, so every CTA ends with
  // at most one short piece instead of 24 CTAs running one whole extra unit
  int64_t units_main;   // regular units dealt in full rounds
  int32_t tail_k;       // pieces per leftover unit (1: no split)
  int64_t tail_lines;   // lines per piece (multiple of the tile)
  uint32_t* pixbits;     // bit (line * S + s): that pixel has a clamped value, or null
};

// idesc for kind::i8 with unsigned 8-bit operands, MN-major A and B, S32 accumulators
__host__ __device__ constexpr uint32_t idesc_u8_s32(int M, int N) {
  return (2u << 4) | (0u << 7) | (0u << 10) | (1u << 15) | (1u << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// TMEM columns per accumulator buffer: full-width block + the bottom-right block
// width of the second box (bytes 128.. of the window): 32, 64 or 128
template <int NCH>
__host__ __device__ constexpr uint32_t gr_w2b() {
  return NCH <= 8 ? 0u : (16 * NCH - 128 <= 32 ? 32u : (16 * NCH - 128 <= 64 ? 64u : 128u));
}
// windows of 129..160 bytes (the c4 shape, B = 57..72) take their column sums from the
// tensor core: the two small MMAs get a 32-column atom of ones appended to B (N = 64), so
// D[m][ones] = sum over lines of byte m, and the scan warps only track the minima
template <int NCH>
__host__ __device__ constexpr bool gr_ones() { return NCH > 8 && gr_w2b<NCH>() == 32u; }
template <int NCH>
__host__ __device__ constexpr int gr_bufcols() {
  return gr_ones<NCH>() ? 256 : ((16 * NCH + (NCH > 8 ? 16 * NCH - 128 : 0)) + 31) / 32 * 32;
}
template <int NCH>
#ifndef GRX_NBUF1
__host__ __device__ constexpr int gr_nbuf() { return 2 * gr_bufcols<NCH>() <= 512 ? 2 : 1; }
#else  // experiment: one accumulator (no MMA runs ahead of the epilogue loads)
__host__ __device__ constexpr int gr_nbuf() { return 1; }
#endif

// below(v, th): some halfword of v is below its threshold (max(v, t) != v)
__device__ __forceinline__ uint32_t gr_below(const uint4& v, const uint32_t (&th)[4]) {
  return (__vmaxu2(v.x, th[0]) ^ v.x) | (__vmaxu2(v.y, th[1]) ^ v.y) |
         (__vmaxu2(v.z, th[2]) ^ v.z) | (__vmaxu2(v.w, th[3]) ^ v.w);
}

// One scan thread's state for one 16-byte chunk of the window: running minima, column sums
// (windows whose sums do not come from the tensor core), clamp thresholds.
struct GrChunkScan {
  uint32_t tm[4];   // min(th, every count so far): differs from th once a count is below it
  uint32_t sm[8];   // column sums
  uint32_t th[4];   // r < th: the count calibrates to 0 (r < ceil(dark)); 0: never
  uint32_t always;  // a dark above every u16 count
  uint32_t hit;     // the unit held a value below dark in this chunk
};

// The scan of NL lines of one chunk, all loads in flight at once: line j of the thread sits
// at addr + j * STRIDE (the thread's lines share their swizzle phase, so the offsets are
// immediates).  The scan warps sit on the stage-release path (a stage is freed by the MMA
// commit AND the 128 scan arrivals), so their instruction count per tile is kernel time:
// the round-2 loop (runtime trip count: a division per tile, an address computation and a
// shared-memory latency per four lines) cost 7 % of the kernel.  The running minima start
// at the clamp thresholds, so "a count below its dark" is four XORs per tile (tm != th);
// then gr_mark_chunk tests the thread's lines one by one.
// The rare path, out of line so that it costs the scan loop no registers: the thread's lines
// (still in shared memory) are tested one by one and the pixels holding a value below dark
// get their bit.  pix0: pixel index of the tile's line 0 at this sample.
template <int NL, uint32_t STRIDE>
__device__ __noinline__ void gr_mark_chunk(uint32_t addr, int line0, int lstep, int valid,
                                           uint32_t t0, uint32_t t1, uint32_t t2, uint32_t t3,
                                           uint32_t always, int64_t pix0, int S,
                                           uint32_t* __restrict__ pixbits) {
  const uint32_t th[4] = {t0, t1, t2, t3};
  uint4 v[NL];
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    v[j] = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
    if (line0 + j * lstep < valid) v[j] = ld_shared_v4(addr + j * STRIDE);
  }
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    if (line0 + j * lstep < valid && (always | gr_below(v[j], th))) {
      const int64_t pix = pix0 + (int64_t)(line0 + j * lstep) * S;
      atomicOr(pixbits + (pix >> 5), 1u << (pix & 31));
    }
  }
}

// the three steps of a chunk's scan, separate so that a thread's two chunks (box 0 and the
// second box) have all their loads in flight before either is reduced or tested: one
// shared-memory latency per tile instead of two
template <int NL, uint32_t STRIDE, bool FULL>
__device__ __forceinline__ void gr_scan_load(uint4 (&v)[NL], uint32_t addr, int line0, int lstep,
                                             int valid) {
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    v[j] = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
    if (FULL || line0 + j * lstep < valid) v[j] = ld_shared_v4(addr + j * STRIDE);
  }
}
template <int NL, bool SUMS, bool FULL>
__device__ __forceinline__ void gr_scan_acc(GrChunkScan& c, const uint4 (&v)[NL], int line0,
                                            int lstep, int valid) {
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    c.tm[0] = __vminu2(c.tm[0], v[j].x), c.tm[1] = __vminu2(c.tm[1], v[j].y);
    c.tm[2] = __vminu2(c.tm[2], v[j].z), c.tm[3] = __vminu2(c.tm[3], v[j].w);
    if (SUMS && (FULL || line0 + j * lstep < valid)) {
      // one IDP.2A per halfword: sm += lo16(v) * 1 + hi16(v) * 0 (or the hi half)
      c.sm[0] = __dp2a_lo(v[j].x, 0x0001u, c.sm[0]), c.sm[1] = __dp2a_lo(v[j].x, 0x0100u, c.sm[1]);
      c.sm[2] = __dp2a_lo(v[j].y, 0x0001u, c.sm[2]), c.sm[3] = __dp2a_lo(v[j].y, 0x0100u, c.sm[3]);
      c.sm[4] = __dp2a_lo(v[j].z, 0x0001u, c.sm[4]), c.sm[5] = __dp2a_lo(v[j].z, 0x0100u, c.sm[5]);
      c.sm[6] = __dp2a_lo(v[j].w, 0x0001u, c.sm[6]), c.sm[7] = __dp2a_lo(v[j].w, 0x0100u, c.sm[7]);
    }
  }
}
__device__ __forceinline__ uint32_t gr_scan_test(const GrChunkScan& c) {
  return c.always | (c.tm[0] ^ c.th[0]) | (c.tm[1] ^ c.th[1]) | (c.tm[2] ^ c.th[2]) |
         (c.tm[3] ^ c.th[3]);
}
template <int NL, uint32_t STRIDE>
__device__ __forceinline__ void gr_scan_hit(GrChunkScan& c, uint32_t addr, int line0, int lstep,
                                            int valid, uint32_t* pixbits, int64_t pix0, int S) {
  if (pixbits != nullptr)
    gr_mark_chunk<NL, STRIDE>(addr, line0, lstep, valid, c.th[0], c.th[1], c.th[2], c.th[3],
                              c.always, pix0, S, pixbits);
  // the minima start afresh, so that later clean tiles skip the per-line test
  c.hit = 1u;
#pragma unroll
  for (int i = 0; i < 4; ++i) c.tm[i] = c.th[i];
}

template <int NCH, int EG = kGrEpiGroups>
__global__ void __launch_bounds__(gr_threads(EG), 1) gram_raw_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                 const __grid_constant__ CUtensorMap tmap1,
                                                                 GramRawParams p) {
  constexpr int kGrStages = gr_stages<NCH>();
  constexpr int kGrEpi = gr_epi(EG);
  constexpr int kGrTmaWarp = (kGrWorkers + kGrEpi) / 32, kGrMmaWarp = kGrTmaWarp + 1;
  constexpr int NW = 16 * NCH;                    // window bytes = MMA N
  constexpr bool TWO_M = NCH > 8;                 // rows 128.. need a second M=128 MMA
  constexpr int N2 = TWO_M ? NW - 128 : 0;        // ... only over columns 128..NW-1
  // a tile = a box of [128 window bytes][Lb lines], 128B-swizzled by TMA (the
  // canonical MN-major SWIZZLE_128B UMMA layout, SBO = 8 lines), plus for wider
  // windows a box of the W2B bytes past 128 in the matching 32/64/128B swizzle
  constexpr uint32_t ATOM = kGrLb * 128u;
  constexpr uint32_t W2B = gr_w2b<NCH>();
  constexpr uint32_t ATOM1 = TWO_M ? kGrLb * W2B : 0u;
  constexpr uint32_t STAGE = ATOM + ATOM1;
  constexpr uint32_t LT1 = W2B == 32 ? 6u : (W2B == 64 ? 4u : 2u);
  // NQ1: 16-byte chunks per line of the second box
  constexpr int NQ1 = W2B > 0 ? (int)W2B / 16 : 1;
  constexpr int BUFC = gr_bufcols<NCH>();
  constexpr bool ONES = gr_ones<NCH>();
  constexpr uint32_t P1OFF = ONES ? 192u : (uint32_t)NW;  // TMEM column of the part-1 block
  constexpr int NBUF = gr_nbuf<NCH>();
  extern __shared__ __align__(1024) uint8_t sm[];
  const int B = p.B;
  uint8_t* stages = sm;
#ifndef GRX_NO_QACC
  double* qacc = reinterpret_cast<double*>(stages + kGrStages * STAGE);
#else  // experiment: no f64 accumulator in shared memory (aliases the ring; timing only)
  double* qacc = reinterpret_cast<double*>(stages + kGrStages * STAGE) - (B * B + B);
#endif
  double* sacc = qacc + B * B;
  uint8_t* ones = reinterpret_cast<uint8_t*>(sacc + B);      // ONES: [128 lines][32 B] of 1
  uint32_t* smin = reinterpret_cast<uint32_t*>(ones + (ONES ? kGrLb * 32 : 0));  // [thread][4]
  uint32_t* ssum = smin + kGrWorkers * 4;                    // [scan thread][8] (not ONES)
  uint32_t* smin1 = ssum + (ONES ? 0 : kGrWorkers * 8);      // the same for the second box
  uint32_t* ssum1 = smin1 + (TWO_M ? kGrWorkers * 4 : 0);
  uint32_t* minv = ssum1 + (TWO_M && !ONES ? kGrWorkers * 8 : 0);  // [2][NCH*8]
  uint32_t* sumv = minv + 2 * NCH * 8;                       // [2][NCH*8]
  double* bandC = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(sumv + 2 * NCH * 8) + 7) & ~uintptr_t(7));  // [B] per unit
  double* bandD = bandC + B;
  double* bandS = bandD + B;
  uint64_t* bars = reinterpret_cast<uint64_t*>(bandS + B);
  uint64_t* full = bars;
  uint64_t* empty = full + kGrStages;
  uint64_t* acc_full = empty + kGrStages;   // [NBUF]
  uint64_t* acc_empty = acc_full + 2;       // [NBUF]
  uint64_t* scan_full = acc_empty + 2;      // [2] unit's min / sums published
  uint64_t* scan_empty = scan_full + 2;     // [2] ... consumed by the epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(scan_empty + 2);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  // round-robin units: at any moment the CTAs work on neighbouring samples of
  // the same lines, so the 16-B chunks two windows share are fetched once (L2)
  const int64_t u0 = blockIdx.x;
  const int64_t u1 = p.units;
  const int64_t ustep = gridDim.x;

  if (tid == 0) {
    for (int s = 0; s < kGrStages; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], kGrWorkers + 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1), mbar_init(&acc_empty[b], kGrEpi);
      mbar_init(&scan_full[b], 1), mbar_init(&scan_empty[b], kGrEpi);
    }
    fence_mbar_init();
  }
  if (warp == kGrMmaWarp) tmem_alloc(tmem_slot, 512);
  // bit 8: this cube's clamp check ran (bit 4 would report a value below dark)
  if (blockIdx.x == 0 && tid == 0) atomicOr(p.flags, 8);
  for (int e = tid; e < B * B + B; e += blockDim.x) qacc[e] = 0.0;
  if (ONES) {
    for (int e = tid; e < kGrLb * 8; e += blockDim.x)
      reinterpret_cast<uint32_t*>(ones)[e] = 0x01010101u;
    fence_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // 32-bit shared addresses for the per-tile barriers and loads (no per-tile conversion)
  const uint32_t full32 = smem_u32(full), empty32 = smem_u32(empty), stages32 = smem_u32(stages);
#ifdef SKYRX_GR_PROFILE
  const unsigned long long kt0 = clock64();
#endif

  auto unit_geom = [&](int64_t u, int& s, int64_t& l0, int64_t& nl) {
    const int64_t ur = u < p.units_main ? u : p.units_main + (u - p.units_main) / p.tail_k;
    s = (int)(ur % p.S);
    const int64_t sp = ur / p.S;
    l0 = sp * p.split_lines;
    nl = p.L - l0 < p.split_lines ? p.L - l0 : p.split_lines;
    if (u >= p.units_main) {  // a piece of a leftover unit
      const int64_t piece = (u - p.units_main) % p.tail_k;
      const int64_t a = piece * p.tail_lines;
      const int64_t b = a + p.tail_lines < nl ? a + p.tail_lines : nl;
      l0 += a;
      nl = b > a ? b - a : 0;
    }
  };

  if (warp == kGrTmaWarp) {
    if ((tid & 31) == 0) {  // ------------------------------------------- TMA producer
      int t = 0;
      for (int64_t u = u0; u < u1; u += ustep) {
        int s;
        int64_t l0, nl;
        unit_geom(u, s, l0, nl);
        const int c0 = (int)(((int64_t)s * B * 2) >> 4);
        const int ntile = (int)((nl + kGrLb - 1) / kGrLb);
        for (int k = 0; k < ntile; ++k, ++t) {
          const int st = t % kGrStages;
          GR_PW(0, mbar_wait(empty32 + 8 * st, ((t / kGrStages) & 1) ^ 1));
          mbar_arrive_expect_tx(&full[st], STAGE);
          tma_load_2d(stages + st * STAGE, &tmap, 16 * c0, (int)(l0 + (int64_t)k * kGrLb),
                      &full[st]);
          if (TWO_M)
            tma_load_2d(stages + st * STAGE + ATOM, &tmap1, 16 * c0 + 128,
                        (int)(l0 + (int64_t)k * kGrLb), &full[st]);
        }
      }
    }
  } else if (warp == kGrMmaWarp) {
    // ------------------------------------------------------------------- MMA issuer
    // Two issue forms, chosen per window class by measurement (tools/time_gr_direct.py,
    // session 6, after the scan rewrite): the whole warp converged with one elected lane
    // issuing is faster for the three-MMA ONES windows (c4 strip 0.487 -> 0.442 ms), lane 0
    // alone for the others (B = 40 / 96 / 128: 0.390 / 0.558 / 1.015 against 0.400 / 0.610 /
    // 1.042 ms).  (Before the scan rewrite lane 0 was faster for the c4 shape too.)
    constexpr bool ELECT = GRX_ELECT_MODE < 0 ? ONES : (GRX_ELECT_MODE != 0);
    if (ELECT || (tid & 31) == 0) {
      constexpr uint32_t id = idesc_u8_s32(128, TWO_M ? 128 : NW);
      constexpr uint32_t id2 = idesc_u8_s32(128, ONES ? 64 : (N2 > 0 ? N2 : 16));
      int t = 0, unit = 0;
      for (int64_t u = u0; u < u1; u += ustep, ++unit) {
        int s;
        int64_t l0, nl;
        unit_geom(u, s, l0, nl);
        const int ntile = (int)((nl + kGrLb - 1) / kGrLb);
        const int buf = NBUF == 2 ? (unit & 1) : 0;
        const int use = NBUF == 2 ? (unit >> 1) : unit;
        GR_PW(1, mbar_wait(&acc_empty[buf], (use & 1) ^ 1));
        tc_fence_after();
        const uint32_t d = tmem + buf * BUFC;
        for (int k = 0; k < ntile; ++k, ++t) {
          const int st = t % kGrStages;
          GR_PW(2, mbar_wait(full32 + 8 * st, (t / kGrStages) & 1));
          tc_fence_after();
          const uint8_t* base = stages + st * STAGE;
          if (!ELECT || elect_one()) {
#pragma unroll
          for (int ks = 0; ks < kGrLb / 32; ++ks) {
            const uint32_t acc = (k > 0 || ks > 0) ? 1u : 0u;
            const uint8_t* kb = base + ks * 4096;  // 32 lines = 4 swizzle atoms of 8 x 128 B
            const uint64_t d0 = smem_desc_sw128(kb, ATOM, 1024);
#ifndef GRX_NO_M1  // ablation switches (tools/build_gr_var.sh), off in the product
            mma_i8(d, d0, d0, id, acc);
#endif
            if (TWO_M) {
              // bytes 128.. in their own (narrower) swizzle: columns 128..NW-1 of rows
              // 0..127, and rows 128..NW-1 x columns 128..NW-1 (the rest is the
              // transpose); the 128-row A of the second MMA re-reads its one atom
              // (LBO 0): rows >= NW-128 are never used
              const uint8_t* b1 = base + ATOM + ks * 32 * W2B;
              const uint64_t d1 = smem_desc_swz(b1, 0, 8 * W2B, LT1);
              // ONES: B = [bytes 128..159 | ones] as two SW32 atoms, LBO = their distance
              const uint64_t d1b =
                  ONES ? smem_desc_swz(b1, (uint32_t)(ones + ks * 32 * W2B - b1), 8 * W2B, LT1)
                       : d1;
#ifndef GRX_NO_M23
              mma_i8(d + 128, d0, d1b, id2, acc);
              mma_i8(d + P1OFF, d1, d1b, id2, acc);
#endif
            }
          }
          mma_commit(&empty[st]);
          }
          if (ELECT) __syncwarp();
        }
        if (!ELECT || elect_one()) mma_commit(&acc_full[buf]);
        if (ELECT) __syncwarp();
      }
    }
  } else if (warp < 4) {  // ---------------------------------------------- scan
    // every thread scans one chunk of box 0 (chunk tid & 7, lines (tid >> 3) + 16 j, j < 8)
    // and one of the second box (chunk 8 + tid % NQ1, lines tid / NQ1 + (128 / NQ1) j,
    // j < NQ1): a quarter-warp reads 128 contiguous bytes (conflict-free), and a thread's
    // lines share their swizzle phase, so their addresses differ by immediates
    const int q0 = tid & 7, ls0 = tid >> 3;
    const int q1 = tid % NQ1, ls1 = tid / NQ1;
    constexpr int LSTEP1 = kGrLb / NQ1;
    const uint32_t off0 = ls0 * 128u + ((uint32_t)(q0 ^ (ls0 & 7)) << 4);
    const uint32_t off1 =
        ATOM + ls1 * W2B + ((uint32_t)(q1 ^ (int)(((uint32_t)ls1 * W2B >> 7) & (NQ1 - 1))) << 4);
    const bool scan0 = q0 < NCH;
    const bool scan1 = TWO_M && 8 + q1 < NCH;
    uint32_t* const pixbits = p.pixbits;  // null: no room for the bitmap, detection only
    // dark levels of a chunk's 8 window halfwords at sample s (0 outside the sample's bands):
    // a count r calibrates to 0 iff (float)r < dark, i.e. r < ceil(dark) (never for
    // dark <= 0 or NaN; always for dark > 65535).  Fetched one unit ahead, before the
    // per-unit reduction, so that the loads' latency is off the first tile's scan
    auto fetch_dark = [&](float (&dk)[8], int s, int chunk, bool on) {
      const int off2 = (int)((((int64_t)s * B * 2) & 15) >> 1);
      const float* drow = p.dark + (int64_t)s * B;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int b = 8 * chunk + i - off2;
        dk[i] = (on && b >= 0 && b < B) ? __ldg(drow + b) : 0.0f;
      }
    };
    float dk0[8], dk1[8];
    if (u0 < u1) {
      int s;
      int64_t l0, nl;
      unit_geom(u0, s, l0, nl);
      fetch_dark(dk0, s, q0, scan0);
      if (TWO_M) fetch_dark(dk1, s, 8 + q1, scan1);
    }
    int t = 0, unit = 0;
    for (int64_t u = u0; u < u1; u += ustep, ++unit) {
      int s;
      int64_t l0, nl;
      unit_geom(u, s, l0, nl);
      const int ntile = (int)((nl + kGrLb - 1) / kGrLb);
      const int last_valid = (int)(nl - (int64_t)(ntile - 1) * kGrLb);  // lines of the last tile
      GrChunkScan c0, c1;
      auto begin = [&](GrChunkScan& c, const float (&dk)[8]) {
#pragma unroll
        for (int i = 0; i < 4; ++i) c.th[i] = 0u;
#pragma unroll
        for (int i = 0; i < 8; ++i) c.sm[i] = 0u;
        c.always = 0u, c.hit = 0u;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          uint32_t t16 = 0u;
          if (dk[i] > 65535.0f) c.always = 1u;
          else if (dk[i] > 0.0f) t16 = (uint32_t)ceilf(dk[i]);
          c.th[i >> 1] |= t16 << (16 * (i & 1));
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) c.tm[i] = c.th[i];
      };
      begin(c0, dk0);
      if (TWO_M) begin(c1, dk1);
      for (int k = 0; k < ntile; ++k, ++t) {
        const int st = t % kGrStages;
        if (tid == 0) GR_PW(3, mbar_wait(full32 + 8 * st, (t / kGrStages) & 1));
        else mbar_wait(full32 + 8 * st, (t / kGrStages) & 1);
#ifndef GRX_NO_SCAN
        {
          const int valid = k == ntile - 1 ? last_valid : kGrLb;
          const uint32_t base = stages32 + st * STAGE;
          auto scan_tile = [&](auto full_tag) {
            constexpr bool FULL = decltype(full_tag)::value;
            uint4 v0[8], v1[NQ1];
            // (wide second boxes: one box after the other, 16 loads in flight would spill)
            if (scan0) gr_scan_load<8, 2048u, FULL>(v0, base + off0, ls0, 16, valid);
            if (NQ1 > 2 && scan0) gr_scan_acc<8, !ONES, FULL>(c0, v0, ls0, 16, valid);
            if (TWO_M && scan1) gr_scan_load<NQ1, 2048u, FULL>(v1, base + off1, ls1, LSTEP1, valid);
            if (NQ1 <= 2 && scan0) gr_scan_acc<8, !ONES, FULL>(c0, v0, ls0, 16, valid);
            if (TWO_M && scan1) gr_scan_acc<NQ1, !ONES, FULL>(c1, v1, ls1, LSTEP1, valid);
          };
          if (valid == kGrLb) scan_tile(std::true_type{});
          else scan_tile(std::false_type{});
          // a count below its dark (rare): its pixels are marked for clamp_fix_kernel
          const uint32_t x0 = scan0 ? gr_scan_test(c0) : 0u;
          const uint32_t x1 = (TWO_M && scan1) ? gr_scan_test(c1) : 0u;
          if (x0 | x1) {
            const int64_t pix0 = (l0 + (int64_t)k * kGrLb) * p.S + s;
            if (x0) gr_scan_hit<8, 2048u>(c0, base + off0, ls0, 16, valid, pixbits, pix0, p.S);
            if (TWO_M && x1)
              gr_scan_hit<NQ1, 2048u>(c1, base + off1, ls1, LSTEP1, valid, pixbits, pix0, p.S);
          }
        }
#endif
        // (one arrival per thread: a __syncwarp + lane-0 arrival measured slower, 0.488 ->
        // 0.493 ms per c4 strip: the warp then waits for its slowest lane before any release)
        mbar_arrive(empty32 + 8 * st);
      }
      if (u + ustep < u1) {  // the next unit's dark levels, in flight during the reduction
        int sn;
        int64_t l0n, nln;
        unit_geom(u + ustep, sn, l0n, nln);
        fetch_dark(dk0, sn, q0, scan0);
        if (TWO_M) fetch_dark(dk1, sn, 8 + q1, scan1);
      }
      // per-unit reduction of the scans (fixed member order per chunk) into buffer ub; a
      // chunk that held a value below dark publishes minima of 0 (below any dark that can
      // clamp), the others 0xffff
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        smin[tid * 4 + i] = c0.hit ? 0u : 0xffffffffu;
        if (TWO_M) smin1[tid * 4 + i] = c1.hit ? 0u : 0xffffffffu;
      }
      if (!ONES) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          ssum[tid * 8 + i] = c0.sm[i];
          if (TWO_M) ssum1[tid * 8 + i] = c1.sm[i];
        }
      }
      const int ub = unit & 1;
      mbar_wait(&scan_empty[ub], ((unit >> 1) & 1) ^ 1);
      asm volatile("bar.sync 1, %0;" ::"n"(kGrWorkers) : "memory");
      if (tid < NCH * 8) {
        const int cc = tid >> 3, qq = tid & 7;
        // members of chunk cc: box 0 -> threads cc + 8 m (m < 16); second box -> threads
        // (cc - 8) + NQ1 m (m < 128 / NQ1)
        const bool b1 = cc >= 8;
        const uint32_t* pm = b1 ? smin1 : smin;
        const uint32_t* ps = b1 ? ssum1 : ssum;
        const int first = b1 ? cc - 8 : cc;
        const int stride = b1 ? NQ1 : 8;
        const int nmem = b1 ? kGrWorkers / NQ1 : kGrWorkers / 8;
        uint32_t mv = 0xffffu, sv = 0;
        for (int m = 0; m < nmem; ++m) {
          const int mt = first + stride * m;
          const uint32_t w = pm[mt * 4 + (qq >> 1)];
          mv = min(mv, (qq & 1) ? (w >> 16) : (w & 0xffffu));
          if (!ONES) sv += ps[mt * 8 + qq];
        }
        minv[ub * NCH * 8 + tid] = mv;
        sumv[ub * NCH * 8 + tid] = sv;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kGrWorkers) : "memory");
      if (tid == 0) mbar_arrive(&scan_full[ub]);
    }
  } else {  // ------------------------------------------------------- epilogue (warps 4 .. 4 + 4G)
    const int te = (tid - kGrWorkers) & 127;  // TMEM lane = byte row of the Gram
    const int eg = (tid - kGrWorkers) >> 7;   // epilogue group
    const int we = warp & 3;
    const uint32_t tq = warp_uniform(tmem + ((uint32_t)(32 * we) << 16));  // lane quarter
    int unit = 0;
    for (int64_t u = u0; u < u1; u += ustep, ++unit) {
      int s;
      int64_t l0, nl;
      unit_geom(u, s, l0, nl);
      const int buf = NBUF == 2 ? (unit & 1) : 0;
      const int use = NBUF == 2 ? (unit >> 1) : unit;
      const int ub = unit & 1;
      if (tid == kGrWorkers) GR_PW(4, mbar_wait(&scan_full[ub], (unit >> 1) & 1));
      else mbar_wait(&scan_full[ub], (unit >> 1) & 1);
      if (tid == kGrWorkers) GR_PW(5, mbar_wait(&acc_full[buf], use & 1));
      else mbar_wait(&acc_full[buf], use & 1);
      tc_fence_after();
      if (nl == 0) {  // an empty tail piece: no tiles, nothing accumulated
        tc_fence_before();
        mbar_arrive(&acc_empty[buf]);
        mbar_arrive(&scan_empty[ub]);
        continue;
      }
#ifdef SKYRX_GR_PROFILE
      const unsigned long long et0 = clock64();
#endif
      const uint32_t* mnv = minv + ub * NCH * 8;
      const uint32_t* smv = sumv + ub * NCH * 8;
      const int off = (int)(((int64_t)s * B * 2) & 15);
      const double Lu = (double)nl;
      const float* drow = p.dark + (int64_t)s * B;
      const float* crow = p.coeff + (int64_t)s * B;
      bool clamp = false;
      // this unit's per-band terms, once, for every epilogue thread
      if (ONES && eg == 0) {  // band sums = 256 sum(hi) + sum(lo) from the ones columns
#pragma unroll
        for (int part = 0; part < 2; ++part) {
          if (part == 1 && 128 + 32 * we >= off + 2 * B) continue;  // warp-uniform
          uint32_t sv[16];
          tmem_ld16(tq + buf * BUFC + (part ? 224u : 160u), sv);
          tmem_ld_wait();
          const uint32_t partner = __shfl_xor_sync(0xffffffffu, sv[0], 1);
          const int rel = 128 * part + te - off;
          if (rel >= 0 && rel < 2 * B && (rel & 1) == 0)
            bandS[rel >> 1] = 256.0 * (double)partner + (double)sv[0];
        }
      }
      for (int bb = tid - kGrWorkers; bb < B; bb += kGrEpi) {
        bandC[bb] = (double)crow[bb] * p.ginv;
        bandD[bb] = (double)drow[bb];
        if (!ONES) bandS[bb] = (double)smv[(off >> 1) + bb];
        clamp |= (float)mnv[(off >> 1) + bb] < drow[bb];
      }
      asm volatile("bar.sync 2, %0;" ::"n"(kGrEpi) : "memory");
#ifdef SKYRX_GR_PROFILE
      const unsigned long long et1 = clock64();
      if (tid == kGrWorkers) gr_prof[blockIdx.x][8] += et1 - et0;
#endif
#pragma unroll
      for (int part = 0; part < (TWO_M ? 2 : 1); ++part) {
        if (part == 1 && 128 + 32 * we >= off + 2 * B) continue;  // warp-uniform
#ifdef GRX_NO_EPI
        continue;
#endif
        const int m = 128 * part + te;
        const int rel = m - off;
        const bool in_band = rel >= 0 && rel < 2 * B;
        const int hi = rel & 1;    // 0: this row is band b's lo byte, 1: its hi byte
        const int b = rel >> 1;
        double Cb = 0.0, db = 0.0, Sb = 0.0;
        if (in_band) Cb = bandC[b], db = bandD[b], Sb = bandS[b];
        // part 0: byte columns 0..NW-1 of the full-width block; part 1: columns 128..NW-1
        const uint32_t taddr = tq + buf * BUFC + (part ? P1OFF : 0);
        const int cc0 = part ? 8 : 0;
        // chunks this warp's rows need (warp-uniform): the lower triangle reaches byte
        // column 128 part + 32 we + 31; part-0 rows also own every column past byte 128
        const int cmax = 128 * part + 32 * we + 31;
        auto needed = [&](int cc) {
          return cc < NCH && (cc * 16 <= cmax || (part == 0 && TWO_M && cc >= 8));
        };
        // two chunks per TMEM wait: the loads queue behind the next unit's MMAs
        for (int cc = cc0 + 2 * eg; cc < NCH; cc += 2 * EG) {
          const bool n0 = needed(cc), n1 = needed(cc + 1);
          if (!n0 && !n1) continue;
          uint32_t v2[32];
          if (n0) tmem_ld16(taddr + (cc - cc0) * 16, v2);
          if (n1) tmem_ld16(taddr + (cc + 1 - cc0) * 16, v2 + 16);
          tmem_ld_wait();
#pragma unroll
          for (int h = 0; h < 2; ++h) {
          if (!(h ? n1 : n0)) continue;
          const int c = cc + h;
          const uint32_t* v = v2 + 16 * h;
          uint32_t pv[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) pv[q] = __shfl_xor_sync(0xffffffffu, v[q], 1);
          if (in_band) {
            // the lo-byte row of the pair takes the even band columns, the hi-byte row
            // the odd ones; each has both rows (own + partner) of the pair
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if ((i & 1) != hi) continue;
              const int reln = c * 16 + 2 * i - off;
              if (reln < 0 || reln >= 2 * B) continue;
              const int b2 = reln >> 1;
              // lower triangle (b2 <= b) from this row pair; a part-0 pair also owns the
              // (b2 > b) entries whose columns lie past byte 128: their part-1 rows
              // only see columns >= 128
              const bool mine = b2 <= b || (part == 0 && TWO_M && c >= 8);
              if (!mine) continue;
              // H_b H_b2, H_b L_b2 + L_b H_b2, L_b L_b2 from (own, partner) rows
              const uint32_t hh = hi ? v[2 * i + 1] : pv[2 * i + 1];
              const uint32_t hl = hi ? v[2 * i] : pv[2 * i];
              const uint32_t lh = hi ? pv[2 * i + 1] : v[2 * i + 1];
              const uint32_t ll = hi ? pv[2 * i] : v[2 * i];
              // exact integer G entry (< 2^48), to f64 through the 2^52 exponent trick
              const uint64_t gi = ((uint64_t)hh << 16) + (((uint64_t)hl + lh) << 8) + ll;
              const double gv = __hiloint2double(0x43300000 | (int)(gi >> 32), (int)(uint32_t)gi) -
                                4503599627370496.0;
              const double C2 = bandC[b2], d2 = bandD[b2], S2 = bandS[b2];
              const double xx = gv - db * S2 - Sb * d2 + Lu * db * d2;
              const int e = b2 <= b ? b * B + b2 : b2 * B + b;
              qacc[e] += Cb * C2 * xx;
            }
          }
          }
        }
        if (in_band && !hi && eg == 0) sacc[b] += Cb * (Sb - Lu * db);
#ifdef SKYRX_GR_PROFILE
        if (tid == kGrWorkers) gr_prof[blockIdx.x][9 + part] += clock64() - et1;
#endif
      }
      // the band terms are rewritten by the next unit only after every thread is done here
      asm volatile("bar.sync 2, %0;" ::"n"(kGrEpi) : "memory");
#ifdef SKYRX_GR_PROFILE
      if (tid == kGrWorkers) gr_prof[blockIdx.x][6] += clock64() - et0;
#endif
      if (clamp) atomicOr(p.flags, 4);
      tc_fence_before();
      mbar_arrive(&acc_empty[buf]);
      mbar_arrive(&scan_empty[ub]);
    }
  }
  // per-CTA partial: Sxx (lower triangle), Sx, n
  __syncthreads();
  if (tid < kGrWorkers) {
    double* out = p.part + (size_t)blockIdx.x * (B * B + B + 1);
    for (int e = tid; e < B * B + B; e += kGrWorkers) out[e] = qacc[e];
    if (tid == 0) {
      double n = 0.0;
      for (int64_t u = u0; u < u1; u += ustep) {
        int s;
        int64_t l0, nl;
        unit_geom(u, s, l0, nl);
        n += (double)nl;
      }
      out[B * B + B] = n;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
#ifdef SKYRX_GR_PROFILE
  if (tid == 0) gr_prof[blockIdx.x][7] += clock64() - kt0;
#endif
  if (warp == kGrMmaWarp) tmem_dealloc(tmem, 512);
}

#ifdef SKYRX_GR_PROFILE
extern "C" __attribute__((visibility("default"))) int skyrx_gr_profile(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, gr_prof, sizeof(gr_prof));
}
#endif

// Deterministic reduction of the per-CTA partials [Sxx | Sx | n]: a block owns 32
// elements (one per lane); its 8 warps sum fixed, contiguous slices of the
// partials in order, then warp 0 adds the 8 slice sums in order.
constexpr int kSumBatch = 19;  // ceil(148 / 8): a warp's slice of the per-CTA partials
__device__ __forceinline__ double part_slice_sum(const double* __restrict__ part, int nparts,
                                                 int stride, int e, int w) {
  const int per = (nparts + 7) / 8;
  const int c0 = w * per, c1 = min(nparts, c0 + per);
  double acc = 0.0;
  if (per <= kSumBatch) {
    // every load of the slice in flight at once, then the same in-order sum
    double v[kSumBatch];
#pragma unroll
    for (int k = 0; k < kSumBatch; ++k)
      v[k] = c0 + k < c1 ? __ldcg(part + (size_t)(c0 + k) * stride + e) : 0.0;
#pragma unroll
    for (int k = 0; k < kSumBatch; ++k)
      if (c0 + k < c1) acc += v[k];
  } else {
    for (int cb = c0; cb < c1; cb += kSumBatch) {  // the same in-order sum, in batches
      double v[kSumBatch];
#pragma unroll
      for (int k = 0; k < kSumBatch; ++k)
        v[k] = cb + k < c1 ? __ldcg(part + (size_t)(cb + k) * stride + e) : 0.0;
#pragma unroll
      for (int k = 0; k < kSumBatch; ++k)
        if (cb + k < c1) acc += v[k];
    }
  }
  return acc;
}

// out = sum of the nparts partials (fixed order); plus, when flags says the clamp
// fix-up ran (256), the sum of its nfix partials (same order rule), added last
__global__ void __launch_bounds__(256) gram_raw_sum_kernel(const double* __restrict__ part,
                                                           int nparts, int stride,
                                                           double* __restrict__ out,
                                                           const double* __restrict__ fix,
                                                           int nfix,
                                                           const int32_t* __restrict__ flags) {
  __shared__ double red[8][32];
  __shared__ double red2[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + lane;
  const bool fixed = fix != nullptr && flags != nullptr && (__ldcg(flags) & 256);
  red[w][lane] = e < stride ? part_slice_sum(part, nparts, stride, e, w) : 0.0;
  red2[w][lane] = (fixed && e < stride) ? part_slice_sum(fix, nfix, stride, e, w) : 0.0;
  __syncthreads();
  if (w == 0 && e < stride) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += red[k][lane];
    if (fixed) {
      double t2 = 0.0;
      for (int k = 0; k < 8; ++k) t2 += red2[k][lane];
      t += t2;
    }
    out[e] = t;
  }
}

// moments about the shift c: s = Sx - n c, Q = Sxx - c Sx^T - Sx c^T + n c c^T.
// own: c is not given but chosen here, c = f32(Sx / n) (written to shift): the sums
// are exact integer Grams calibrated in f64, so any c near the mean centres them to
// ~1e-13, and the separate shift pass over the cube is not needed
__global__ void gram_raw_center_kernel(const double* __restrict__ tot, int B,
                                       double* __restrict__ shift, int own,
                                       double* __restrict__ moments) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  const double* sx = tot + B * B;
  const double n = tot[B * B + B];
  auto c_of = [&](int i) -> double {
    return own ? (n > 0.0 ? (double)(float)(sx[i] / n) : 0.0) : shift[i];
  };
  if (e < B * B) {
    const int i = e / B, j = e - i * B;
    if (j > i) return;
    const double ci = c_of(i), cj = c_of(j);
    const double q = tot[i * B + j] - ci * sx[j] - sx[i] * cj + n * ci * cj;
    moments[1 + B + (size_t)i * B + j] = q;
    moments[1 + B + (size_t)j * B + i] = q;
  } else if (e < B * B + B) {
    const int i = e - B * B;
    const double ci = c_of(i);
    moments[1 + i] = sx[i] - n * ci;
    if (own) shift[i] = ci;
  } else if (e == B * B + B) {
    moments[0] = n;
  }
}

// ------------------------------------------------------------------ clamp fix-up
// A raw count below its dark level calibrates to 0 (calibrate.py:99, max(r - d, 0)),
// which breaks the raw-byte algebra x = C (r - d) the Gram above relies on.  Instead of
// redoing the cube in f64 (round 1: ~20x the fast path at c4), the clamped pixels'
// exact corrections are added to the uncentred sums: with x the unclamped and x' the
// true radiance (x'_b = 0 where r_b < d_b), dx = x' - x is -x on the clamped bands and
//     sum x' x'^T = sum x x^T + sum (x dx^T + dx x^T + dx dx^T),   sum x' = sum x + sum dx.
// The scan warps of gram_raw_kernel mark the pixels: a thread whose tile minima fall below
// its thresholds rescans its part of the tile (still in shared memory) and sets bit
// (line * S + s) of a pixel bitmap for every pixel with a value below dark (atomicOr:
// order-free).  Round 2 had a separate marking launch that streamed the cube again (355 us
// of the 0.01 %-sub-dark c4 strip).  Then, a no-op (one flags read per CTA) when nothing
// clamped:
//  clamp_fix_kernel   CTA c walks a fixed contiguous range of the bitmap in pixel order,
//                     stages the clamped pixels 16 at a time and adds, pixel by pixel,
//                     only the row / column of each clamped band into a shared-memory
//                     triangle (thread t takes entry (t, c)): a deterministic per-CTA
//                     partial, joined to the Gram partials in gram_raw_sum_kernel's
//                     fixed-order sum.
constexpr int kFixThreads = 256;
#ifndef GRX_FIX_BATCH
#define GRX_FIX_BATCH 16
#endif
#ifndef GRX_FIX_PER_SM
#define GRX_FIX_PER_SM 5
#endif
constexpr int kFixBatch = GRX_FIX_BATCH;  // clamped pixels staged per round
// clamp_fix CTAs: the per-pixel chain (one barrier per clamped pixel, B threads busy) is
// latency-bound, so five co-resident CTAs per SM (what shared memory allows) walk a fifth of the bitmap range each
// (0.01 % sub-dark c4 strip: 404 us with one CTA per SM)
static inline int fix_grid(int B) {
  return B <= 80 ? GRX_FIX_PER_SM * kSMs : (B <= 128 ? 2 * kSMs : kSMs);
}

__global__ void __launch_bounds__(kFixThreads) clamp_fix_kernel(
    const uint16_t* __restrict__ raw, GramRawParams p, const uint32_t* __restrict__ pixbits,
    double* __restrict__ outpart) {
  // shared: dQ (packed lower triangle, T) | xs, dx ([kFixBatch][B]) | clamped-band masks
  extern __shared__ __align__(16) double fx[];
  const int B = p.B;
  const int T = B * (B + 1) / 2;
  const int work = B * B + B + 1;
  double* dq = fx;
  double* xs = dq + T;
  double* dx = xs + kFixBatch * B;
  uint32_t* km = reinterpret_cast<uint32_t*>(dx + kFixBatch * B);  // [kFixBatch][4] (B<=128)
  __shared__ int64_t list[kFixBatch];
  __shared__ int cnt[kFixThreads];
  __shared__ int nlist;
  const int tid = threadIdx.x;
  if (!(*reinterpret_cast<volatile int32_t*>(p.flags) & 4)) return;  // nothing clamped
  for (int e = tid; e < T; e += kFixThreads) dq[e] = 0.0;
  double as = 0.0;  // thread t < B: sum of dx_t
  const int64_t nwords = (p.L * p.S + 31) / 32;
  const int64_t per = (nwords + gridDim.x - 1) / gridDim.x;
  const int64_t w0 = blockIdx.x * per, w1 = min(nwords, w0 + per);
  // walk the range in fixed order, kFixThreads words per round
  for (int64_t wb = w0; wb < w1; wb += kFixThreads) {
    const int64_t wi = wb + tid;
    const uint32_t bits = wi < w1 ? pixbits[wi] : 0u;
    __syncthreads();
    cnt[tid] = __popc(bits);
    __syncthreads();
    if (tid < 32) {  // exclusive prefix over the 256 counts (one warp, 8 per lane)
      int v[8], tsum = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = cnt[tid * 8 + k], tsum += v[k];
      int incl = tsum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, incl, o);
        if (tid >= o) incl += n;
      }
      int run = incl - tsum;
#pragma unroll
      for (int k = 0; k < 8; ++k) cnt[tid * 8 + k] = run, run += v[k];
      if (tid == 31) nlist = incl;
    }
    __syncthreads();
    const int total = nlist, mybase = cnt[tid];
    for (int k0 = 0; k0 < total; k0 += kFixBatch) {
      {  // this batch's pixels, in bitmap order
        uint32_t bb = bits;
        int rank = mybase;
        while (bb && rank < k0 + kFixBatch) {
          const int bit = __ffs(bb) - 1;
          bb &= bb - 1;
          if (rank >= k0) list[rank - k0] = wi * 32 + bit;
          ++rank;
        }
      }
      for (int t = tid; t < kFixBatch * 4; t += kFixThreads) km[t] = 0u;
      __syncthreads();
      const int nb = total - k0 < kFixBatch ? total - k0 : kFixBatch;
      for (int t = tid; t < nb * B; t += kFixThreads) {
        const int k = t / B, b = t - k * B;
        const int64_t pix = list[k];
        const int s = (int)(pix - (pix / p.S) * p.S);
        const uint16_t r = __ldg(raw + pix * B + b);
        const float df = __ldg(p.dark + (int64_t)s * B + b);
        const double x = (double)__ldg(p.coeff + (int64_t)s * B + b) * p.ginv *
                         ((double)r - (double)df);
        const bool c = (float)r < df;
        xs[t] = x;
        dx[t] = c ? -x : 0.0;
        if (c) atomicOr(km + k * 4 + (b >> 5), 1u << (b & 31));
      }
      __syncthreads();
      // pixel by pixel (a barrier between pixels): for each clamped band c, thread t < B
      // adds entry (max(t, c), min(t, c)); a pair of clamped bands is added once (by the
      // smaller band's pass), so no two threads touch one entry within a pixel
      for (int k = 0; k < nb; ++k) {
        if (tid < B) {
          const int t = tid;
          const double* xk = xs + k * B;
          const double* dk = dx + k * B;
          const uint32_t* mk = km + k * 4;
          const double xt = xk[t], dt = dk[t];
          as += dt;
          const bool tcl = dt != 0.0 || ((mk[t >> 5] >> (t & 31)) & 1u);
          for (int m = 0; m < 4; ++m) {
            uint32_t mm = mk[m];
            while (mm) {
              const int c = 32 * m + __ffs(mm) - 1;
              mm &= mm - 1;
              if (tcl && t < c) continue;  // added in band t's pass as (c, t)
              const int i = t > c ? t : c, j = t > c ? c : t;
              dq[i * (i + 1) / 2 + j] += xt * dk[c] + dt * xk[c] + dt * dk[c];
            }
          }
        }
        __syncthreads();
      }
    }
  }
  __syncthreads();
  // this CTA's partial [dSxx (lower, row-major i >= j) | dSx | dn = 0]
  double* out = outpart + (size_t)blockIdx.x * work;
  for (int e = tid; e < B * B; e += kFixThreads) {
    const int i = e / B, j = e - i * B;
    out[e] = j > i ? 0.0 : dq[i * (i + 1) / 2 + j];
  }
  for (int b = tid; b < B; b += kFixThreads) out[B * B + b] = as;
  if (tid == 0) out[B * B + B] = 0.0;
  if (blockIdx.x == 0 && tid == 0) atomicOr(p.flags, 256);  // clamps corrected
}

static size_t clamp_fix_smem(int B) {
  return ((size_t)B * (B + 1) / 2 + 2 * (size_t)kFixBatch * B) * 8 + kFixBatch * 16;
}

// reduce the per-CTA partials [Sxx | Sx | n] (deterministic) and centre them on shift
int gram_raw_sum_and_center(const double* part, int grid, int bands, double* shift, int own,
                            double* moments, cudaStream_t st, const double* fix, int nfix,
                            const int32_t* flags) {
  const int work = bands * bands + bands + 1;
  double* tot = const_cast<double*>(part) + (size_t)(kSMs + fix_grid(bands)) * work;  // after the partials
  gram_raw_sum_kernel<<<ceil_div(work, 32), 256, 0, st>>>(part, grid, work, tot, fix, nfix,
                                                          flags);
  SKYRX_CHECK_LAUNCH("gram_raw_sum_kernel");
  gram_raw_center_kernel<<<ceil_div(work, 256), 256, 0, st>>>(tot, bands, shift, own, moments);
  SKYRX_CHECK_LAUNCH("gram_raw_center_kernel");
  return SKYRX_OK;
}

int raww_atoms(int bands);
int stats_raw_wide(const uint16_t* raw, int64_t lines, int32_t samples, int32_t bands,
                   const float* dark, const float* coeff, double gain, double* shift, int own,
                   double* moments, int32_t* flags, void* workspace, cudaStream_t st);

static int nch_for(int B) {
  // widest window over all samples: start offset in its 16-B chunk + 2B bytes
  int maxoff = 0;
  for (int s = 0; s < 8; ++s) maxoff = maxoff > ((s * B * 2) & 15) ? maxoff : ((s * B * 2) & 15);
  return (maxoff + 2 * B + 15) / 16;
}

template <int NCH, int EG = kGrEpiGroups>
static int launch_gram_raw(const CUtensorMap& map, const uint16_t* raw, GramRawParams p,
                           double* moments, double* shift, int own, cudaStream_t st) {
  constexpr uint32_t W2B = gr_w2b<NCH>();
  constexpr uint32_t STAGE = kGrLb * (128u + W2B);
  CUtensorMap map1 = map;
  if (W2B > 0) {  // the bytes past 128 of the window: narrower box, matching swizzle
    const cuuint64_t line_bytes = (cuuint64_t)p.S * p.B * 2;
    cuuint64_t dims[2] = {line_bytes, (cuuint64_t)p.L};
    cuuint64_t strides[1] = {line_bytes};
    cuuint32_t box[2] = {W2B, (cuuint32_t)kGrLb};
    cuuint32_t estr[2] = {1, 1};
    const CUresult r = tensor_map_encoder()(
        &map1, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)raw, dims, strides, box, estr,
        CU_TENSOR_MAP_INTERLEAVE_NONE,
        W2B == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                  : (W2B == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B),
        GRX_L2PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    SKYRX_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  }
  constexpr int kGrStages = gr_stages<NCH>();
#ifndef GRX_NO_QACC
  const size_t qbytes = ((size_t)p.B * p.B + p.B) * 8;
#else
  const size_t qbytes = 0;
#endif
  const size_t smem = kGrStages * (size_t)STAGE + qbytes +
                      (size_t)kGrWorkers * 16 * (NCH > 8 ? 2 : 1) * (gr_ones<NCH>() ? 1 : 3) + NCH * 8 * 16 + 3 * (size_t)p.B * 8 +
                      (gr_ones<NCH>() ? kGrLb * 32 : 0) +
                      16 * 8 + 1024;
  int grid = kSMs;
#ifdef GRX_NSPLIT_ENV  // experiment: fewer CTAs than SMs
  if (const char* e = getenv("SKYRX_GR_GRID")) grid = atoi(e) > 0 ? atoi(e) : grid;
#endif
  if (p.units < grid) grid = (int)p.units;
  // tail balancing (see GramRawParams): rem leftover units into tail_k pieces each
  p.units_main = p.units;
  p.tail_k = 1;
  p.tail_lines = p.split_lines;
  {
    const int64_t rem = p.units % grid;
    if (rem > 0 && 2 * rem <= grid) {
      const int k = (int)(grid / rem);
      const int64_t tl = ((p.split_lines + k - 1) / k + kGrLb - 1) / kGrLb * kGrLb;
      if (k > 1 && tl < p.split_lines) {
        p.units_main = p.units - rem;
        p.tail_k = k;
        p.tail_lines = tl;
        p.units = p.units_main + rem * k;
      }
    }
  }
  cudaFuncSetAttribute(gram_raw_kernel<NCH, EG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  // the scan warps mark every pixel holding a value below dark while its tile is on chip
  if (p.pixbits != nullptr)
    cudaMemsetAsync(p.pixbits, 0, (size_t)((p.L * p.S + 31) / 32) * 4, st);
  gram_raw_kernel<NCH, EG><<<grid, gr_threads(EG), smem, st>>>(map, map1, p);
  SKYRX_CHECK_LAUNCH("gram_raw_kernel");
  // exact corrections of the clamped pixels (no-op passes when nothing clamped)
  const int fgrid = fix_grid(p.B);
  const int work = p.B * p.B + p.B + 1;
  const size_t fsm = clamp_fix_smem(p.B);
  if (fsm > 48 * 1024)
    cudaFuncSetAttribute(clamp_fix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm);
  if (p.pixbits != nullptr) {
    clamp_fix_kernel<<<fgrid, kFixThreads, fsm, st>>>(raw, p, p.pixbits,
                                                       p.part + (size_t)grid * work);
    SKYRX_CHECK_LAUNCH("clamp_fix_kernel");
  }  // no bitmap room (workspace from skyrx_stats_raw_workspace): flag 4 stays uncorrected
  return gram_raw_sum_and_center(p.part, grid, p.B, shift, own, moments, st,
                                 p.part + (size_t)grid * work, fgrid, p.flags);
}

}  // namespace skyrx

using namespace skyrx;

extern "C" int skyrx_stats_raw_supported(int64_t lines, int32_t samples, int32_t bands,
                                         const void* raw) {
  if (bands < 1 || lines < 1 || samples < 1) return 0;
  if (((uintptr_t)raw & 15) != 0) return 0;
  if (((int64_t)samples * bands * 2) % 16 != 0) return 0;  // TMA line stride
  if (nch_for(bands) > 16 && raww_atoms(bands) > 5) return 0;  // wide path: <= 640 B windows
  if (lines > ((int64_t)1 << 31) - 1) return 0;
  return tensor_map_encoder() != nullptr ? 1 : 0;
}

extern "C" size_t skyrx_stats_raw_workspace(int32_t bands) {
  // [kSMs + fix_grid(B) partials (Gram CTAs, clamp fix-up CTAs) | total] doubles
  return (size_t)(kSMs + fix_grid(bands) + 1) * ((size_t)bands * bands + bands + 1) * sizeof(double);
}

extern "C" size_t skyrx_stats_raw_workspace_for(int64_t lines, int32_t samples,
                                                int32_t bands) {
  // ... plus the pixel bitmap of the clamp correction (L S bits)
  return skyrx_stats_raw_workspace(bands) + (size_t)((lines * samples + 31) / 32) * 4 + 16;
}

static int stats_raw_impl(const uint16_t* raw, int64_t lines, int32_t samples, int32_t bands,
                          const float* dark, const float* coeff, double gain, double* shift,
                          int own, double* moments, int32_t* flags, void* workspace,
                          size_t workspace_bytes, void* stream) {
  SKYRX_REQUIRE(skyrx_stats_raw_supported(lines, samples, bands, raw),
                "raw-byte tensor-core moments unsupported for this shape/alignment");
  SKYRX_REQUIRE(gain > 0.0, "every line gain must be positive");
  SKYRX_REQUIRE(workspace_bytes >= skyrx_stats_raw_workspace(bands), "workspace too small");
  const int nch = nch_for(bands);
  if (nch > 16)  // windows past 256 bytes: the multi-pass wide kernel (gram_raww.cu)
    return stats_raw_wide(raw, lines, samples, bands, dark, coeff, gain, shift, own, moments,
                          flags, workspace, as_stream(stream));
  // 2-D byte view (byte within line, line); boxes of 128 bytes x Lb lines, swizzled
  const cuuint64_t line_bytes = (cuuint64_t)samples * bands * 2;
  cuuint64_t dims[2] = {line_bytes, (cuuint64_t)lines};
  cuuint64_t strides[1] = {line_bytes};
  cuuint32_t box[2] = {128, (cuuint32_t)kGrLb};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMap map;
  CUresult r = tensor_map_encoder()(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)raw, dims, strides,
                                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                    CU_TENSOR_MAP_SWIZZLE_128B, GRX_L2PROMO,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SKYRX_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  GramRawParams p{};
  p.dark = dark;
  p.coeff = coeff;
  p.ginv = 1.0 / gain;
  p.part = reinterpret_cast<double*>(workspace);
  p.pixbits = workspace_bytes >= skyrx_stats_raw_workspace_for(lines, samples, bands)
                  ? reinterpret_cast<uint32_t*>(p.part + (size_t)(kSMs + fix_grid(bands) + 1) *
                                                             ((size_t)bands * bands + bands + 1))
                  : nullptr;
  p.flags = flags;
  p.L = lines;
  p.S = samples;
  p.B = bands;
  p.nsplit = (int)((lines + kGrMaxUnitLines - 1) / kGrMaxUnitLines);
  // also split so that there are at least ~2 units per SM
  // and into enough units (>= 8 per SM) that the static round-robin tail stays small
  while ((int64_t)samples * p.nsplit < 8 * kSMs && lines / (p.nsplit + 1) >= 4 * kGrLb) ++p.nsplit;
#ifdef GRX_NSPLIT_ENV  // experiment: units per sample column from the environment
  if (const char* e = getenv("SKYRX_GR_NSPLIT")) p.nsplit = atoi(e) > 0 ? atoi(e) : p.nsplit;
#endif
  p.split_lines = (lines + p.nsplit - 1) / p.nsplit;
  p.split_lines = ((p.split_lines + kGrLb - 1) / kGrLb) * kGrLb;
  p.nsplit = (int)((lines + p.split_lines - 1) / p.split_lines);
  p.units = (int64_t)samples * p.nsplit;
  cudaStream_t st = as_stream(stream);
  // long units (>= 32 tiles): two epilogue groups are enough and leave the scan warps more
  // issue slots (strips of B = 40 / 70 / 96 / 128: 0.391 / 0.442 / 0.565 / 1.017 ->
  // 0.367 / 0.434 / 0.540 / 0.990 ms); short units (c1 strips, c2 chunks) are
  // epilogue-bound and keep three
  const bool long_units = kGrEpiGroups == 3 && p.split_lines >= 32 * kGrLb;
  switch (nch) {
#define SKYRX_NCH(k)                                                                  \
  case k:                                                                             \
    return long_units ? launch_gram_raw<k, 2>(map, raw, p, moments, shift, own, st)   \
                      : launch_gram_raw<k>(map, raw, p, moments, shift, own, st);
    SKYRX_NCH(1) SKYRX_NCH(2) SKYRX_NCH(3) SKYRX_NCH(4) SKYRX_NCH(5) SKYRX_NCH(6) SKYRX_NCH(7)
    SKYRX_NCH(8) SKYRX_NCH(9) SKYRX_NCH(10) SKYRX_NCH(11) SKYRX_NCH(12) SKYRX_NCH(13)
    SKYRX_NCH(14) SKYRX_NCH(15) SKYRX_NCH(16)
#undef SKYRX_NCH
  }
  set_error("unsupported band count %d", bands);
  return SKYRX_ERR_ARG;
}

extern "C" int skyrx_stats_raw(const uint16_t* raw, int64_t lines, int32_t samples, int32_t bands,
                               const float* dark, const float* coeff, double gain,
                               const double* shift, double* moments, int32_t* flags,
                               void* workspace, size_t workspace_bytes, void* stream) {
  return stats_raw_impl(raw, lines, samples, bands, dark, coeff, gain,
                        const_cast<double*>(shift), 0, moments, flags, workspace,
                        workspace_bytes, stream);
}

extern "C" int skyrx_stats_raw_own_shift(const uint16_t* raw, int64_t lines, int32_t samples,
                                         int32_t bands, const float* dark, const float* coeff,
                                         double gain, double* shift, double* moments,
                                         int32_t* flags, void* workspace, size_t workspace_bytes,
                                         void* stream) {
  return stats_raw_impl(raw, lines, samples, bands, dark, coeff, gain, shift, 1, moments, flags,
                        workspace, workspace_bytes, stream);
}
