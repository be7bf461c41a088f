// K2-RAW for WIDE windows (128 < B <= 272, BASELINE config 3): the exact raw-byte
// Gram of gram_raw.cu when the 2B-byte window of a sample is wider than 256 bytes.
//
// The byte Gram of a 560-byte window (B = 270) is 14 blocks of 128 x 128 in its
// lower triangle — more than TMEM's 512 columns — so it is computed in PASSES of
// up to four blocks (512 TMEM columns), each pass streaming the cube once:
//   1. raww_scan_kernel: per work unit (sample, line range) the per-band column
//      sums m_s and minima (clamp check: flags |= 4 below dark, 8 = check ran);
//   2. raww_gram_kernel, pass p: tcgen05.mma kind::i8 (u8 x u8 -> s32, exact) of
//      the pass's blocks for every tile of every unit, TMA 128-line x 128-byte
//      SWIZZLE_128B boxes of all window atoms; at the end of a unit the epilogue
//      warps turn the integer blocks into calibrated f64 sums C_b C_b2 (G - d m^T
//      - m d^T + L d d^T) and accumulate them into the CTA's partial in global
//      memory (each band pair belongs to exactly one block, hence one pass);
//   3. the partials are reduced and centred by gram_raw.cu's deterministic kernels.
// Warps of the Gram kernel: 4 x kEpiGroups epilogue (TMEM lane quarters), TMA, MMA.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tma.cuh"
#include "umma.cuh"

namespace skyrx {
using namespace umma;

namespace raww {

#ifndef RAWW_LB
#define RAWW_LB 64
#endif
// lines per tile: 64, so a stage (every window atom: 5 x 8 KB at B = 270) leaves room for
// five stages in flight (2.24 ms against 2.76 ms for 2 stages of 128 lines, B = 270)
constexpr int kLb = RAWW_LB;
// epilogue: kEpiGroups groups of 4 warps (one per TMEM lane quarter); group g takes the
// pass's blocks g, g + kEpiGroups, ...  The pass's blocks fill TMEM, so the epilogue is
// not overlapped with the tensor core: four groups drain a unit's four blocks in parallel
#ifndef RAWW_EPI_GROUPS
#define RAWW_EPI_GROUPS 4
#endif
constexpr int kEpiGroups = RAWW_EPI_GROUPS;
constexpr int kEpiThreads = 128 * kEpiGroups;
constexpr int kTmaWarp = kEpiThreads / 32, kMmaWarp = kTmaWarp + 1;
constexpr int kThreads = kEpiThreads + 64;
constexpr int kMaxStages = 6;
constexpr int kMaxAtoms = 5;        // window <= 640 bytes
constexpr uint32_t kAtom = kLb * 128u;

constexpr int kMaxPass = 4;

struct Params {
  const float* dark;
  const float* coeff;
  double ginv;
  double* part;          // per CTA: Sxx[B*B] (lower), Sx[B], n  (zeroed before the launch)
  const uint32_t* usum;  // per unit: column sums of the window's u16 lanes [units][NW/2]
  int64_t L;
  int32_t S, B;
  int32_t na;            // window atoms (128 B each)
  int32_t nw16;          // u16 lanes per window (= 64 * na)
  int64_t split_lines;
  int64_t units;
  // All passes run in ONE launch, as a thread-block CLUSTER of npass CTAs per group of
  // units: CTA rank r of a cluster computes pass r's blocks of the window for every unit
  // of its group.  Each tile's window atoms are fetched once per cluster and multicast
  // into every CTA's stage (rank r issues atoms a = r mod npass), and a stage is refilled
  // only after the MMAs of all npass CTAs released it (multicast commits), so the cube
  // streams from HBM once for all passes (ncu: 5.1 GB of DRAM reads at B = 270 against
  // 10.3 GB for unicast CTA groups and 4 x 4.6 GB for one launch per pass).
  int32_t npass, ngroups;
  int32_t nblk[kMaxPass];                 // blocks in each pass (<= 4)
  int32_t blk_r[kMaxPass][4], blk_c[kMaxPass][4];  // their (row atom, column atom)
  int32_t nstages;                        // TMA ring depth (<= kMaxStages), all atoms per stage
};

__device__ __forceinline__ void unit_geom(const Params& p, int64_t u, int& s, int64_t& l0,
                                          int64_t& nl) {
  s = (int)(u % p.S);
  l0 = (u / p.S) * p.split_lines;
  nl = p.L - l0 < p.split_lines ? p.L - l0 : p.split_lines;
}

__host__ __device__ constexpr uint32_t idesc_u8(int M, int N) {
  return (2u << 4) | (0u << 7) | (0u << 10) | (1u << 15) | (1u << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// per unit: column sums and minima of every u16 lane of the 16-B aligned window.
// A thread owns one 16-B vector (8 lanes) of one unit's window and walks its lines
// with 16-B loads (a warp covers 512 contiguous bytes of a line), 4 lines deep.
__global__ void __launch_bounds__(256) raww_scan_kernel(const uint16_t* __restrict__ raw,
                                                        Params p,
                                                        const float* __restrict__ dark,
                                                        uint32_t* __restrict__ usum,
                                                        int32_t* __restrict__ flags) {
  const int B = p.B;
  const int64_t pitch = (int64_t)p.S * B;  // u16 per line
  const int nv = p.nw16 / 8;
  // a work item = (unit, vector, slice of <= kScanSlice lines): integer sums of the slices
  // are added atomically (exact, order-free), so a long unit still spreads over the GPU
  constexpr int64_t kScanSlice = 1024;
  const int64_t nsl = (p.split_lines + kScanSlice - 1) / kScanSlice;
  bool clamp = false;
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < p.units * nsl * nv;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t uz = it / nv;
    const int v = (int)(it - uz * nv);
    const int64_t u = uz / nsl, z = uz - u * nsl;
    int s;
    int64_t l0, nl;
    unit_geom(p, u, s, l0, nl);
    l0 += z * kScanSlice;
    nl = nl - z * kScanSlice < kScanSlice ? nl - z * kScanSlice : kScanSlice;
    if (nl <= 0) continue;
    const int64_t w0 = ((int64_t)s * B * 2 & ~(int64_t)15) >> 1;  // first u16 of the window
    const int off = (int)(((int64_t)s * B * 2 & 15) >> 1);
    const int64_t col = w0 + 8 * v;
    uint32_t sum[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t mn[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
    if (col < pitch) {  // line ends are 16-B multiples: a vector is all in or all out
      const uint4* c = reinterpret_cast<const uint4*>(raw + l0 * pitch + col);
      const int64_t vp = pitch / 8;  // uint4 per line
      int64_t l = 0;
      auto acc = [&](const uint4 q) {
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          sum[2 * i] += w[i] & 0xFFFFu;
          sum[2 * i + 1] += w[i] >> 16;
          mn[i] = __vminu2(mn[i], w[i]);
        }
      };
      for (; l + 4 <= nl; l += 4) {
        uint4 q[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) q[i] = __ldg(c + (l + i) * vp);
#pragma unroll
        for (int i = 0; i < 4; ++i) acc(q[i]);
      }
      for (; l < nl; ++l) acc(__ldg(c + l * vp));
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int b = 8 * v + i - off;
        const uint32_t m = (i & 1) ? (mn[i >> 1] >> 16) : (mn[i >> 1] & 0xFFFFu);
        if (b >= 0 && b < B && (float)m < __ldg(dark + (int64_t)s * B + b)) clamp = true;
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) atomicAdd(&usum[u * p.nw16 + 8 * v + i], sum[i]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(flags, 8);
  if (__any_sync(0xffffffffu, clamp) && (threadIdx.x & 31) == 0) atomicOr(flags, 4);
}

__global__ void __launch_bounds__(kThreads, 1) raww_gram_kernel(
    const __grid_constant__ CUtensorMap tmap, const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int ps = blockIdx.x % p.npass;  // this CTA's pass = its rank in the cluster
  const bool first_pass = ps == 0;
  const int nblk = p.nblk[ps];
  const uint32_t STAGE = (uint32_t)p.na * kAtom;  // every atom of the window, slot = atom
  const int kStages = p.nstages;
  const uint16_t all_ctas = (uint16_t)((1u << p.npass) - 1u);
  uint8_t* stages = sm;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stages + kStages * STAGE);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* acc_full = bars + 2 * kStages;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);  // band terms follow
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int B = p.B;
  const int64_t u0 = blockIdx.x / p.npass, ustep = p.ngroups;
  if (tid == 0) {
    // full: this CTA's producer arms it; empty: one multicast commit per cluster CTA
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], p.npass);
    mbar_init(acc_full, 1), mbar_init(acc_empty, kEpiThreads);
    fence_mbar_init();
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();  // every CTA's barriers exist before any multicast lands on them
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kTmaWarp) {
    if ((tid & 31) == 0) {  // ------------------------------------------- TMA producer
      int t = 0;
      for (int64_t u = u0; u < p.units; u += ustep) {
        int s;
        int64_t l0, nl;
        unit_geom(p, u, s, l0, nl);
        const int c0 = (int)(((int64_t)s * B * 2) & ~(int64_t)15);
        const int ntile = (int)((nl + kLb - 1) / kLb);
        for (int k = 0; k < ntile; ++k, ++t) {
          const int st = t % kStages;
          mbar_wait(&empty[st], ((t / kStages) & 1) ^ 1);  // every cluster CTA released st
          mbar_arrive_expect_tx(&full[st], STAGE);          // all atoms land here
          for (int a = ps; a < p.na; a += p.npass)
            tma_load_2d_mc(stages + st * STAGE + a * kAtom, &tmap, c0 + 128 * a,
                           (int)(l0 + (int64_t)k * kLb), &full[st], all_ctas);
        }
      }
    }
  } else if (warp == kMmaWarp) {
    {  // --------------------------------- MMA issuer (whole warp, one elected lane issues)
      constexpr uint32_t id = idesc_u8(128, 128);
      // every operand descriptor is the stage-0 / atom-0 / k-step-0 one plus an offset in
      // its start-address field (16-byte units, bits 0-13; smem < 256 KB never carries):
      // one add per MMA instead of rebuilding both descriptors from parameter-space loads
      // (the single issuing thread, not the tensor core, bounded the kernel:
      // ~30 instructions per 64-clock MMA)
      const uint64_t d0 = smem_desc_sw128(stages, kAtom, 1024);
      uint32_t ao[4], bo[4];
#pragma unroll
      for (int bk = 0; bk < 4; ++bk) {
        ao[bk] = bk < nblk ? (uint32_t)p.blk_r[ps][bk] * (kAtom >> 4) : 0u;
        bo[bk] = bk < nblk ? (uint32_t)p.blk_c[ps][bk] * (kAtom >> 4) : 0u;
      }
      const uint32_t stage16 = STAGE >> 4;
      int t = 0, unit = 0, st = 0;
      uint32_t sph = 0;
      for (int64_t u = u0; u < p.units; u += ustep, ++unit) {
        int s;
        int64_t l0, nl;
        unit_geom(p, u, s, l0, nl);
        const int ntile = (int)((nl + kLb - 1) / kLb);
        mbar_wait(acc_empty, (unit & 1) ^ 1);
        tc_fence_after();
        for (int k = 0; k < ntile; ++k, ++t) {
          mbar_wait(&full[st], sph);
          tc_fence_after();
          const uint64_t ds = d0 + (uint64_t)(st * stage16);
          if (elect_one()) {
#pragma unroll
            for (int ks = 0; ks < kLb / 32; ++ks) {
              const uint32_t acc = (k > 0 || ks > 0) ? 1u : 0u;
              const uint64_t dk = ds + (uint64_t)(ks * (4096 >> 4));
#pragma unroll
              for (int bk = 0; bk < 4; ++bk)
                if (bk < nblk) mma_i8(tmem + 128 * bk, dk + ao[bk], dk + bo[bk], id, acc);
            }
            mma_commit_mc(&empty[st], all_ctas);  // release st in every cluster CTA
          }
          __syncwarp();
          if (++st == kStages) st = 0, sph ^= 1;
        }
        if (elect_one()) mma_commit(acc_full);
        __syncwarp();
      }
    }
  } else {  // ---------------------------------------------------- epilogue (warps 0..kTmaWarp-1)
    const int te = tid & 127;  // byte row within the row atom = TMEM lane
    const int grp = tid >> 7;
    const uint32_t tq = warp_uniform(tmem + ((uint32_t)(32 * (warp & 3)) << 16));
    double* part = p.part + (size_t)blockIdx.x * ((size_t)B * B + B + 1);
    double* bandC = reinterpret_cast<double*>(bars + 2 * kStages + 2 + 2);  // [B] per unit
    double* bandD = bandC + B;
    double* bandS = bandD + B;
    double nsum = 0.0;
    int unit = 0;
    for (int64_t u = u0; u < p.units; u += ustep, ++unit) {
      int s;
      int64_t l0, nl;
      unit_geom(p, u, s, l0, nl);
      const uint32_t* us = p.usum + u * p.nw16;
      const int off = (int)(((int64_t)s * B * 2) & 15);
      const double Lu = (double)nl;
      const float* drow = p.dark + (int64_t)s * B;
      const float* crow = p.coeff + (int64_t)s * B;
      // this unit's per-band terms, once, for the four epilogue warps
      for (int b = tid; b < B; b += kEpiThreads) {
        bandC[b] = (double)crow[b] * p.ginv;
        bandD[b] = (double)drow[b];
        bandS[b] = (double)us[(off >> 1) + b];
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
      mbar_wait(acc_full, unit & 1);
      tc_fence_after();
      for (int bk = grp; bk < nblk; bk += kEpiGroups) {
        const int mr = p.blk_r[ps][bk], mc = p.blk_c[ps][bk];
        const int m = 128 * mr + te;
        const int rel = m - off;
        const bool in_band = rel >= 0 && rel < 2 * B;
        const int hi = rel & 1;  // 0: this row is band b's lo byte, 1: its hi byte
        const int b = rel >> 1;
        double Cb = 0.0, db = 0.0, Sb = 0.0;
        if (in_band) Cb = bandC[b], db = bandD[b], Sb = bandS[b];
        const uint32_t taddr = tq + 128 * bk;
        for (int cc = 0; cc < 8; cc += 2) {  // two chunks per TMEM wait
          uint32_t v2[32];
          tmem_ld16(taddr + cc * 16, v2);
          tmem_ld16(taddr + (cc + 1) * 16, v2 + 16);
          tmem_ld_wait();
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t* v = v2 + 16 * h;
            uint32_t pv[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) pv[q] = __shfl_xor_sync(0xffffffffu, v[q], 1);
            if (!in_band) continue;
            // the lo-byte row of a band's pair takes the even band columns, the hi-byte row
            // the odd ones; each has both rows (own + partner)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              if ((i & 1) != hi) continue;
              const int reln = 128 * mc + (cc + h) * 16 + 2 * i - off;
              if (reln < 0 || reln >= 2 * B) continue;
              const int b2 = reln >> 1;
              if (b2 > b) continue;  // lower triangle (only the diagonal block has any)
              const uint32_t hh = hi ? v[2 * i + 1] : pv[2 * i + 1];
              const uint32_t hl = hi ? v[2 * i] : pv[2 * i];
              const uint32_t lh = hi ? pv[2 * i + 1] : v[2 * i + 1];
              const uint32_t ll = hi ? pv[2 * i] : v[2 * i];
              // exact integer G entry (< 2^48) to f64 through the 2^52 exponent trick
              const uint64_t gi = ((uint64_t)hh << 16) + (((uint64_t)hl + lh) << 8) + ll;
              const double gv =
                  __hiloint2double(0x43300000 | (int)(gi >> 32), (int)(uint32_t)gi) -
                  4503599627370496.0;
              const double C2 = bandC[b2], d2 = bandD[b2], S2 = bandS[b2];
              const double xx = gv - db * S2 - Sb * d2 + Lu * db * d2;
              // fire-and-forget RED: one thread owns each entry of this CTA's partial,
              // so the adds land in program (unit) order — deterministic — and the
              // epilogue never waits on a global read-modify-write round trip
              atomicAdd(part + (size_t)b * B + b2, Cb * C2 * xx);
            }
          }
        }
      }
      if (first_pass && grp == 0) {  // band sums: sum x = C_b (m_b - L d_b)
        for (int b = te; b < B; b += 128)
          part[(size_t)B * B + b] += bandC[b] * (bandS[b] - Lu * bandD[b]);
        nsum += Lu;
      }
      tc_fence_before();
      mbar_arrive(acc_empty);
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");  // band terms reused next unit
    }
    if (first_pass && tid == 0) part[(size_t)B * B + B] = nsum;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kMmaWarp) tmem_dealloc(tmem, 512);
  cluster_sync_all();  // no CTA leaves while a peer may still multicast into it
}

}  // namespace raww

int gram_raw_sum_and_center(const double* part, int grid, int bands, double* shift, int own,
                            double* moments, cudaStream_t st, const double* fix, int nfix,
                            const int32_t* flags);

// window atoms for B (16-B aligned start, widest offset over the samples)
int raww_atoms(int bands) {
  int maxoff = 0;
  for (int s = 0; s < 8; ++s) maxoff = maxoff > ((s * bands * 2) & 15) ? maxoff : ((s * bands * 2) & 15);
  return (maxoff + 2 * bands + 127) / 128;
}

int stats_raw_wide(const uint16_t* raw, int64_t lines, int32_t samples, int32_t bands,
                   const float* dark, const float* coeff, double gain, double* shift, int own,
                   double* moments, int32_t* flags, void* workspace, cudaStream_t st) {
  using namespace raww;
  Params p{};
  p.dark = dark;
  p.coeff = coeff;
  p.ginv = 1.0 / gain;
  p.part = reinterpret_cast<double*>(workspace);
  p.L = lines;
  p.S = samples;
  p.B = bands;
  p.na = raww_atoms(bands);
  SKYRX_REQUIRE(p.na <= kMaxAtoms, "wide raw-byte moments support windows <= 640 bytes");
  p.nw16 = 64 * p.na;
  // lower-triangle blocks (row atom >= column atom), at most four per pass (TMEM)
  static const int8_t plan3[][4][2] = {{{0, 0}, {1, 0}, {1, 1}, {-1, -1}},
                                       {{2, 0}, {2, 1}, {2, 2}, {-1, -1}}};
  static const int8_t plan4[][4][2] = {{{0, 0}, {1, 0}, {1, 1}, {2, 0}},
                                       {{2, 1}, {2, 2}, {3, 1}, {3, 2}},
                                       {{3, 0}, {3, 3}, {-1, -1}, {-1, -1}}};
  static const int8_t plan5[][4][2] = {{{0, 0}, {1, 0}, {1, 1}, {2, 0}},
                                       {{2, 1}, {2, 2}, {3, 1}, {3, 2}},
                                       {{3, 0}, {3, 3}, {4, 0}, {4, 3}},
                                       {{4, 1}, {4, 2}, {4, 4}, {-1, -1}}};
  int8_t gen[1][4][2];
  const int8_t(*plan)[4][2] = nullptr;
  int npass = 0;
  if (p.na == 3) plan = plan3, npass = 2;
  else if (p.na == 4) plan = plan4, npass = 3;
  else if (p.na == 5) plan = plan5, npass = 4;
  else {  // one or two atoms: every block in one pass
    int nb = 0;
    for (int a = 0; a < p.na; ++a)
      for (int c = 0; c <= a; ++c) gen[0][nb][0] = (int8_t)a, gen[0][nb][1] = (int8_t)c, ++nb;
    for (; nb < 4; ++nb) gen[0][nb][0] = gen[0][nb][1] = -1;
    plan = gen, npass = 1;
  }
  p.npass = npass;
  for (int ps = 0; ps < npass; ++ps) {
    p.nblk[ps] = 0;
    for (int i = 0; i < 4 && plan[ps][i][0] >= 0; ++i) {
      p.blk_r[ps][i] = plan[ps][i][0], p.blk_c[ps][i] = plan[ps][i][1];
      ++p.nblk[ps];
    }
  }
  const size_t stage = (size_t)p.na * kAtom;
  p.nstages = (int)std::min<size_t>(kMaxStages, (kSmemMax - 12288) / stage);
  const size_t smem = p.nstages * stage + 16 * 8 + 3 * (size_t)bands * 8 + 1024;
  cudaFuncSetAttribute(raww_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // one wave of clusters: as many as fit at once (a cluster's CTAs share a GPC)
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)npass;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(npass * (kSMs / npass));
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, raww_gram_kernel, &cfg) != cudaSuccess ||
      nclusters < 1)
    nclusters = kSMs / npass;
  // long units: the epilogue (integer blocks -> calibrated f64) is not overlapped with the
  // tensor core (the pass's blocks fill TMEM), so fewer, longer units (>= 4 per group)
  int64_t nsplit = (lines + 16383) / 16384;
  while ((int64_t)samples * nsplit < 4 * nclusters && lines / (nsplit + 1) >= 4 * kLb) ++nsplit;
  p.split_lines = (lines + nsplit - 1) / nsplit;
  p.split_lines = (p.split_lines + kLb - 1) / kLb * kLb;
  nsplit = (lines + p.split_lines - 1) / p.split_lines;
  p.units = (int64_t)samples * nsplit;
  p.ngroups = p.units < nclusters ? (int)p.units : nclusters;
  const int grid = p.ngroups * p.npass;
  cfg.gridDim = dim3(grid);
  const size_t stride = (size_t)bands * bands + bands + 1;
  cudaMemsetAsync(p.part, 0, (size_t)grid * stride * sizeof(double), st);
  uint32_t* usum = nullptr;
  const size_t usum_n = (size_t)p.units * p.nw16;
  SKYRX_REQUIRE(cudaMallocAsync(&usum, usum_n * sizeof(uint32_t), st) == cudaSuccess,
                "cudaMallocAsync failed");
  p.usum = usum;
  cudaMemsetAsync(usum, 0, usum_n * sizeof(uint32_t), st);
  raww_scan_kernel<<<kSMs * 8, 256, 0, st>>>(raw, p, dark, usum, flags);
  SKYRX_CHECK_LAUNCH("raww_scan_kernel");
  // 2-D byte view of the cube, 128-byte x 128-line swizzled boxes
  const cuuint64_t line_bytes = (cuuint64_t)samples * bands * 2;
  cuuint64_t dims[2] = {line_bytes, (cuuint64_t)lines};
  cuuint64_t strides[1] = {line_bytes};
  cuuint32_t box[2] = {128, (cuuint32_t)kLb};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMap map;
  const CUresult r = tensor_map_encoder()(
      &map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void*)raw, dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SKYRX_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  SKYRX_REQUIRE(cudaLaunchKernelEx(&cfg, raww_gram_kernel, map, p) == cudaSuccess,
                "raww_gram_kernel cluster launch failed");
  SKYRX_CHECK_LAUNCH("raww_gram_kernel");
  cudaFreeAsync(usum, st);
  return gram_raw_sum_and_center(p.part, grid, bands, shift, own, moments, st, nullptr, 0,
                                 nullptr);
}

}  // namespace skyrx
