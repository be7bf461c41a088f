// Tile schedule shared by the tensor-core kernels (K2 moments, K4 scores).
//
// A tile is up to 128 pixel rows = R lines x W samples of one "sample block"
// [s0, s0 + W): every line segment of a tile is contiguous in the BIP cube, so
// the producer fetches a tile with R 1-D bulk copies (cp.async.bulk, TMA
// engine) and the calibration tables of the block (dark, coeff: W x B f32)
// stay resident in shared memory while the CTA walks down the lines.
// S = 900 uses W = 32 (R = 4): 28 full blocks + one 4-sample block that packs
// 32 lines per tile, so rows are >= 97% occupied.
#pragma once
#include "common.cuh"

namespace skyrx {

struct TileSched {
  int32_t S, B, W, nb, wl;    // samples, bands, block width, #blocks, last block width
  int32_t R, rl;              // lines per tile in full / last block
  int64_t L, ng, ngl, items;  // lines, tiles per full / last block, total tiles
};

inline bool tc_sched(int64_t L, int32_t S, int32_t B, int32_t Wmax, TileSched& t) {
  t.S = S;
  t.B = B;
  t.L = L;
  t.W = S < Wmax ? S : Wmax;
  t.nb = (S + t.W - 1) / t.W;
  t.wl = S - (t.nb - 1) * t.W;
  t.R = 128 / t.W;
  t.rl = 128 / t.wl;
  if (t.rl > 128) t.rl = 128;
  t.ng = (L + t.R - 1) / t.R;
  t.ngl = (L + t.rl - 1) / t.rl;
  t.items = (int64_t)(t.nb - 1) * t.ng + t.ngl;
  // every bulk copy (line segment) must be 16-B sized and aligned
  const bool ok = ((int64_t)S * B) % 8 == 0 && ((int64_t)t.W * B) % 8 == 0 &&
                  ((int64_t)t.wl * B) % 8 == 0;
  return ok;
}

struct TileInfo {
  int32_t block, s0, w, r, rows;  // rows = r * w (<= 128)
  int64_t line0, nlines;
};

__host__ __device__ __forceinline__ TileInfo tile_info(const TileSched& t, int64_t item) {
  TileInfo ti;
  const int64_t full = (int64_t)(t.nb - 1) * t.ng;
  int64_t g;
  if (item < full) {
    ti.block = (int32_t)(item / t.ng);
    g = item - (int64_t)ti.block * t.ng;
    ti.w = t.W;
    ti.r = t.R;
  } else {
    ti.block = t.nb - 1;
    g = item - full;
    ti.w = t.wl;
    ti.r = t.rl;
  }
  ti.s0 = ti.block * t.W;
  ti.line0 = g * ti.r;
  ti.nlines = t.L - ti.line0 < ti.r ? t.L - ti.line0 : ti.r;
  ti.rows = (int32_t)(ti.nlines * ti.w);
  return ti;
}

// next tile in item order (same order as tile_info): down the lines of the
// current block, then the next block — no divisions on the per-tile path
__host__ __device__ __forceinline__ void tile_advance(const TileSched& t, TileInfo& ti) {
  if (ti.line0 + ti.r < t.L) {
    ti.line0 += ti.r;
  } else {
    ti.block += 1;
    ti.s0 += t.W;
    ti.line0 = 0;
    const bool last = ti.block == t.nb - 1;
    ti.w = last ? t.wl : t.W;
    ti.r = last ? t.rl : t.R;
  }
  ti.nlines = t.L - ti.line0 < ti.r ? t.L - ti.line0 : ti.r;
  ti.rows = (int32_t)(ti.nlines * ti.w);
}

// jump `step` tiles ahead in item order (round-robin schedules); g is the
// tile's index inside its block and is updated with it
__host__ __device__ __forceinline__ void tile_step(const TileSched& t, TileInfo& ti, int64_t& g,
                                                   int64_t step) {
  g += step;
  int64_t ngb = ti.block == t.nb - 1 ? t.ngl : t.ng;
  while (g >= ngb && ti.block < t.nb - 1) {
    g -= ngb;
    ti.block += 1;
    ngb = ti.block == t.nb - 1 ? t.ngl : t.ng;
  }
  const bool last = ti.block == t.nb - 1;
  ti.s0 = ti.block * t.W;
  ti.w = last ? t.wl : t.W;
  ti.r = last ? t.rl : t.R;
  ti.line0 = g * ti.r;
  ti.nlines = t.L - ti.line0 < ti.r ? t.L - ti.line0 : ti.r;
  ti.rows = (int32_t)(ti.nlines * ti.w);
}

// ----------------------------------------------------------------------------
// Block-pinned schedule (score kernel): every CTA stays in ONE sample block (its
// calibration tables never change) and walks that block's line groups
// round-robin with the other CTAs of the block.  CTAs are spread over the blocks
// in proportion to their tiles, so at any moment the grid reads a narrow band of
// consecutive lines across ALL blocks: contiguous DRAM streaming (a bulk-copy
// probe, tools/tma_probe.cu, gives 6.7 TB/s for that order vs 4.6 TB/s when all
// CTAs sweep the lines of one block together).
constexpr int kMaxPlanCtas = 160;
struct CtaPlan {
  int16_t block[kMaxPlanCtas];  // sample block of CTA c
  int16_t rank[kMaxPlanCtas];   // its rank among the CTAs of that block
  int16_t count[kMaxPlanCtas];  // number of CTAs on that block
};

__host__ __device__ __forceinline__ int64_t block_groups(const TileSched& t, int b) {
  return b == t.nb - 1 ? t.ngl : t.ng;
}

__host__ __device__ __forceinline__ TileInfo tile_at(const TileSched& t, int b, int64_t g) {
  TileInfo ti;
  const bool last = b == t.nb - 1;
  ti.block = b;
  ti.s0 = b * t.W;
  ti.w = last ? t.wl : t.W;
  ti.r = last ? t.rl : t.R;
  ti.line0 = g * ti.r;
  ti.nlines = t.L - ti.line0 < ti.r ? t.L - ti.line0 : ti.r;
  ti.rows = (int32_t)(ti.nlines * ti.w);
  return ti;
}

__host__ __device__ __forceinline__ void tile_next_in_block(const TileSched& t, TileInfo& ti,
                                                            int64_t step) {
  ti.line0 += step * ti.r;
  ti.nlines = t.L - ti.line0 < ti.r ? t.L - ti.line0 : ti.r;
  ti.rows = (int32_t)(ti.nlines * ti.w);
}

// host: spread `grid` CTAs over the blocks in proportion to their tiles (>= 1 each);
// returns the grid actually used (>= number of blocks)
inline int plan_ctas(const TileSched& t, int grid, CtaPlan& cp) {
  if (grid < t.nb) grid = t.nb;
  if (grid > kMaxPlanCtas) grid = kMaxPlanCtas;  // nb <= kMaxPlanCtas (checked by caller)
  int cnt[kMaxPlanCtas];
  int used = 0;
  for (int b = 0; b < t.nb; ++b) {
    const double share = (double)grid * (double)block_groups(t, b) / (double)t.items;
    cnt[b] = share < 1.0 ? 1 : (int)share;
    used += cnt[b];
  }
  while (used > grid) {  // rounding overshoot: take from the block with the most CTAs
    int bb = 0;
    for (int b = 1; b < t.nb; ++b) if (cnt[b] > cnt[bb]) bb = b;
    --cnt[bb];
    --used;
  }
  while (used < grid) {  // give the rest to the blocks with the most tiles per CTA
    int bb = 0;
    double best = -1.0;
    for (int b = 0; b < t.nb; ++b) {
      const double load = (double)block_groups(t, b) / cnt[b];
      if (load > best) best = load, bb = b;
    }
    ++cnt[bb];
    ++used;
  }
  // interleave the blocks in CTA order (CTA c -> block c % nb pattern as far as counts allow)
  int next[kMaxPlanCtas] = {0};
  int c = 0;
  while (c < grid) {
    for (int b = 0; b < t.nb && c < grid; ++b) {
      if (next[b] < cnt[b]) {
        cp.block[c] = (int16_t)b;
        cp.rank[c] = (int16_t)next[b]++;
        cp.count[c] = (int16_t)cnt[b];
        ++c;
      }
    }
  }
  return grid;
}

}  // namespace skyrx
