// Synthetic push-broom raw cubes on the device (bench / test inputs only).
//
// Bit-identical twin of oracle/synth.py generate_lines(): the same 32-bit
// integer hashes and the same sequence of individually rounded f32 operations
// (__fadd_rn/__fmul_rn/__fdiv_rn/__fsqrt_rn, rintf), so any line block of any
// config regenerates exactly on CPU for parity checks.  One thread per
// (pixel, band) element keeps the uint16 stores coalesced.
#include "common.cuh"

namespace skyrx {

constexpr int kRLatent = 6;
constexpr int kNAnom = 32;
constexpr int kCell = 16;
constexpr uint32_t kPCell24 = 129496;  // see oracle/synth.py P_CELL24

__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}

__device__ __forceinline__ float ih4(uint32_t h) {
  const int s = (int)(h & 255u) + (int)((h >> 8) & 255u) + (int)((h >> 16) & 255u) +
                (int)(h >> 24) - 510;
  return __fmul_rn((float)s, 0x1.bb688cp-8f /* f32(1/sqrt(21845)) = oracle/synth.py INV_IH4 */);
}

struct SynthParams {
  uint32_t seedkey, cellkey;
  int32_t samples, bands, components;
  const uint32_t* cw24;
  const float *mean, *factor, *sd, *aspec, *asd, *xbar, *dark, *coeff;
  int64_t line0, nlines;
};

__global__ void __launch_bounds__(256) synth_kernel(SynthParams p, uint16_t* __restrict__ out) {
  const int B = p.bands;
  const int64_t total = p.nlines * (int64_t)p.samples * B;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pl = e / B;  // pixel within the block
    const int b = (int)(e - pl * B);
    const int64_t lrel = pl / p.samples;
    const int s = (int)(pl - lrel * p.samples);
    const int64_t l = p.line0 + lrel;
    const uint64_t g = (uint64_t)l * (uint64_t)p.samples + (uint64_t)s;
    const uint32_t pk = fmix32((uint32_t)g ^ fmix32((uint32_t)(g >> 32) ^ p.seedkey));
    const uint32_t hb1 = fmix32(pk ^ ((uint32_t)b * 0x85EBCA77u + 0xC2B2AE3Du));
    const float n1 = ih4(hb1);
    // anomaly cell
    const int64_t ncs = (p.samples + kCell - 1) / kCell;
    const uint64_t cell = (uint64_t)((l / kCell) * ncs + (s / kCell));
    const uint32_t ck = fmix32((uint32_t)cell ^ p.cellkey);
    int aidx = -1;
    if ((ck >> 8) < kPCell24) {
      const uint32_t h2 = fmix32(ck + 0x68E31DA4u);
      const int side = (int)(h2 % 6u) + 3;
      const int span = 17 - side;
      const int ol = (int)((h2 >> 8) % (uint32_t)span);
      const int os = (int)((h2 >> 16) % (uint32_t)span);
      const int dl = (int)(l % kCell) - ol;
      const int ds = (s % kCell) - os;
      if (dl >= 0 && dl < side && ds >= 0 && ds < side) aidx = (int)((h2 >> 24) % (uint32_t)kNAnom);
    }
    float t;
    if (aidx >= 0) {
      t = __fadd_rn(p.aspec[aidx * B + b], __fmul_rn(p.asd[b], n1));
    } else {
      const uint32_t u24 = fmix32(pk) >> 8;
      int k = 0;
      for (int c = 0; c < p.components - 1; ++c) k += (p.cw24[c] <= u24) ? 1 : 0;
      t = p.mean[k * B + b];
      const float* fr = p.factor + ((size_t)k * B + b) * kRLatent;
#pragma unroll
      for (int j = 0; j < kRLatent; ++j) {
        const float gj = ih4(fmix32(pk + (uint32_t)(1 + j) * 0x9E3779B9u));
        t = __fadd_rn(t, __fmul_rn(fr[j], gj));
      }
      t = __fadd_rn(t, __fmul_rn(p.sd[k * B + b], n1));
    }
    t = fmaxf(t, 0.0f);
    const uint32_t hb2 = fmix32(pk ^ ((uint32_t)b * 0x85EBCA77u + 2u * 0xC2B2AE3Du));
    const float n2 = ih4(hb2);
    float q = __fmul_rn(t, p.xbar[b]);
    q = __fsqrt_rn(q);
    q = __fmul_rn(q, 0.02f);
    t = __fadd_rn(t, __fmul_rn(q, n2));
    const size_t tb = (size_t)s * B + b;
    float dn = __fadd_rn(__fdiv_rn(t, p.coeff[tb]), p.dark[tb]);
    dn = rintf(dn);
    dn = fminf(fmaxf(dn, 0.0f), 4095.0f);
    out[e] = (uint16_t)dn;
  }
}

}  // namespace skyrx

using namespace skyrx;

extern "C" int skyrx_synth_raw(uint32_t seedkey, uint32_t cellkey, int32_t samples,
                               int32_t bands, int32_t components, const uint32_t* cw24,
                               const float* mean, const float* factor, const float* sd,
                               const float* aspec, const float* asd, const float* xbar,
                               const float* dark, const float* coeff, int64_t line0,
                               int64_t nlines, uint16_t* out, void* stream) {
  SKYRX_REQUIRE(samples > 0 && bands > 0 && components >= 1 && nlines >= 0,
                "bad synth arguments");
  SynthParams p{seedkey, cellkey, samples, bands, components, cw24, mean, factor, sd,
                aspec,   asd,     xbar,    dark,  coeff,      line0, nlines};
  const int64_t total = nlines * (int64_t)samples * bands;
  if (total == 0) return SKYRX_OK;
  int64_t blocks = ceil_div<int64_t>(total, 256);
  if (blocks > (int64_t)kSMs * 32) blocks = (int64_t)kSMs * 32;
  synth_kernel<<<(int)blocks, 256, 0, as_stream(stream)>>>(p, out);
  SKYRX_CHECK_LAUNCH("skyrx_synth_raw");
  return SKYRX_OK;
}
