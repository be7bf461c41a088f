// K5 — score maximum, normalisation, threshold masks and the top-0.1% select.
//
// rx.py:100-105 normalize_scores (f32 division by f32(max)), rx.py:108-112
// threshold_scores (strict > in f32), cube.py:174-176 max_score, and the new
// R-TOPK row: mask = delta > delta_(k+1), k = ceil(N/1000).
// The select is an exact 3-digit (11/11/10-bit) radix select over
// order-preserving u32 keys: integer histogram atomics only, so the threshold
// is exact and deterministic.  HBM-bound: each digit re-reads the scores
// (4 B/px); the mask pass reads 4 B and writes 1 B per pixel.
#include "common.cuh"

namespace skyrx {

// workspace layout (uint32 words)
constexpr int kHistBins = 2048;
struct TopkState {
  uint32_t prefix;   // key bits selected so far
  uint32_t ncand;    // skyrx_topk_mask: candidates appended by the mask pass
  uint64_t rank;     // 1-based rank (from the top) still to find inside the prefix
  uint32_t all;      // 1 -> k >= n: select everything
  uint32_t done;     // skyrx_topk_mask: CTAs of the mask pass that finished
};

__global__ void max_kernel(const float* __restrict__ v, int64_t n, uint32_t* __restrict__ out) {
  uint32_t m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, f2ord(v[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

__global__ void normalize_kernel(const float* __restrict__ v, int64_t n,
                                 const uint32_t* __restrict__ max_key, float* __restrict__ out) {
  const float m = ord2f(*max_key);
  const bool scale = m > 0.0f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = scale ? __fdiv_rn(v[i], m) : v[i];
}

__global__ void threshold_kernel(const float* __restrict__ v, int64_t n, float t,
                                 uint8_t* __restrict__ mask) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    mask[i] = v[i] > t;
}

__global__ void transmit_kernel(const float* __restrict__ v, int64_t n, double m,
                                double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double r = (double)v[i] / m;  // rx.py:124 sqrt(clip(v / max, 0))
    out[i] = m > 0.0 ? sqrt(r > 0.0 ? r : 0.0) : 0.0;
  }
}

__global__ void mask_gt_kernel(const float* __restrict__ v, int64_t n,
                               const float* __restrict__ thr, uint8_t* __restrict__ mask) {
  const float t = *thr;
  const int64_t n4 = n / 4;
  const float4* v4 = reinterpret_cast<const float4*>(v);
  uint32_t* m4 = reinterpret_cast<uint32_t*>(mask);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 x = v4[i];
    if (t == -INFINITY) {  // k >= n (topk_threshold's "select all"): oracle's np.ones
      m4[i] = 0x01010101u;
      continue;
    }
    m4[i] = (uint32_t)(x.x > t) | ((uint32_t)(x.y > t) << 8) | ((uint32_t)(x.z > t) << 16) |
            ((uint32_t)(x.w > t) << 24);
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    mask[i] = t == -INFINITY || v[i] > t;
}

__global__ void mask_gt_scalar_kernel(const float* __restrict__ v, int64_t n,
                                      const float* __restrict__ thr, uint8_t* __restrict__ mask) {
  const float t = *thr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    mask[i] = t == -INFINITY || v[i] > t;
}

__device__ __forceinline__ void digit_params(int digit, int& shift, int& bits) {
  // digit 0: bits 31..21, digit 1: 20..10, digit 2: 9..0
  if (digit == 0) shift = 21, bits = 11;
  else if (digit == 1) shift = 10, bits = 11;
  else shift = 0, bits = 10;
}

__global__ void topk_init_kernel(int64_t n, int64_t k, TopkState* st, uint32_t* hist) {
  for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) hist[i] = 0;
  if (threadIdx.x == 0) {
    st->prefix = 0;
    st->ncand = 0;
    st->done = 0;
    st->rank = (uint64_t)k + 1;
    st->all = (k >= n) ? 1u : 0u;
  }
}

__global__ void __launch_bounds__(512) topk_hist_kernel(const float* __restrict__ v, int64_t n,
                                                        int digit,
                                                        const TopkState* __restrict__ st,
                                                        uint32_t* __restrict__ hist) {
  __shared__ uint32_t sh[kHistBins];
  if (st->all) return;
  for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  int shift, bits;
  digit_params(digit, shift, bits);
  const int hi_shift = shift + bits;  // bits above this digit must equal the prefix
  const uint32_t prefix = st->prefix;
  const uint32_t mask = (1u << bits) - 1u;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t key = f2ord(v[i]);
    const bool match = (hi_shift >= 32) ? true : ((key >> hi_shift) == prefix);
    if (match) atomicAdd(&sh[(key >> shift) & mask], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kHistBins; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// one CTA of 256 threads: suffix counts over the bins from the top (each thread owns
// 8 consecutive bins), pick the bin holding the target rank
__global__ void __launch_bounds__(256) topk_pick_kernel(int digit, TopkState* st, uint32_t* hist,
                                                        float* thr) {
  __shared__ uint64_t wsum[8];
  __shared__ int found_bin;
  __shared__ uint64_t found_cum;
  if (st->all) {
    if (threadIdx.x == 0 && digit == 2) *thr = -INFINITY;
    return;
  }
  int shift, bits;
  digit_params(digit, shift, bits);
  const int nb = 1 << bits;
  const int per = nb / 256;           // 8 (11-bit digits) or 4 (10-bit)
  const int t = threadIdx.x;
  // thread t owns bins [nb - per*(t+1), nb - per*t): thread 0 holds the top bins
  const int hi = nb - per * t;
  uint32_t c[8];
  uint64_t mine = 0;
  for (int q = 0; q < per; ++q) c[q] = hist[hi - 1 - q], mine += c[q];
  // exclusive prefix over threads (= count of all bins above this thread's bins)
  uint64_t incl = mine;
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if ((t & 31) >= o) incl += v;
  }
  if ((t & 31) == 31) wsum[t >> 5] = incl;
  if (t == 0) found_bin = 0, found_cum = 0;
  __syncthreads();
  uint64_t before = incl - mine;
  for (int w = 0; w < (t >> 5); ++w) before += wsum[w];
  const uint64_t rank = st->rank;
  if (before < rank && before + mine >= rank) {  // exactly one thread (rank <= total)
    uint64_t cum = before;
    int q = 0;
    for (; q < per - 1; ++q) {
      if (cum + c[q] >= rank) break;
      cum += c[q];
    }
    found_bin = hi - 1 - q;
    found_cum = cum;
  }
  __syncthreads();
  if (t == 0) {
    // rank beyond every bin (cannot happen with a consistent histogram): keep bin 0
    st->rank = rank - found_cum;
    st->prefix = (st->prefix << bits) | (uint32_t)found_bin;
    if (digit == 2) *thr = ord2f(st->prefix);
  }
  __syncthreads();
  for (int i = t; i < kHistBins; i += blockDim.x) hist[i] = 0;
}

// ---------------------------------------------------------------------------
// One-pass select + mask (skyrx_topk_mask).  After the digit-0 histogram (fused
// into the score kernel, or one topk_hist pass) every CTA of the mask pass
// picks the digit-0 bin itself (the same suffix scan as topk_pick_kernel, on
// read-only bins), then streams the scores once: keys above the bin are in the
// mask, keys below are not, keys inside it are written 0 and appended as
// (index, key) candidates.  The last CTA to finish (atomic count) then runs
// digits 1 and 2 on the candidates only and sets the mask bytes of those above
// the threshold.  The threshold and mask are the ones the 3 x (hist + pick) +
// mask_gt sequence gives (same bins, same picks); it reads the scores once
// instead of three times and is one launch instead of six.

// block-wide (NT threads) pick over nb = 2^bits bins from the top: the bin that
// holds `rank` and the count above it
template <int NT>
__device__ __forceinline__ void pick_bin(const uint32_t* hist, int bits, uint64_t rank,
                                         int& bin_out, uint64_t& cum_out, uint64_t* wsum,
                                         int* sbin, uint64_t* scum) {
  const int nb = 1 << bits;
  const int per = nb / NT;
  const int t = threadIdx.x;
  const int hi = nb - per * t;
  uint32_t c[8];
  uint64_t mine = 0;
  for (int q = 0; q < per; ++q) c[q] = hist[hi - 1 - q], mine += c[q];
  uint64_t incl = mine;
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if ((t & 31) >= o) incl += v;
  }
  if ((t & 31) == 31) wsum[t >> 5] = incl;
  if (t == 0) *sbin = 0, *scum = 0;
  __syncthreads();
  uint64_t before = incl - mine;
  for (int w = 0; w < (t >> 5); ++w) before += wsum[w];
  if (before < rank && before + mine >= rank) {
    uint64_t cum = before;
    int q = 0;
    for (; q < per - 1; ++q) {
      if (cum + c[q] >= rank) break;
      cum += c[q];
    }
    *sbin = hi - 1 - q;
    *scum = cum;
  }
  __syncthreads();
  bin_out = *sbin;
  cum_out = *scum;
  __syncthreads();
}

// digits 1 and 2 over the candidates (or, if they overflowed the buffer, over
// every score inside the digit-0 bin), the threshold, and the mask bytes of the
// candidates above it; leaves the workspace as topk_pick(2) does.  Block-wide.
template <int NT>
__device__ void topk_mask_finish(const float* __restrict__ v, int64_t n, TopkState* st,
                                 uint32_t* hist, uint8_t* mask, const uint2* cand, uint32_t cap,
                                 float* thr, uint32_t* sh, uint64_t* wsum, int* sbin,
                                 uint64_t* scum) {
  const int t = threadIdx.x;
  int bin;
  uint64_t cum;
  uint64_t rank = st->rank;
  pick_bin<NT>(hist, 11, rank, bin, cum, wsum, sbin, scum);
  rank -= cum;
  uint32_t prefix = (uint32_t)bin;
  const uint32_t nc = __ldcg(&st->ncand);
  const bool over = nc > cap;
  for (int digit = 1; digit < 3; ++digit) {
    const int shift = digit == 1 ? 10 : 0, bits = digit == 1 ? 11 : 10;
    const int hs = shift + bits;
    const uint32_t dm = (1u << bits) - 1u;
    for (int i = t; i < kHistBins; i += NT) sh[i] = 0;
    __syncthreads();
    if (!over) {
      // four independent loads in flight per thread (the loop is latency-bound)
      for (uint32_t j0 = t; j0 < nc; j0 += 4 * NT) {
        uint32_t key[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t j = j0 + u * NT;
          key[u] = j < nc ? __ldcg(&cand[j].y) : 0u;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (j0 + u * NT < nc && (key[u] >> hs) == prefix)
            atomicAdd(&sh[(key[u] >> shift) & dm], 1u);
      }
    } else {
      for (int64_t j = t; j < n; j += NT) {
        const uint32_t key = f2ord(v[j]);
        if ((key >> hs) == prefix) atomicAdd(&sh[(key >> shift) & dm], 1u);
      }
    }
    __syncthreads();
    pick_bin<NT>(sh, bits, rank, bin, cum, wsum, sbin, scum);
    rank -= cum;
    prefix = (prefix << bits) | (uint32_t)bin;
  }
  const float tv = ord2f(prefix);
  const uint32_t b0 = prefix >> 21;
  if (!over) {
    for (uint32_t j0 = t; j0 < nc; j0 += 4 * NT) {
      uint2 c[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t j = j0 + u * NT;
        c[u] = j < nc ? __ldcg(&cand[j]) : make_uint2(0u, 0u);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (j0 + u * NT < nc && ord2f(c[u].y) > tv) mask[c[u].x] = 1;
    }
  } else {
    for (int64_t j = t; j < n; j += NT) {
      const float x = v[j];
      if ((f2ord(x) >> 21) == b0 && x > tv) mask[j] = 1;
    }
  }
  for (int i = t; i < kHistBins; i += NT) hist[i] = 0;
  if (t == 0) {
    st->rank = rank;
    st->prefix = prefix;
    st->done = 0;
    *thr = tv;
  }
}

#ifndef MASKX_THREADS  // experiment switches (threads per CTA, CTAs per SM of the mask pass)
#define MASKX_THREADS 512
#endif
#ifndef MASKX_PERSM
#define MASKX_PERSM 4
#endif
constexpr int kMaskThreads = MASKX_THREADS;
__global__ void __launch_bounds__(kMaskThreads) topk_mask_pass_kernel(
    const float* __restrict__ v, int64_t n, TopkState* st, uint32_t* hist,
    uint8_t* __restrict__ mask, uint2* __restrict__ cand, uint32_t cap, float* thr) {
  __shared__ uint32_t sh[kHistBins];
  __shared__ uint64_t wsum[kMaskThreads / 32];
  __shared__ int sbin;
  __shared__ uint64_t scum;
  __shared__ int last;
  const bool all = st->all != 0;
  int bin = 0;
  uint64_t cum = 0;
  if (!all) pick_bin<kMaskThreads>(hist, 11, st->rank, bin, cum, wsum, &sbin, &scum);
  const uint32_t b0 = (uint32_t)bin;
  const int lane = threadIdx.x & 31;
  const int64_t n4 = n / 4;
  const float4* v4 = reinterpret_cast<const float4*>(v);
  uint32_t* m4 = reinterpret_cast<uint32_t*>(mask);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // every thread of a warp runs the same number of iterations (ballots below)
  const int64_t iters = (n4 + stride - 1) / stride;
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t i = it * stride + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool ok = i < n4;
    float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ok) x = __ldcs(v4 + i);
    const float xv[4] = {x.x, x.y, x.z, x.w};
    uint32_t word = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t key = f2ord(xv[q]);
      const uint32_t d0 = key >> 21;
      bool in = false;
      if (all) {
        word |= 1u << (8 * q);  // k >= n: every score, -inf and NaN included
      } else {
        word |= (uint32_t)(d0 > b0) << (8 * q);
        in = ok && d0 == b0;
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, in);
      if (bal) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&st->ncand, (uint32_t)__popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        const uint32_t slot = base + __popc(bal & ((1u << lane) - 1u));
        if (in && slot < cap) cand[slot] = make_uint2((uint32_t)(4 * i + q), key);
      }
    }
    if (ok) m4[i] = word;
  }
  // the n % 4 tail (block 0)
  if (blockIdx.x == 0) {
    for (int64_t i = n4 * 4 + threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t key = f2ord(v[i]);
      if (all) {
        mask[i] = 1;
      } else {
        mask[i] = (key >> 21) > b0;
        if ((key >> 21) == b0) {
          const uint32_t slot = atomicAdd(&st->ncand, 1u);
          if (slot < cap) cand[slot] = make_uint2((uint32_t)i, key);
        }
      }
    }
  }
  // the last CTA to finish runs digits 1 and 2 on the candidates
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&st->done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (all) {
    if (threadIdx.x == 0) *thr = -INFINITY, st->done = 0;
    return;
  }
  topk_mask_finish<kMaskThreads>(v, n, st, hist, mask, cand, cap, thr, sh, wsum, &sbin, &scum);
}

static int grid_n(int64_t n, int threads, int per_sm) {
  int64_t b = ceil_div<int64_t>(n, threads);
  const int64_t cap = (int64_t)kSMs * per_sm;
  if (b > cap) b = cap;
  return (int)(b < 1 ? 1 : b);
}

}  // namespace skyrx

using namespace skyrx;

extern "C" int skyrx_max(const float* v, int64_t n, uint32_t* max_bits, void* stream) {
  if (n <= 0) return SKYRX_OK;
  max_kernel<<<grid_n(n, 256, 8), 256, 0, as_stream(stream)>>>(v, n, max_bits);
  SKYRX_CHECK_LAUNCH("skyrx_max");
  return SKYRX_OK;
}

extern "C" int skyrx_normalize(const float* v, int64_t n, const uint32_t* max_bits, float* out,
                               void* stream) {
  if (n <= 0) return SKYRX_OK;
  normalize_kernel<<<grid_n(n, 256, 8), 256, 0, as_stream(stream)>>>(v, n, max_bits, out);
  SKYRX_CHECK_LAUNCH("skyrx_normalize");
  return SKYRX_OK;
}

extern "C" int skyrx_threshold(const float* v, int64_t n, float t, uint8_t* mask,
                               void* stream) {
  if (n <= 0) return SKYRX_OK;
  threshold_kernel<<<grid_n(n, 256, 8), 256, 0, as_stream(stream)>>>(v, n, t, mask);
  SKYRX_CHECK_LAUNCH("skyrx_threshold");
  return SKYRX_OK;
}

static_assert(sizeof(TopkState) <= 32, "the histogram starts 32 bytes into the workspace");

extern "C" size_t skyrx_topk_workspace(void) {
  return sizeof(TopkState) + 16 + kHistBins * sizeof(uint32_t);
}

extern "C" int skyrx_topk_threshold(const float* v, int64_t n, int64_t k, float* thr,
                                    void* workspace, void* stream) {
  SKYRX_REQUIRE(n >= 0 && k >= 0, "bad top-k arguments n=%lld k=%lld", (long long)n,
                (long long)k);
  SKYRX_REQUIRE(((uintptr_t)workspace % 16) == 0, "top-k workspace must be 16-B aligned");
  cudaStream_t st = as_stream(stream);
  TopkState* state = reinterpret_cast<TopkState*>(workspace);
  uint32_t* hist = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(workspace) + 32);
  topk_init_kernel<<<1, 256, 0, st>>>(n, k, state, hist);
  for (int digit = 0; digit < 3; ++digit) {
    if (n > 0) topk_hist_kernel<<<grid_n(n, 512, 4), 512, 0, st>>>(v, n, digit, state, hist);
    topk_pick_kernel<<<1, 256, 0, st>>>(digit, state, hist, thr);
  }
  SKYRX_CHECK_LAUNCH("skyrx_topk_threshold");
  return SKYRX_OK;
}

extern "C" int skyrx_topk_init(int64_t n_total, int64_t k, void* workspace, void* stream) {
  SKYRX_REQUIRE(n_total >= 0 && k >= 0, "bad top-k arguments n=%lld k=%lld", (long long)n_total,
                (long long)k);
  SKYRX_REQUIRE(((uintptr_t)workspace % 16) == 0, "top-k workspace must be 16-B aligned");
  topk_init_kernel<<<1, 256, 0, as_stream(stream)>>>(
      n_total, k, reinterpret_cast<TopkState*>(workspace), skyrx_topk_histogram(workspace));
  SKYRX_CHECK_LAUNCH("skyrx_topk_init");
  return SKYRX_OK;
}

extern "C" int skyrx_topk_hist(const float* v, int64_t n, int32_t digit, void* workspace,
                               void* stream) {
  SKYRX_REQUIRE(digit >= 0 && digit < 3 && n >= 0, "bad top-k digit %d / n %lld", digit,
                (long long)n);
  if (n == 0) return SKYRX_OK;
  topk_hist_kernel<<<grid_n(n, 512, 4), 512, 0, as_stream(stream)>>>(
      v, n, digit, reinterpret_cast<TopkState*>(workspace), skyrx_topk_histogram(workspace));
  SKYRX_CHECK_LAUNCH("skyrx_topk_hist");
  return SKYRX_OK;
}

extern "C" int skyrx_topk_pick(int32_t digit, void* workspace, float* thr, void* stream) {
  SKYRX_REQUIRE(digit >= 0 && digit < 3, "bad top-k digit %d", digit);
  topk_pick_kernel<<<1, 256, 0, as_stream(stream)>>>(
      digit, reinterpret_cast<TopkState*>(workspace), skyrx_topk_histogram(workspace), thr);
  SKYRX_CHECK_LAUNCH("skyrx_topk_pick");
  return SKYRX_OK;
}

extern "C" int skyrx_topk_mask(const float* v, int64_t n, int32_t hist0_done, float* thr,
                               uint8_t* mask, void* workspace, void* cand, int64_t cand_cap,
                               void* stream) {
  SKYRX_REQUIRE(n >= 0 && cand_cap >= 0, "bad top-k mask arguments n=%lld cap=%lld",
                (long long)n, (long long)cand_cap);
  SKYRX_REQUIRE(((uintptr_t)v % 16) == 0 && ((uintptr_t)mask % 4) == 0 &&
                    ((uintptr_t)cand % 8) == 0,
                "skyrx_topk_mask: scores 16-B, mask 4-B and candidates 8-B aligned");
  cudaStream_t st = as_stream(stream);
  TopkState* state = reinterpret_cast<TopkState*>(workspace);
  uint32_t* hist = skyrx_topk_histogram(workspace);
  // candidate indices are 32-bit: larger inputs take the in-bin rescan
  const uint32_t cap = n < (int64_t)0xFFFFFFFFu
                           ? (uint32_t)(cand_cap < (int64_t)0xFFFFFFFFu ? cand_cap : 0xFFFFFFFEu)
                           : 0u;
  if (n > 0 && !hist0_done)
    topk_hist_kernel<<<grid_n(n, 512, 4), 512, 0, st>>>(v, n, 0, state, hist);
  topk_mask_pass_kernel<<<grid_n(n / 4 + 1, kMaskThreads, MASKX_PERSM), kMaskThreads, 0, st>>>(
      v, n, state, hist, mask, reinterpret_cast<uint2*>(cand), cap, thr);
  SKYRX_CHECK_LAUNCH("skyrx_topk_mask");
  return SKYRX_OK;
}

extern "C" uint32_t* skyrx_topk_histogram(void* workspace) {
  return reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(workspace) + 32);
}

extern "C" int32_t skyrx_topk_hist_len(void) { return kHistBins; }

extern "C" int skyrx_mask_gt(const float* v, int64_t n, const float* thr, uint8_t* mask,
                             void* stream) {
  if (n <= 0) return SKYRX_OK;
  const bool aligned = ((uintptr_t)v % 16 == 0) && ((uintptr_t)mask % 4 == 0);
  if (aligned) {
    mask_gt_kernel<<<grid_n(n / 4 + 1, 256, 8), 256, 0, as_stream(stream)>>>(v, n, thr, mask);
  } else {
    mask_gt_scalar_kernel<<<grid_n(n, 256, 8), 256, 0, as_stream(stream)>>>(v, n, thr, mask);
  }
  SKYRX_CHECK_LAUNCH("skyrx_mask_gt");
  return SKYRX_OK;
}

extern "C" int skyrx_transmit_domain(const float* v, int64_t n, double max_score, double* out,
                                     void* stream) {
  if (n <= 0) return SKYRX_OK;
  transmit_kernel<<<grid_n(n, 256, 8), 256, 0, as_stream(stream)>>>(v, n, max_score, out);
  SKYRX_CHECK_LAUNCH("skyrx_transmit_domain");
  return SKYRX_OK;
}
