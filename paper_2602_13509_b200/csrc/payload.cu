// Link payload epilogue: the per-pixel words of the air-side line
// packets, datalink.py:141-177, bit-exact.
//   word 0: RGB565 of the pixel's colour normalised to the cube's channel maxima,
//           round-half-up in f64: q = floor(x / max * levels + 0.5) clipped (datalink.py:141-152)
//   word 1: IEEE half of sqrt(score / max_score) in f64 (datalink.py:163-168)
// The cube maxima are order-preserving u32 keys reduced on the device (atomicMax,
// exact), so the whole epilogue runs without a host round trip.
#include <cuda_fp16.h>

#include "common.cuh"

namespace skyrx {

__global__ void link_maxima_kernel(const float* __restrict__ scores, const float* __restrict__ rgb,
                                   int64_t n, uint32_t* __restrict__ keys) {
  uint32_t m[4] = {0, 0, 0, 0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    m[0] = max(m[0], f2ord(scores[i]));
#pragma unroll
    for (int c = 0; c < 3; ++c) m[1 + c] = max(m[1 + c], f2ord(rgb[3 * i + c]));
  }
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t v = m[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0 && v) atomicMax(&keys[c], v);
  }
}

__device__ __forceinline__ uint32_t quantize(float x, double mx, double levels) {
  if (!(mx > 0.0)) return 0u;
  const double q = floor(__dadd_rn(__dmul_rn(__ddiv_rn((double)x, mx), levels), 0.5));
  if (!(q >= 0.0)) return 0u;  // negative or NaN (numpy's uint16 cast of NaN gives 0)
  return (uint32_t)(q > levels ? levels : q);
}

struct LinkMax {
  double s, r, g, b;
};

__device__ __forceinline__ LinkMax link_max(const uint32_t* keys, double4 mh) {
  // maxima: device keys (the cube's own, no host round trip) or caller values
  if (keys) return {(double)ord2f(keys[0]), (double)ord2f(keys[1]), (double)ord2f(keys[2]),
                    (double)ord2f(keys[3])};
  return {mh.x, mh.y, mh.z, mh.w};
}

__device__ __forceinline__ uint32_t payload_word(const float* __restrict__ scores,
                                                 const float* __restrict__ rgb, int64_t i,
                                                 const LinkMax& m) {
  const uint32_t c565 = (quantize(rgb[3 * i], m.r, 31.0) << 11) |
                        (quantize(rgb[3 * i + 1], m.g, 63.0) << 5) |
                        quantize(rgb[3 * i + 2], m.b, 31.0);
  uint32_t h = 0;
  if (m.s > 0.0) {
    const __half hv = __double2half(__dsqrt_rn(__ddiv_rn((double)scores[i], m.s)));
    h = (uint32_t)*reinterpret_cast<const uint16_t*>(&hv);
  }
  return c565 | (h << 16);  // little-endian [rgb565, half]
}

__global__ void link_payload_kernel(const float* __restrict__ scores,
                                    const float* __restrict__ rgb, int64_t n,
                                    const uint32_t* __restrict__ keys, double4 mh,
                                    uint32_t* __restrict__ payload) {
  const LinkMax m = link_max(keys, mh);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    payload[i] = payload_word(scores, rgb, i, m);
}

// Where the packet rows go. Plain packets: row l at l * pitch. Frames (datalink.py:243-285):
// groups of gk packets, each followed by gr parity rows (gstride = gk + gr rows of 8 + packet
// bytes), the packet at word off_w = 2 after the frame head; heads (u32 group id, u8 index,
// u8 kind, u16 length) are written for data and parity rows alike.
struct PacketLayout {
  int64_t pitch_w;  // row pitch in words
  int gk, gstride, off_w;
  int gr;           // parity rows per group (frames only)
  int gid0;         // first group id (frames only)
  int frames;       // 1: write frame heads
};

// Whole line packets (datalink.py:176-189): the host-built 128-byte headers with the cube
// maxima patched in from the device keys (header bytes 32..47, `ffff` of datalink.py:49),
// then the payload words, one 128 + 4S byte packet per line.
__global__ void link_packets_kernel(const float* __restrict__ scores,
                                    const float* __restrict__ rgb, int lines, int samples,
                                    const uint32_t* __restrict__ keys,
                                    const uint32_t* __restrict__ headers,
                                    uint32_t* __restrict__ out, PacketLayout lay) {
  const LinkMax m = link_max(keys, make_double4(0, 0, 0, 0));
  const int64_t row = 32 + samples, total = (int64_t)lines * row;
  const int64_t groups = lay.frames ? lines / lay.gk : 0;
  const int64_t heads = groups * lay.gstride;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total + heads;
       w += (int64_t)gridDim.x * blockDim.x) {
    if (w >= total) {  // frame head of row h
      const int64_t h = w - total;
      const int g = (int)(h / lay.gstride), idx = (int)(h - (int64_t)g * lay.gstride);
      uint32_t* dst = out + h * lay.pitch_w;
      dst[0] = (uint32_t)(lay.gid0 + g);
      dst[1] = (uint32_t)idx | ((idx >= lay.gk ? 1u : 0u) << 8) | ((uint32_t)(4 * row) << 16);
      continue;
    }
    const int64_t line = w / row;
    const int c = (int)(w - line * row);
    uint32_t v;
    if (c >= 32) {
      v = payload_word(scores, rgb, line * samples + (c - 32), m);
    } else if (c >= 8 && c < 12) {
      const uint32_t key = keys[c - 8];
      v = key ? __float_as_uint(ord2f(key)) : 0u;
    } else {
      v = headers[line * 32 + c];
    }
    const int64_t r = (line / lay.gk) * lay.gstride + line % lay.gk;
    out[r * lay.pitch_w + lay.off_w + c] = v;
  }
}

}  // namespace skyrx

using namespace skyrx;

extern "C" int skyrx_link_maxima(const float* scores, const float* rgb, int64_t n, uint32_t* keys,
                                 void* stream) {
  SKYRX_REQUIRE(n >= 0, "bad pixel count");
  cudaStream_t st = as_stream(stream);
  cudaMemsetAsync(keys, 0, 4 * sizeof(uint32_t), st);
  if (n > 0) {
    const int grid = (int)std::min<int64_t>(ceil_div<int64_t>(n, 256), 4 * kSMs);
    link_maxima_kernel<<<grid, 256, 0, st>>>(scores, rgb, n, keys);
  }
  SKYRX_CHECK_LAUNCH("skyrx_link_maxima");
  return SKYRX_OK;
}

extern "C" int skyrx_link_payload(const float* scores, const float* rgb, int64_t n,
                                  const uint32_t* keys, const double* max_host,
                                  uint16_t* payload, void* stream) {
  SKYRX_REQUIRE(keys != nullptr || max_host != nullptr, "need keys or host maxima");
  SKYRX_REQUIRE(n >= 0, "bad pixel count");
  if (n == 0) return SKYRX_OK;
  SKYRX_REQUIRE(((uintptr_t)payload & 3) == 0, "payload must be 4-byte aligned");
  const int grid = (int)std::min<int64_t>(ceil_div<int64_t>(n, 256), 8 * kSMs);
  const double4 mh = keys ? make_double4(0, 0, 0, 0)
                          : make_double4(max_host[0], max_host[1], max_host[2], max_host[3]);
  link_payload_kernel<<<grid, 256, 0, as_stream(stream)>>>(scores, rgb, n, keys, mh,
                                                           reinterpret_cast<uint32_t*>(payload));
  SKYRX_CHECK_LAUNCH("skyrx_link_payload");
  return SKYRX_OK;
}

static int launch_packets(const float* scores, const float* rgb, int lines, int samples,
                          const uint32_t* keys, const uint8_t* headers, uint8_t* out,
                          const PacketLayout& lay, void* stream, const char* what) {
  SKYRX_REQUIRE(lines >= 0 && samples >= 0 && keys != nullptr, "bad packet geometry");
  SKYRX_REQUIRE((((uintptr_t)headers | (uintptr_t)out) & 3) == 0,
                "headers / packets must be 4-byte aligned");
  const int64_t total = (int64_t)lines * (32 + samples) +
                        (lay.frames ? (int64_t)(lines / lay.gk) * lay.gstride : 0);
  if (total == 0) return SKYRX_OK;
  const int grid = (int)std::min<int64_t>(ceil_div<int64_t>(total, 256), 8 * kSMs);
  link_packets_kernel<<<grid, 256, 0, as_stream(stream)>>>(
      scores, rgb, lines, samples, keys, reinterpret_cast<const uint32_t*>(headers),
      reinterpret_cast<uint32_t*>(out), lay);
  SKYRX_CHECK_LAUNCH(what);
  return SKYRX_OK;
}

extern "C" int skyrx_link_packets(const float* scores, const float* rgb, int lines, int samples,
                                  const uint32_t* keys, const uint8_t* headers, uint8_t* packets,
                                  void* stream) {
  const PacketLayout lay{32 + samples, max(lines, 1), max(lines, 1), 0, 0, 0, 0};
  return launch_packets(scores, rgb, lines, samples, keys, headers, packets, lay, stream,
                        "skyrx_link_packets");
}

extern "C" int skyrx_link_frames(const float* scores, const float* rgb, int lines, int samples,
                                 const uint32_t* keys, const uint8_t* headers, int group_k,
                                 int group_r, int gid0, uint8_t* frames, void* stream) {
  SKYRX_REQUIRE(group_k >= 1 && group_r >= 0 && group_k + group_r <= 256,
                "bad group geometry");
  SKYRX_REQUIRE(lines % group_k == 0, "line count not a multiple of group size");
  SKYRX_REQUIRE(128 + 4 * (int64_t)samples < 65536, "packet too long for a frame");
  const PacketLayout lay{34 + samples, group_k, group_k + group_r, 2, group_r, gid0, 1};
  return launch_packets(scores, rgb, lines, samples, keys, headers, frames, lay, stream,
                        "skyrx_link_frames");
}
