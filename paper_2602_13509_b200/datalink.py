"""Air-side link payload, next to the RX path.

Drop-in for the per-pixel encodings of skyrx.datalink (datalink.py:141-177) and
for ``packetize_cube`` (datalink.py:205-240): the words of every line packet
(RGB565 of the colour normalised to the cube maxima, half-precision
sqrt(score / max)) come from one device kernel over the whole cube
(csrc/payload.cu); only the 128-byte headers are packed on the host.
"""

from __future__ import annotations

import struct

import numpy as np
import torch

from . import _dev, _lib, errors

PACKET_MAGIC = b"SKRX"           # datalink.py:31-36
PACKET_VERSION = 1
HEADER_LEN = 128
PAYLOAD_SAMPLES = 900
PACKET_LEN = HEADER_LEN + PAYLOAD_SAMPLES * 4
_HEAD = struct.Struct("<4sHHIIIIQffff")
_INS = struct.Struct("<Qddffff")


def _keys_to_floats(keys: torch.Tensor) -> list[float]:
    out = []
    for u in keys.cpu().numpy().astype(np.uint64):
        u = int(u)
        b = (u & 0x7FFFFFFF) if (u & 0x80000000) else (~u & 0xFFFFFFFF)
        out.append(float(np.array([b], np.uint32).view(np.float32)[0]))
    return out


def link_payload(rgb, scores):
    """(lines, samples, 3) f32 colours + (lines, samples) f32 scores -> the payload words
    (lines, samples, 2) u16 on the device and the cube maxima (max_score, max_r,
    max_g, max_b) as python floats (datalink.py:219-222)."""
    rgb_d = _dev.to_device(rgb, torch.float32).contiguous()
    sc_d = _dev.to_device(scores, torch.float32).contiguous()
    if tuple(rgb_d.shape[:-1]) != tuple(sc_d.shape) or rgb_d.shape[-1] != 3:
        raise ValueError("rgb must be (..., 3) over the same pixels as scores")
    n = sc_d.numel()
    keys = _dev.zeros((4,), torch.int32)
    s = _dev.stream_ptr()
    _lib.call("skyrx_link_maxima", sc_d.data_ptr(), rgb_d.data_ptr(), n, keys.data_ptr(), s)
    out = _dev.empty(tuple(sc_d.shape) + (2,), torch.int16)
    _lib.call("skyrx_link_payload", sc_d.data_ptr(), rgb_d.data_ptr(), n, keys.data_ptr(),
              None, out.data_ptr(), s)
    maxima = _keys_to_floats(keys) if n else [0.0, 0.0, 0.0, 0.0]
    return out.view(torch.uint16), maxima


def _encode(rgb, scores, maxima):
    """One row's words with caller-given maxima (the reference's per-row helpers)."""
    rgb_d = _dev.to_device(rgb, torch.float32).contiguous()
    sc_d = _dev.to_device(scores, torch.float32).contiguous()
    mh = (_lib.C.c_double * 4)(*[float(m) for m in maxima])
    out = _dev.empty(tuple(sc_d.shape) + (2,), torch.int16)
    _lib.call("skyrx_link_payload", sc_d.data_ptr(), rgb_d.data_ptr(), sc_d.numel(), None, mh,
              out.data_ptr(), _dev.stream_ptr())
    return out.view(torch.uint16).cpu().numpy()


def pack_rgb565(rgb_row, max_r: float, max_g: float, max_b: float) -> np.ndarray:
    """datalink.py:148-152 (maxima <= 0 quantise to 0, as the reference)."""
    rgb_row = np.asarray(rgb_row, np.float32)
    zeros = np.zeros(rgb_row.shape[:-1], np.float32)
    return _encode(rgb_row, zeros, [0.0, max_r, max_g, max_b])[..., 0]


def encode_scores_half(score_row, max_score: float) -> np.ndarray:
    """datalink.py:163-168: u16 bits of half(sqrt(score / max_score))."""
    score_row = np.asarray(score_row, np.float32)
    rgb = np.zeros(score_row.shape + (3,), np.float32)
    return _encode(rgb, score_row, [float(max_score), 0.0, 0.0, 0.0])[..., 1]


def _headers(cube_id: int, lines: int, samples: int, line_meta) -> np.ndarray:
    """(lines, 128) u8 headers (datalink.py:73-89) with zero maxima: the packet kernel
    patches the cube maxima in from the device (bytes 32..47)."""
    buf = bytearray(lines * HEADER_LEN)
    for i in range(lines):
        m = line_meta[i]
        o = i * HEADER_LEN
        _HEAD.pack_into(buf, o, PACKET_MAGIC, PACKET_VERSION, HEADER_LEN, cube_id, i, lines,
                        samples, m.exposure_start_us, 0.0, 0.0, 0.0, 0.0)
        b = m.ins_before
        _INS.pack_into(buf, o + _HEAD.size, b.timestamp_us, b.lat_deg, b.lon_deg, b.alt_m,
                       b.roll_deg, b.pitch_deg, b.yaw_deg)
        a = m.ins_after
        _INS.pack_into(buf, o + _HEAD.size + _INS.size, a.timestamp_us, a.lat_deg, a.lon_deg,
                       a.alt_m, a.roll_deg, a.pitch_deg, a.yaw_deg)
    return np.frombuffer(bytes(buf), np.uint8).reshape(lines, HEADER_LEN)


def cube_packets(cube_id: int, rgb, scores, line_meta) -> torch.Tensor:
    """Every line packet of a cube as one device matrix (lines, 3728) u8, without a host
    round trip for the maxima (datalink.py:205-240 + 176-189)."""
    rgb_d = _dev.to_device(rgb, torch.float32).contiguous()
    sc_d = _dev.to_device(scores, torch.float32).contiguous()
    lines = int(sc_d.shape[0])
    if rgb_d.shape[0] != lines or len(line_meta) != lines:
        raise ValueError("rgb, scores, and line_meta must cover the same lines")
    samples = int(rgb_d.shape[1]) if rgb_d.dim() == 3 else -1
    if (samples != PAYLOAD_SAMPLES or tuple(rgb_d.shape[1:]) != (PAYLOAD_SAMPLES, 3)
            or tuple(sc_d.shape[1:]) != (PAYLOAD_SAMPLES,)):
        raise ValueError(f"rows must be ({PAYLOAD_SAMPLES}, 3) rgb and ({PAYLOAD_SAMPLES},) score")
    s = _dev.stream_ptr()
    keys = _dev.empty((4,), torch.int32)
    _lib.call("skyrx_link_maxima", sc_d.data_ptr(), rgb_d.data_ptr(), sc_d.numel(),
              keys.data_ptr(), s)
    heads = _dev.to_device(_headers(cube_id, lines, samples, line_meta))
    out = _dev.empty((lines, PACKET_LEN), torch.uint8)
    _lib.call("skyrx_link_packets", sc_d.data_ptr(), rgb_d.data_ptr(), lines, samples,
              keys.data_ptr(), heads.data_ptr(), out.data_ptr(), s)
    return out


def packetize_cube(cube_id: int, rgb, scores, line_meta) -> list[bytes]:
    """datalink.py:205-240: every line of a cube to its 3728-byte packet, in line order;
    payload words and maxima from one device pass (cube_packets)."""
    if int(np.shape(scores)[0]) != int(np.shape(rgb)[0]) or len(line_meta) != int(
            np.shape(rgb)[0]):
        raise ValueError("rgb, scores, and line_meta must cover the same lines")
    host = _dev.to_host(cube_packets(cube_id, rgb, scores, line_meta))
    return [row.tobytes() for row in host]


# ---------------------------------------------------------------- frames (datalink.py:243-285)
FRAME_DATA = 0
FRAME_PARITY = 1
_FRAME = struct.Struct("<IBBH")
FRAME_OVERHEAD = _FRAME.size
_CODEC = None


def _codec():
    global _CODEC
    if _CODEC is None:
        from .fec import GROUP_DATA, GROUP_PARITY, ErasureCode

        _CODEC = ErasureCode(GROUP_DATA, GROUP_PARITY)
    return _CODEC


def make_frame(group_id: int, index: int, kind: int, payload: bytes) -> bytes:
    return _FRAME.pack(group_id, index, kind, len(payload)) + payload


def parse_frame(frame: bytes) -> tuple[int, int, int, bytes]:
    """datalink.py:247-261."""
    from .fec import GROUP_DATA, GROUP_PARITY

    if len(frame) < FRAME_OVERHEAD:
        raise errors.FormatError(f"short frame: {len(frame)} bytes")
    group_id, index, kind, plen = _FRAME.unpack_from(frame, 0)
    if len(frame) != FRAME_OVERHEAD + plen:
        raise errors.FormatError(
            f"frame length {len(frame)} != header claim {plen + FRAME_OVERHEAD}")
    if kind == FRAME_DATA and not 0 <= index < GROUP_DATA:
        raise errors.FormatError(f"data frame index {index} outside 0..{GROUP_DATA - 1}")
    if kind == FRAME_PARITY and not GROUP_DATA <= index < GROUP_DATA + GROUP_PARITY:
        raise errors.FormatError(f"parity frame index {index} outside {GROUP_DATA}.."
                                 f"{GROUP_DATA + GROUP_PARITY - 1}")
    if kind not in (FRAME_DATA, FRAME_PARITY):
        raise errors.FormatError(f"unknown frame kind {kind}")
    return group_id, index, kind, frame[FRAME_OVERHEAD:]


def _frames(cube_id: int, data: np.ndarray, parity: np.ndarray) -> list[bytes]:
    k, p = data.shape[1], parity.shape[1]
    out = []
    for g in range(data.shape[0]):
        gid = cube_id * data.shape[0] + g
        out.extend(make_frame(gid, i, FRAME_DATA, data[g, i].tobytes()) for i in range(k))
        out.extend(make_frame(gid, k + i, FRAME_PARITY, parity[g, i].tobytes())
                   for i in range(p))
    return out


def _group_parity(packets_d: torch.Tensor):
    codec = _codec()
    lines, n = packets_d.shape
    k = codec.data_count
    if lines % k != 0:
        raise ValueError(f"line count {lines} not a multiple of group size {k}")
    data = packets_d.view(lines // k, k, n)
    return data, codec.encode_groups(data)


def frames_for_cube(cube_id: int, packets) -> list[bytes]:
    """datalink.py:264-285: packets 50 at a time, each group followed by 25 parity frames;
    the parity of all groups from one device launch."""
    from .fec import GROUP_DATA

    if len(packets) % GROUP_DATA != 0:
        raise ValueError(
            f"line count {len(packets)} not a multiple of group size {GROUP_DATA}")
    if not len(packets):
        return []
    length = len(packets[0])
    if any(len(p) != length for p in packets):
        raise ValueError("invalid group: payload lengths differ")
    host = np.frombuffer(b"".join(packets), np.uint8).reshape(len(packets), length)
    data, parity = _group_parity(_dev.to_device(host))
    return _frames(cube_id, host.reshape(data.shape), _dev.to_host(parity))


def cube_frames_device(cube_id: int, rgb, scores, line_meta) -> torch.Tensor:
    """The cube's whole frame stream as one device matrix (frames, 8 + 3728) u8, in link
    order: packets written straight into their frame rows (skyrx_link_frames), then every
    group's parity rows by one RS launch over those rows (skyrx_gf_matmul)."""
    codec = _codec()
    k, r = codec.data_count, codec.parity_count
    rgb_d = _dev.to_device(rgb, torch.float32).contiguous()
    sc_d = _dev.to_device(scores, torch.float32).contiguous()
    lines = int(sc_d.shape[0])
    if rgb_d.shape[0] != lines or len(line_meta) != lines:
        raise ValueError("rgb, scores, and line_meta must cover the same lines")
    if (tuple(rgb_d.shape[1:]) != (PAYLOAD_SAMPLES, 3)
            or tuple(sc_d.shape[1:]) != (PAYLOAD_SAMPLES,)):
        raise ValueError(f"rows must be ({PAYLOAD_SAMPLES}, 3) rgb and ({PAYLOAD_SAMPLES},) score")
    if lines % k != 0:
        raise ValueError(f"line count {lines} not a multiple of group size {k}")
    groups = lines // k
    s = _dev.stream_ptr()
    keys = _dev.empty((4,), torch.int32)
    _lib.call("skyrx_link_maxima", sc_d.data_ptr(), rgb_d.data_ptr(), sc_d.numel(),
              keys.data_ptr(), s)
    heads = _dev.to_device(_headers(cube_id, lines, PAYLOAD_SAMPLES, line_meta))
    pitch = FRAME_OVERHEAD + PACKET_LEN
    frames = _dev.empty((groups * (k + r), pitch), torch.uint8)
    _lib.call("skyrx_link_frames", sc_d.data_ptr(), rgb_d.data_ptr(), lines, PAYLOAD_SAMPLES,
              keys.data_ptr(), heads.data_ptr(), k, r, cube_id * groups, frames.data_ptr(), s)
    if r and groups:
        base = frames.data_ptr() + FRAME_OVERHEAD
        _lib.call("skyrx_gf_matmul", codec._parity_d.data_ptr(), 0, r, k, base, pitch,
                  (k + r) * pitch, PACKET_LEN, base + k * pitch, pitch, (k + r) * pitch, groups,
                  s)
    return frames


def cube_frames(cube_id: int, rgb, scores, line_meta) -> list[bytes]:
    """The air side's transmit stage (pipeline.py:176-180) fused on the device:
    frames_for_cube(packetize_cube(...)) with one D2H of the finished frame stream."""
    host = _dev.to_host(cube_frames_device(cube_id, rgb, scores, line_meta))
    return [row.tobytes() for row in host]
