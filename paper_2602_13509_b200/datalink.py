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

from . import _dev, _lib

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


def _pack_ins(s) -> bytes:
    return _INS.pack(s.timestamp_us, s.lat_deg, s.lon_deg, s.alt_m, s.roll_deg, s.pitch_deg,
                     s.yaw_deg)


def packetize_cube(cube_id: int, rgb, scores, line_meta) -> list[bytes]:
    """datalink.py:205-240: every line of a cube to its 3728-byte packet, in line order;
    the payload words of the whole cube from one device pass."""
    lines = int(np.shape(scores)[0])
    if np.shape(rgb)[0] != lines or len(line_meta) != lines:
        raise ValueError("rgb, scores, and line_meta must cover the same lines")
    samples = int(np.shape(rgb)[1])
    if samples != PAYLOAD_SAMPLES:
        raise ValueError(f"rows must be ({PAYLOAD_SAMPLES}, 3) rgb and ({PAYLOAD_SAMPLES},) score")
    words, (ms, mr, mg, mb) = link_payload(rgb, scores)
    payload = words.cpu().numpy()
    out = []
    for i in range(lines):
        m = line_meta[i]
        head = _HEAD.pack(PACKET_MAGIC, PACKET_VERSION, HEADER_LEN, cube_id, i, lines, samples,
                          m.exposure_start_us, ms, mr, mg, mb)
        out.append(head + _pack_ins(m.ins_before) + _pack_ins(m.ins_after)
                   + payload[i].astype("<u2").tobytes())
    return out
