"""`.hsc` cube files (formats.py:1-136 of the reference), the air pipeline's ingest.

Same layout and FormatError texts as the reference. `read_cube` reads the payload
straight into pinned (page-locked) host memory, or through it onto the device
(`device=True`), so a cube reaches HBM at the PCIe rate with no intermediate host copy.
"""

from __future__ import annotations

import os
import struct

import numpy as np
import torch

from . import _dev, errors
from .cube import InsSample, LineMeta, RadianceCube, RawCube

HSC_MAGIC = b"HSC1"
HSC_VERSION = 1
_HSC_HEAD = struct.Struct("<4sHHIII")
_LINE_REC = struct.Struct("<Qf4x")
_INS_BLOCK = struct.Struct("<Qddffff")
LINE_RECORD_SIZE = _LINE_REC.size + 2 * _INS_BLOCK.size
_DTYPES = {0: (np.dtype("<u2"), torch.uint16), 1: (np.dtype("<f4"), torch.float32)}


def _ins_bytes(s) -> bytes:
    return _INS_BLOCK.pack(s.timestamp_us, s.lat_deg, s.lon_deg, s.alt_m, s.roll_deg,
                           s.pitch_deg, s.yaw_deg)


def pack_line_meta(m) -> bytes:
    return _LINE_REC.pack(m.exposure_start_us, m.gain) + _ins_bytes(m.ins_before) + _ins_bytes(
        m.ins_after)


def unpack_line_meta(buf, offset: int) -> LineMeta:
    exposure, gain = _LINE_REC.unpack_from(buf, offset)
    o = offset + _LINE_REC.size
    return LineMeta(exposure, gain, InsSample(*_INS_BLOCK.unpack_from(buf, o)),
                    InsSample(*_INS_BLOCK.unpack_from(buf, o + _INS_BLOCK.size)))


_READ_CHUNK = 64 << 20
_READ_THREADS = 8


def _read_parallel(fd: int, dst: memoryview, offset: int, size: int, need: int) -> None:
    """Payload bytes -> dst with positional reads from several threads (the syscalls release
    the GIL; one thread tops out near 7 GB/s copying out of the page cache)."""
    def read_range(lo: int, hi: int) -> None:
        while lo < hi:
            n = os.preadv(fd, [dst[lo:hi]], offset + lo)
            if n <= 0:
                raise errors.FormatError(f"truncated payload: file is {size} bytes, need {need}")
            lo += n

    total = len(dst)
    spans = [(lo, min(lo + _READ_CHUNK, total)) for lo in range(0, total, _READ_CHUNK)]
    if len(spans) == 1:
        read_range(*spans[0])
        return
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(min(_READ_THREADS, len(spans))) as ex:
        for fut in [ex.submit(read_range, lo, hi) for lo, hi in spans]:
            fut.result()


def write_cube(path, cube) -> None:
    """formats.py:79-95 (device cubes are brought to the host first)."""
    name = type(cube).__name__
    if name == "RawCube":
        code, dt = 0, "<u2"
    elif name == "RadianceCube":
        code, dt = 1, "<f4"
    else:
        raise TypeError(f"not a cube: {type(cube)!r}")
    v = cube.values
    arr = _dev.to_host(v) if isinstance(v, torch.Tensor) else np.asarray(v)
    arr = np.ascontiguousarray(arr, dtype=dt)
    with open(path, "wb") as f:
        f.write(_HSC_HEAD.pack(HSC_MAGIC, HSC_VERSION, code, cube.lines, cube.samples,
                               cube.bands))
        f.write(np.asarray(cube.wavelengths_nm).astype("<f4").tobytes())
        f.write(b"".join(pack_line_meta(m) for m in cube.line_meta))
        f.write(memoryview(arr).cast("B"))


def read_cube(path, *, device: bool = False):
    """formats.py:98-136.  Values land in pinned host memory (a numpy view of it), or on
    the device with `device=True` (the cube then holds a CUDA tensor)."""
    with open(path, "rb") as f:
        size = os.fstat(f.fileno()).st_size
        head = f.read(_HSC_HEAD.size)
        if len(head) < _HSC_HEAD.size:
            raise errors.FormatError(f"truncated header: {size} bytes at offset 0")
        magic, version, code, lines, samples, bands = _HSC_HEAD.unpack(head)
        if magic != HSC_MAGIC:
            raise errors.FormatError(f"bad magic {magic!r} at offset 0")
        if version != HSC_VERSION:
            raise errors.FormatError(f"unsupported version {version} at offset 4")
        if code not in _DTYPES:
            raise errors.FormatError(f"unknown dtype code {code} at offset 6")
        npdt, tdt = _DTYPES[code]
        off = _HSC_HEAD.size
        wl_bytes, meta_bytes = bands * 4, lines * LINE_RECORD_SIZE
        payload = lines * samples * bands * npdt.itemsize
        need = off + wl_bytes + meta_bytes + payload
        if size != need:
            raise errors.FormatError(
                f"truncated payload: file is {size} bytes, need {need} "
                f"(payload starts at offset {off + wl_bytes + meta_bytes})")
        wl = np.frombuffer(f.read(wl_bytes), "<f4").astype(np.float64)
        mbuf = f.read(meta_bytes)
        meta = tuple(unpack_line_meta(mbuf, i * LINE_RECORD_SIZE) for i in range(lines))
        host = torch.empty((lines, samples, bands), dtype=tdt,
                           pin_memory=torch.cuda.is_available())
        if payload:
            _read_parallel(f.fileno(), memoryview(host.view(torch.uint8).numpy().reshape(-1)),
                           off + wl_bytes + meta_bytes, size, need)
    if device:
        values = host.to(_dev.require_cuda(), non_blocking=True)
        torch.cuda.current_stream().synchronize()  # the pinned buffer is released below
    else:
        values = host.numpy()
    cls = RawCube if code == 0 else RadianceCube
    return cls(values, wl, meta)
