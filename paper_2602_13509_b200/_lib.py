"""ctypes binding of libskyrx_b200.so (include/skyrx_b200.h).

This is the reference-side binding a maintainer of `skyrx` would add
(INTEGRATION.md): plain C entry points, device pointers as c_void_p, the
CUDA stream as c_void_p.  ctypes.CDLL releases the GIL for the duration of
every call, so the calibrate and detect pipeline stages can run on separate
threads as pipeline.py:182-208 does.

There is no fallback: if the library is missing or no sm_100 device is
visible, every op raises.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libskyrx_b200.so"

OK, ERR_ARG, ERR_CUDA, ERR_INSUFFICIENT, ERR_NONFINITE, ERR_NOT_PD, ERR_RANGE = range(7)


def flags_range(f: int) -> bool:
    """Moments that must be recomputed (common.cuh flags_range): the int8 quantiser
    overflowed (2), or a value clamped at 0 (4) that the raw-byte pass did not correct
    (256 = clamp_fix_kernel corrected it)."""
    f = int(f)
    return bool(f & 2) or (bool(f & 4) and not f & 256)
IN_RAW_U16, IN_F32, IN_F64 = 0, 1, 2

vp, i32, i64, u32, f32, f64, sz = (C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_float,
                                   C.c_double, C.c_size_t)

# name -> (restype, argtypes); mirrors include/skyrx_b200.h one to one
SIGNATURES = {
    "skyrx_version": (C.c_char_p, []),
    "skyrx_last_error": (C.c_char_p, []),
    "skyrx_device_check": (C.c_int, []),
    "skyrx_calibrate": (C.c_int, [vp, i64, i32, i32, vp, vp, vp, vp, i32, i32, vp, vp, vp, vp]),
    "skyrx_bin_radiance": (C.c_int, [vp, i64, i32, i32, vp, i32, i32, vp, vp, vp, vp]),
    "skyrx_moments_len": (sz, [i32]),
    "skyrx_stats_shift": (C.c_int, [i32, vp, i64, i32, i32, vp, vp, vp, vp, vp]),
    "skyrx_stats_workspace": (C.c_int, [i64, i32, i32, C.POINTER(sz)]),
    "skyrx_stats_accumulate": (C.c_int, [i32, vp, i64, i32, i32, vp, vp, vp, vp, i32, vp, vp,
                                         vp, sz, vp]),
    "skyrx_stats_tc_supported": (C.c_int, [i64, i32, i32, vp]),
    "skyrx_stats_tc_workspace": (sz, [i32]),
    "skyrx_quant_shift": (C.c_int, [i32, vp, i64, i32, i32, vp, vp, vp, vp, vp, vp]),
    "skyrx_stats_tc": (C.c_int, [vp, i64, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
    "skyrx_stats_tc_f32": (C.c_int, [vp, i64, i32, i32, vp, vp, vp, vp, vp, sz, vp]),
    "skyrx_stats_raw_supported": (C.c_int, [i64, i32, i32, vp]),
    "skyrx_stats_raw_workspace": (sz, [i32]),
    "skyrx_stats_raw_workspace_for": (sz, [i64, i32, i32]),
    "skyrx_stats_raw": (C.c_int, [vp, i64, i32, i32, vp, vp, f64, vp, vp, vp, vp, sz, vp]),
    "skyrx_stats_raw_own_shift": (C.c_int, [vp, i64, i32, i32, vp, vp, f64, vp, vp, vp, vp, sz, vp]),
    "skyrx_moments_fold":(C.c_int, [vp, vp, i32, f64, vp]),
    "skyrx_moments_fold_keep":(C.c_int, [vp, vp, i32, f64, vp, vp]),
    "skyrx_stats_finalize": (C.c_int, [vp, vp, vp, i32, i32, vp, vp, vp, vp, vp, vp, i32, vp,
                                       vp, vp, vp]),
    "skyrx_whiten_prepare": (C.c_int, [vp, vp, i32, vp, vp, i32, vp, vp]),
    "skyrx_score": (C.c_int, [i32, vp, i64, i32, i32, vp, vp, vp, vp, vp, i32, vp, vp, vp]),
    "skyrx_wpack_bytes": (sz, [i32]),
    "skyrx_pack_whiten": (C.c_int, [vp, i32, i32, vp, vp]),
    "skyrx_score_tc_supported": (C.c_int, [i64, i32, i32, vp]),
    "skyrx_score_tc": (C.c_int, [vp, i64, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
    "skyrx_score_rec_bytes": (sz, [i32]),
    "skyrx_score_prep": (C.c_int, [vp, vp, i32, i32, vp, vp, f64, i32, vp, vp]),
    "skyrx_score_tcs_supported": (C.c_int, [i64, i32, i32, vp]),
    "skyrx_score_tcs": (C.c_int, [vp, i64, i32, i32, vp, vp, vp, vp, vp, vp]),
    "skyrx_scorew_rec_bytes": (sz, [i32]),
    "skyrx_scorew_prep": (C.c_int, [vp, vp, i32, i32, vp, vp, f64, i32, vp, vp]),
    "skyrx_scorew_supported": (C.c_int, [i64, i32, i32, vp]),
    "skyrx_scorew": (C.c_int, [vp, i64, i32, i32, vp, vp, vp, vp, vp, vp]),
    "skyrx_mahalanobis_sq":(C.c_int, [i32, vp, i64, i32, vp, vp, vp, vp, vp]),
    "skyrx_max": (C.c_int, [vp, i64, vp, vp]),
    "skyrx_normalize": (C.c_int, [vp, i64, vp, vp, vp]),
    "skyrx_threshold": (C.c_int, [vp, i64, f32, vp, vp]),
    "skyrx_transmit_domain": (C.c_int, [vp, i64, f64, vp, vp]),
    "skyrx_topk_workspace": (sz, []),
    "skyrx_topk_threshold": (C.c_int, [vp, i64, i64, vp, vp, vp]),
    "skyrx_mask_gt": (C.c_int, [vp, i64, vp, vp, vp]),
    "skyrx_topk_init": (C.c_int, [i64, i64, vp, vp]),
    "skyrx_topk_hist": (C.c_int, [vp, i64, i32, vp, vp]),
    "skyrx_topk_pick": (C.c_int, [i32, vp, vp, vp]),
    "skyrx_topk_histogram": (vp, [vp]),
    "skyrx_topk_hist_len": (i32, []),
    "skyrx_topk_mask": (C.c_int, [vp, i64, i32, vp, vp, vp, vp, i64, vp]),
    "skyrx_link_maxima": (C.c_int, [vp, vp, i64, vp, vp]),
    "skyrx_link_payload": (C.c_int, [vp, vp, i64, vp, C.POINTER(f64), vp, vp]),
    "skyrx_link_packets": (C.c_int, [vp, vp, i32, i32, vp, vp, vp, vp]),
    "skyrx_link_frames": (C.c_int, [vp, vp, i32, i32, vp, vp, i32, i32, i32, vp, vp]),
    "skyrx_gf_matmul": (C.c_int, [vp, i64, i32, i32, vp, i64, i64, i64, vp, i64, i64, i32, vp]),
    "skyrx_gf_invert": (C.c_int, [vp, i32, vp, i32, vp, vp, i32, vp, vp, vp]),
    "skyrx_synth_raw": (C.c_int, [u32, u32, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                  i64, i64, vp, vp]),
}

_lock = threading.Lock()
_lib = None


class SkyrxCudaError(RuntimeError):
    """A CUDA or argument error inside libskyrx_b200."""


def load(path: Path | str = LIB_PATH) -> C.CDLL:
    """Load (once) and type the shared library; raises if it is not built."""
    global _lib
    with _lock:
        if _lib is None:
            p = Path(path)
            if not p.exists():
                raise SkyrxCudaError(
                    f"{p.name} is not built; run `python -m paper_2602_13509_b200.build` "
                    "(there is no CPU fallback)")
            lib = C.CDLL(str(p))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
        return _lib


def last_error() -> str:
    return (load().skyrx_last_error() or b"").decode(errors="replace")


CALLS: dict = {}   # entry point -> number of calls this process made (diagnostics)


def call(name: str, *args) -> int:
    """Invoke an int-returning entry point; raise on a non-OK status."""
    CALLS[name] = CALLS.get(name, 0) + 1
    rc = getattr(load(), name)(*args)
    if rc != OK:
        msg = last_error()
        if rc == ERR_ARG:
            raise ValueError(msg)
        raise SkyrxCudaError(f"{name} failed ({rc}): {msg}")
    return rc
