"""Patch an imported reference `skyrx` to use the B200 library (drop-in switch).

The reference chooses its kernel backend at import (_accel.py:21-31) and its
pipeline binds calibrate_bin_rgb / compute_stats / rx_scores by name at import
(pipeline.py:29, 45), so a drop-in must replace those bindings too.
"""

from __future__ import annotations

import importlib
import sys

from . import _accel, air, calibrate, datalink, errors, fec, rx

_TARGETS = {
    "calibrate": {
        "apply_calibration": calibrate.apply_calibration,
        "calibrate_bin_rgb": calibrate.calibrate_bin_rgb,
        "discard_oob_bands": calibrate.discard_oob_bands,
        "bin_bands": calibrate.bin_bands,
        "extract_rgb": calibrate.extract_rgb,
    },
    "rx": {
        "compute_stats": rx.compute_stats,
        "rx_scores": rx.rx_scores,
        "normalize_scores": rx.normalize_scores,
        "threshold_scores": rx.threshold_scores,
        "transmit_domain": rx.transmit_domain,
    },
    "datalink": {
        "pack_rgb565": datalink.pack_rgb565,
        "encode_scores_half": datalink.encode_scores_half,
        "packetize_cube": datalink.packetize_cube,
        "frames_for_cube": datalink.frames_for_cube,
    },
    "fec": {
        "ErasureCode": fec.ErasureCode,
        "gf_mat_inv": fec.gf_mat_inv,
    },
    "_accel": {
        "mahalanobis_sq": _accel.mahalanobis_sq,
        "gf256_matmul": fec.gf256_matmul,
    },
    "pipeline": {
        "calibrate_bin_rgb": calibrate.calibrate_bin_rgb,
        "compute_stats": rx.compute_stats,
        "rx_scores": rx.rx_scores,
        "transmit_domain": rx.transmit_domain,
        "packetize_cube": datalink.packetize_cube,
        "frames_for_cube": datalink.frames_for_cube,
        "run_air": air.run_air,
    },
    "": {
        "compute_stats": rx.compute_stats,
        "rx_scores": rx.rx_scores,
        "normalize_scores": rx.normalize_scores,
        "threshold_scores": rx.threshold_scores,
    },
}


def install(skyrx_module=None) -> list[str]:
    base = skyrx_module or sys.modules.get("skyrx") or importlib.import_module("skyrx")
    name = base.__name__
    ref_err = sys.modules.get(f"{name}.errors")
    if ref_err is None:
        try:
            ref_err = importlib.import_module(f"{name}.errors")
        except ImportError:
            ref_err = None
    for cls in ("FormatError", "ProtocolError"):  # raise the reference's own classes
        if ref_err is not None and hasattr(ref_err, cls):
            setattr(errors, cls, getattr(ref_err, cls))
    patched = []
    for sub, attrs in _TARGETS.items():
        mod = base if not sub else sys.modules.get(f"{name}.{sub}")
        if mod is None:
            try:
                mod = importlib.import_module(f"{name}.{sub}")
            except ImportError:
                continue
        for attr, fn in attrs.items():
            if hasattr(mod, attr):
                setattr(mod, attr, fn)
                patched.append(f"{mod.__name__}.{attr}")
    return patched
