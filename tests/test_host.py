"""CPU-side checks: the C ABI library, host logic and the no-fallback rule."""

import ctypes
import re
import sys
import types
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "skyrx_b200.h"


def header_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(skyrx_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def built_lib():
    from paper_2602_13509_b200 import build

    return build.build()


def test_header_declares_the_boundary():
    syms = header_symbols()
    for need in ("skyrx_calibrate", "skyrx_stats_accumulate", "skyrx_stats_finalize",
                 "skyrx_score", "skyrx_mahalanobis_sq", "skyrx_topk_threshold"):
        assert need in syms


def test_library_exports_every_header_symbol(built_lib):
    lib = ctypes.CDLL(str(built_lib))
    missing = [s for s in header_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_ctypes_signatures_cover_header(built_lib):
    from paper_2602_13509_b200 import _lib

    assert set(_lib.SIGNATURES) == set(header_symbols())
    lib = _lib.load()
    assert b"sm_100a" in lib.skyrx_version()
    assert lib.skyrx_moments_len(70) == 1 + 70 + 70 * 70


def test_sm100a_code_in_library(built_lib):
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(built_lib)], capture_output=True,
                         text=True)
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_without_gpu(built_lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    import paper_2602_13509_b200 as P

    raw = P.RawCube(np.zeros((4, 4, 3), np.uint16), np.linspace(400, 1000, 3),
                    gains=np.ones(4, np.float32))
    tables = P.CalibrationTables(np.zeros((4, 3)), np.ones((4, 3)))
    from paper_2602_13509_b200._lib import SkyrxCudaError

    with pytest.raises(SkyrxCudaError, match="no CUDA device"):
        P.apply_calibration(raw, tables)
    with pytest.raises(SkyrxCudaError):
        P.detect(raw, tables)


def test_host_side_errors_precede_device(built_lib):
    # the reference's ValueErrors are raised before any device work
    import paper_2602_13509_b200 as P

    raw = P.RawCube(np.zeros((2, 3, 24), np.uint16), np.linspace(400, 1000, 24),
                    gains=np.ones(2, np.float32))
    with pytest.raises(ValueError, match="invalid tables"):
        P.apply_calibration(raw, P.CalibrationTables(np.zeros((3, 23)), np.ones((3, 23))))
    bad = P.RawCube(np.zeros((2, 3, 4), np.uint16), np.linspace(400, 1000, 4),
                    gains=np.array([1.0, 0.0], np.float32))
    with pytest.raises(ValueError, match="every line gain must be positive"):
        P.apply_calibration(bad, P.CalibrationTables(np.zeros((3, 4)), np.ones((3, 4))))
    with pytest.raises(ValueError, match="positive"):
        P.CalibrationTables(np.zeros((2, 2)), np.zeros((2, 2)))
    with pytest.raises(ValueError, match="threshold"):
        P.threshold_scores(P.ScoreMap(np.zeros((2, 2))), 1.5)
    small = P.RadianceCube(np.ones((1, 3, 4), np.float32), np.linspace(400, 1000, 4))
    with pytest.raises(ValueError, match="insufficient"):
        P.compute_stats(small)
    with pytest.raises(ValueError, match="divisible"):
        P.bin_bands(P.RadianceCube(np.ones((1, 2, 7), np.float32), np.linspace(400, 1000, 7)), 4)


def test_device_scene_tables_match_oracle():
    # the product's generator recipe must equal the oracle's frozen one
    from oracle import synth as osynth
    from paper_2602_13509_b200.synth import Scene

    for args in ((1, 900, 70, 5), (3, 64, 270, 8), (5, 40, 128, 5)):
        t = osynth.make_tables(*args)
        s = Scene(*args)
        for name in ("cw24", "mean", "factor", "sd", "aspec", "asd", "xbar", "dark", "coeff"):
            assert np.array_equal(getattr(t, name), getattr(s, name)), name
        assert (s.seedkey, s.cellkey) == (t.seedkey, t.cellkey)


def test_install_patches_pipeline_bindings():
    import paper_2602_13509_b200 as P
    from paper_2602_13509_b200 import calibrate, datalink, errors, fec, rx

    fake = types.ModuleType("skyrx")
    subs = {}
    for sub in ("calibrate", "rx", "_accel", "datalink", "fec", "errors", "pipeline"):
        m = types.ModuleType(f"skyrx.{sub}")
        for attr in ("apply_calibration", "calibrate_bin_rgb", "compute_stats", "rx_scores",
                     "mahalanobis_sq", "transmit_domain", "packetize_cube", "pack_rgb565", "frames_for_cube",
                     "ErasureCode", "gf256_matmul", "run_air"):
            setattr(m, attr, None)
        subs[sub] = m
    fake.compute_stats = None
    saved_err = (errors.FormatError, errors.ProtocolError)

    class RefProtocolError(ValueError):
        pass

    subs["errors"].ProtocolError = RefProtocolError
    saved = {k: sys.modules.get(k) for k in ["skyrx"] + [f"skyrx.{s}" for s in subs]}
    try:
        sys.modules["skyrx"] = fake
        for s, m in subs.items():
            sys.modules[f"skyrx.{s}"] = m
        patched = P.install(fake)
        assert subs["pipeline"].compute_stats is rx.compute_stats
        assert subs["pipeline"].calibrate_bin_rgb is calibrate.calibrate_bin_rgb
        assert subs["_accel"].mahalanobis_sq is not None
        assert fake.compute_stats is rx.compute_stats
        assert "skyrx.pipeline.rx_scores" in patched
        assert subs["pipeline"].packetize_cube is datalink.packetize_cube
        assert subs["datalink"].pack_rgb565 is datalink.pack_rgb565
        assert subs["pipeline"].frames_for_cube is datalink.frames_for_cube
        assert subs["pipeline"].run_air is P.run_air
        assert subs["fec"].ErasureCode is fec.ErasureCode
        assert errors.ProtocolError is RefProtocolError
        assert subs["_accel"].gf256_matmul is fec.gf256_matmul
    finally:
        errors.FormatError, errors.ProtocolError = saved_err
        for k, v in saved.items():
            if v is None:
                sys.modules.pop(k, None)
            else:
                sys.modules[k] = v


def test_topk_count_definition():
    from paper_2602_13509_b200.rx import topk_count
    from oracle.skyrx_oracle import topk_count as ok

    for n in (0, 1, 999, 1000, 1001, 1843200, 224100, 8388608, 14745600, 268435456):
        assert topk_count(n) == ok(n)
    assert topk_count(1843200) == 1844
