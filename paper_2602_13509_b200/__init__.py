"""paper_2602_13509_b200: B200-native calibrate + RX hot path of skyrx (arXiv 2602.13509).

Mirrors the reference package's public surface (skyrx/__init__.py:3-35 plus
skyrx.calibrate and skyrx._accel.mahalanobis_sq) and runs it in hand-written
sm_100a CUDA kernels behind the C ABI in include/skyrx_b200.h.
"""

from .cube import (
    GroundTruthMask,
    InsSample,
    LineMeta,
    RadianceCube,
    RawCube,
    ScoreMap,
    band_nearest,
)
from .calibrate import (
    CalibrationTables,
    apply_calibration,
    bin_bands,
    calibrate_bin_rgb,
    discard_oob_bands,
    extract_rgb,
)
from .rx import (
    CubeStats,
    DetectPlan,
    DeviceStats,
    compute_stats,
    detect,
    detect_batch,
    normalize_scores,
    rx_scores,
    threshold_scores,
    topk_mask,
    transmit_domain,
)
from .stream import ChunkResult, StreamingRX
from .strips import StripBatch, StripsResult, detect_strips, shard_strips
from .datalink import (cube_frames, encode_scores_half, frames_for_cube, link_payload,
                       pack_rgb565, packetize_cube)
from .air import AirResult, StageTiming, run_air
from .fec import ErasureCode
from .formats import read_cube, write_cube

__version__ = "0.1.0"

__all__ = [
    "GroundTruthMask", "InsSample", "LineMeta", "RadianceCube", "RawCube", "ScoreMap",
    "band_nearest", "CalibrationTables", "apply_calibration", "bin_bands", "calibrate_bin_rgb",
    "discard_oob_bands", "extract_rgb", "CubeStats", "DetectPlan", "DeviceStats",
    "compute_stats", "detect", "detect_batch", "normalize_scores", "rx_scores", "threshold_scores",
    "topk_mask", "transmit_domain", "StreamingRX", "ChunkResult", "install",
    "StripBatch", "StripsResult", "detect_strips", "shard_strips", "__version__",
    "link_payload", "pack_rgb565", "encode_scores_half", "packetize_cube", "frames_for_cube",
    "cube_frames", "ErasureCode", "run_air", "AirResult", "StageTiming", "read_cube",
    "write_cube",
]


def install(skyrx_module=None):
    """Route an imported reference ``skyrx`` package through this library.

    Patches skyrx.calibrate / skyrx.rx / skyrx._accel and the names
    skyrx.pipeline bound at import (pipeline.py:29, 45), like selecting a
    backend with SKYRX_NO_NUMBA (_accel.py:21-31).  Returns the list of
    patched attributes.
    """
    from .install import install as _install

    return _install(skyrx_module)
