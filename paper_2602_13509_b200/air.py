"""The air side's four-stage pipeline on CUDA streams.

Drop-in for `skyrx.pipeline.run_air` (pipeline.py:152-235) given a flight's cubes: the same
stages (save -> calibrate -> detect -> transmit), each on its own worker thread with a
bounded queue of `queue_depth` cubes between stages (pipeline.py:132-149, 182-208), the same
stage-isolation contract (a stage that raises drops that cube, logged as
"(cube_id, '<stage>: <error>')") and the same outputs (frames, per-cube StageTiming, raw
ScoreMaps, RGB images, dropped list).

What is B200-specific is what flows between the stages: device tensors on per-stage CUDA
streams, ordered by CUDA events, not host arrays.
  save       ingest (.hsc straight into pinned memory, formats.read_cube) + optional .hsc
             write + the raw cube's H2D on the save stream
  calibrate  fused calibrate -> OOB discard -> 4x bin -> RGB (skyrx_calibrate), in HBM
  detect     moments + factor (compute_stats) + scores (rx_scores) in HBM; the only host
             sync of the cube is the stats check (non-finite / not-PD raise here, as in the
             reference)
  transmit   device line packets + RS parity of every group (datalink.cube_frames), one D2H
             of packets + parity, frames assembled on the host
Results do not depend on scheduling, so the frame stream is byte-identical for any
queue depth (pipeline.py:7-8; tests/test_gpu_air.py).  Stage times are device times of the
stage's work (CUDA events on its stream) plus the host work it does.
"""

from __future__ import annotations

import logging
import queue
import sys
import threading
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _dev, formats
from .calibrate import calibrate_bin_rgb, tables_of
from .cube import RawCube, ScoreMap
from .datalink import cube_frames_device
from .rx import compute_stats, rx_scores

log = logging.getLogger("paper_2602_13509_b200.air")

_DONE = object()
STAGES = ("save", "calibrate", "detect", "transmit")


@dataclass(frozen=True)
class StageTiming:
    """evaluate.py:97-109: seconds spent on one cube in each air-side stage."""

    save_s: float
    calibrate_s: float
    detect_s: float
    transmit_s: float

    STAGES = STAGES

    def as_tuple(self) -> tuple[float, float, float, float]:
        return (self.save_s, self.calibrate_s, self.detect_s, self.transmit_s)


@dataclass
class AirResult:
    """pipeline.py:119-127: everything the air side produced, in cube order."""

    frames: list
    timings: list
    scores: list
    rgb: list
    dropped: list


_tls = threading.local()


class _Timer:
    """Host seconds + device seconds (event pair on the stage's stream) of one stage; the
    device interval starts once the upstream stage's work is done (see _adopt)."""

    def __init__(self, stream: torch.cuda.Stream):
        self.stream = stream
        self.t0 = time.perf_counter()
        self.host = 0.0
        self.a = torch.cuda.Event(enable_timing=True)
        self.b = torch.cuda.Event(enable_timing=True)
        self.a.record(stream)
        _tls.timer = self

    def stop(self):
        self.b.record(self.stream)
        self.host = time.perf_counter() - self.t0
        return self

    def seconds(self) -> float:
        self.b.synchronize()
        return max(self.host, self.a.elapsed_time(self.b) * 1e-3)


def _worker(name, fn, stream, q_in, q_out, dropped, lock):
    dev = _dev.require_cuda()
    torch.cuda.set_device(dev)
    with torch.cuda.stream(stream):
        while True:
            item = q_in.get()
            if item is _DONE:
                q_out.put(_DONE)
                return
            cube_id, payload, timing = item
            t = _Timer(stream)
            try:
                result = fn(cube_id, payload)
            except Exception as exc:  # noqa: BLE001 - stage isolation is the contract
                log.error("cube %d dropped in %s stage: %s", cube_id, name, exc)
                with lock:
                    dropped.append((cube_id, f"{name}: {exc}"))
                continue
            timing[name] = t.stop()
            q_out.put((cube_id, result, timing))


def _handoff(stream: torch.cuda.Stream) -> torch.cuda.Event:
    """The event the next stage waits on: this stage's work on its stream is done."""
    ev = torch.cuda.Event()
    ev.record(stream)
    return ev


def _adopt(ev: torch.cuda.Event, tensors):
    """Order this stage's stream after the upstream event and tell the caching allocator
    the handed-over tensors are in use on this stream too."""
    s = torch.cuda.current_stream()
    s.wait_event(ev)
    for t in tensors:
        if isinstance(t, torch.Tensor) and t.is_cuda:
            t.record_stream(s)
    timer = getattr(_tls, "timer", None)
    if timer is not None:
        timer.a.record(s)


class _Staging:
    """Reused pinned buffers for the transmit stage's D2H: a fresh cudaHostAlloc per cube
    (what a pinned to_host would do for results that are kept) stalls the other stages'
    CUDA calls; results are copied out of the staging into ordinary host memory."""

    def __init__(self):
        self.bufs: dict = {}

    def fetch(self, tensors):
        s = torch.cuda.current_stream()
        outs = []
        for i, t in enumerate(tensors):
            nbytes = t.numel() * t.element_size()
            buf = self.bufs.get(i)
            if buf is None or buf.numel() < nbytes:
                buf = self.bufs[i] = torch.empty(max(nbytes, 1), dtype=torch.uint8,
                                                 pin_memory=True)
            view = buf[:nbytes].view(t.dtype).view(t.shape)
            view.copy_(t, non_blocking=True)
            outs.append(view)
        s.synchronize()
        return [o.numpy() for o in outs]


def run_air(config, data, *, mode: str = "precise") -> AirResult:
    """pipeline.py:152-235 over `data.cubes` (RawCube objects or `.hsc` paths) with
    `data.tables`.  `config` needs `bin_factor`, `queue_depth`, `out_dir` (a reference
    PipelineConfig works; its `validate()` is called).  Scene synthesis (pipeline.py:91-103)
    is the reference's generator and out of scope: pass the flight's cubes."""
    if hasattr(config, "validate"):
        config.validate()
    elif getattr(config, "queue_depth", 1) < 1:
        raise ValueError("queue depth must be >= 1")
    if data is None:
        # scene synthesis is the reference's generator (pipeline.py:91-103), not this path:
        # use the caller's own `synthesize` when the config is the reference's
        mod = sys.modules.get(type(config).__module__)
        synthesize = getattr(mod, "synthesize", None)
        if synthesize is None:
            raise ValueError("run_air needs the flight's cubes (data=None needs the "
                             "reference's synthesize)")
        data = synthesize(config)
    tables = tables_of(data.tables)
    factor = int(getattr(config, "bin_factor", 4))
    depth = int(getattr(config, "queue_depth", 3))
    out_dir = getattr(config, "out_dir", None)
    out_dir = Path(out_dir) if out_dir is not None else None
    if out_dir is not None:
        out_dir.mkdir(parents=True, exist_ok=True)
    _dev.require_cuda()
    streams = {n: torch.cuda.Stream() for n in STAGES}

    def save_stage(cube_id: int, item):
        if isinstance(item, (str, Path)):
            cube = formats.read_cube(item)        # payload straight into pinned memory
        else:
            cube = item
        if out_dir is not None:
            formats.write_cube(out_dir / f"cube_{cube_id:04d}.hsc", cube)
        v = cube.values
        if isinstance(v, torch.Tensor):
            dv = v.to(_dev.require_cuda(), non_blocking=v.is_pinned()) if not v.is_cuda else v
        else:
            dv = _dev.to_device(np.asarray(v), torch.uint16)
        dev_cube = RawCube(dv, cube.wavelengths_nm, cube.line_meta)
        return dev_cube, _handoff(streams["save"])

    def calibrate_stage(cube_id: int, payload):
        raw, ev = payload
        _adopt(ev, [raw.values])
        binned, rgb = calibrate_bin_rgb(raw, tables, factor=factor)
        return (binned, rgb), _handoff(streams["calibrate"])

    def detect_stage(cube_id: int, payload):
        (binned, rgb), ev = payload
        _adopt(ev, [binned.values, rgb])
        stats = compute_stats(binned, mode=mode)
        scores = rx_scores(binned, stats, mode=mode)
        return (binned.line_meta, rgb, scores), _handoff(streams["detect"])

    staging = _Staging()

    def transmit_stage(cube_id: int, payload):
        (line_meta, rgb, scores), ev = payload
        _adopt(ev, [scores.values, rgb])
        fr = cube_frames_device(cube_id, rgb, scores.values, line_meta)
        fh, rh, sh = staging.fetch([fr, rgb, scores.values])
        return [row.tobytes() for row in fh], rh.copy(), ScoreMap(sh.copy())

    fns = dict(save=save_stage, calibrate=calibrate_stage, detect=detect_stage,
               transmit=transmit_stage)
    queues = [queue.Queue(maxsize=depth) for _ in range(len(STAGES) + 1)]
    dropped: list = []
    lock = threading.Lock()
    workers = [threading.Thread(target=_worker, args=(n, fns[n], streams[n], queues[i],
                                                      queues[i + 1], dropped, lock), daemon=True)
               for i, n in enumerate(STAGES)]
    for w in workers:
        w.start()

    def feed():
        for cube_id, raw in enumerate(data.cubes):
            queues[0].put((cube_id, raw, {}))
        queues[0].put(_DONE)

    feeder = threading.Thread(target=feed, daemon=True)
    feeder.start()
    finished = {}
    while True:
        item = queues[-1].get()
        if item is _DONE:
            break
        cube_id, result, timing = item
        finished[cube_id] = (result, timing)
    feeder.join()
    for w in workers:
        w.join()

    out = AirResult(frames=[], timings=[], scores=[], rgb=[], dropped=sorted(dropped))
    for cube_id in sorted(finished):
        (frames, rgb, scores), timing = finished[cube_id]
        out.frames.extend(frames)
        out.timings.append(StageTiming(*(timing[n].seconds() for n in STAGES)))
        out.scores.append(scores)
        out.rgb.append(rgb)
    return out
