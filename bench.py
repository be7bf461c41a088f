"""Throughput of the fused calibrate + RX hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--config c4|c1|c3|c5] [--impl b200|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Default workload = BASELINE config 4 ("multi-strip batch"): 64 independent
strips of 16384 lines x 900 samples x 70 bands of 12-bit raw counts, each
with its own seeded mixture (seed 4000+i) and its own background; strips are
dealt round-robin to ranks (no collective).  One step = every strip of this
rank through raw -> shift -> fused calibrate+moments -> batched Cholesky /
inverse -> fused calibrate+score -> top-0.1% radix select -> mask.  Inputs
are generated on the device (bit-identical to oracle/synth.py) and resident
in HBM before timing; the inputs (132 GB at N=1) exceed L2 many times over.

`value` = pixels of all ranks / max-over-ranks device time of K steps.
`e2e`   = the same path through the public API `detect()` on HOST numpy
          cubes (H2D of raw + D2H of scores, mask and stats inside the
          timed region), over a bounded number of strips per step.
`--impl reference` times the CPU oracle port (oracle/skyrx_oracle.py, the
reference's numpy/LAPACK path) on a bounded sample on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "c1": dict(lines=2048, samples=900, bands=70, components=5, seed=1, strips=1),
    "c2": dict(lines=249, samples=900, bands=70, components=5, seed=2, strips=1, chunks=60,
               forget=0.99),
    "c3": dict(lines=8192, samples=1024, bands=270, components=8, seed=3, strips=1),
    "c4": dict(lines=16384, samples=900, bands=70, components=5, seed=4000, strips=64),
    "c5": dict(lines=131072, samples=2048, bands=128, components=5, seed=5, strips=1),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--strips", type=int, default=None, help="override strip count (testing)")
    ap.add_argument("--lines", type=int, default=None, help="override lines per strip (testing)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-strips", type=int, default=4)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the oracle check of strip 0 after the timed region")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch every step eagerly instead of replaying one captured CUDA graph")
    return ap.parse_args()


def bytes_per_pixel(bands: int) -> int:
    # 2B raw read (moments) + 2B raw read (score) + 4 (f32 delta) + 1 (mask)
    return 4 * bands + 5


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = Path(f"/tmp/skyrx_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None or not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        if not self.path.read_text().strip():  # timed region shorter than one period
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu),
                                      f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=20).stdout
                self.path.write_text(out)
            except (OSError, subprocess.TimeoutExpired):
                pass
        sm, smax, reasons, power = [], None, set(), []
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.path.read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
                power.append(float(parts[3]))
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w": statistics.median(power) if power else None,
                "power_w_max": max(power) if power else None}


# ----------------------------------------------------------------------------- reference arm
def import_reference():
    """The UNMODIFIED reference package, installed once with
    ``pip install --no-index --no-build-isolation --no-deps --target baseline/_ref``
    from a copy of /root/reference/pkg.  None when absent."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "skyrx" / "rx.py").exists():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_skyrx_ref")
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import skyrx._accel
    import skyrx.calibrate
    import skyrx.cube
    import skyrx.rx
    return skyrx


def host_info():
    info = {"cpu_count": os.cpu_count()}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        import threadpoolctl

        info["blas_threads"] = sorted({d.get("num_threads") for d in
                                       threadpoolctl.threadpool_info()
                                       if d.get("user_api") == "blas"})
    except Exception:
        pass
    return info


class ReferenceDetect:
    """One bounded sample of the workload through the reference's own public API:
    skyrx.calibrate.apply_calibration -> skyrx.rx.compute_stats -> skyrx.rx.rx_scores
    (its default numba scorer, _accel.py:75-90, or the numpy one with ``numpy=True``,
    _accel.py:33-47) -> the top-0.1 % mask (R-TOPK is not in the reference: the
    oracle's np.partition restatement).  Falls back to the oracle port when the
    reference is not installed."""

    def __init__(self, raw, dark, coeff, B, numpy_scorer=False):
        from oracle import skyrx_oracle as O

        self.O = O
        self.raw, self.dark, self.coeff = raw, dark, coeff
        self.sk = import_reference()
        self.kind = "reference" if self.sk is not None else "port"
        if self.sk is not None:
            sk = self.sk
            ins = sk.cube.InsSample(0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0)
            meta = tuple(sk.cube.LineMeta(i, 1.0, ins, ins) for i in range(raw.shape[0]))
            self.cube = sk.cube.RawCube(raw, np.linspace(400, 1000, B), meta)
            self.tables = sk.calibrate.CalibrationTables(dark, coeff)
            self.scorer = (sk._accel.mahalanobis_sq_numpy if numpy_scorer
                           else sk._accel.mahalanobis_sq)
            self.backend = ("numpy (SKYRX_NO_NUMBA path)" if numpy_scorer or not
                            sk._accel.HAS_NUMBA else "numba (default)")
        else:
            self.backend = "oracle port (numpy/OpenBLAS/LAPACK)"

    def __call__(self):
        if self.sk is None:
            return self.O.detect(self.raw, self.dark, self.coeff, np.ones(self.raw.shape[0]))
        sk = self.sk
        keep = sk._accel.mahalanobis_sq
        sk._accel.mahalanobis_sq = self.scorer   # rx.py:96 looks it up per call
        try:
            rad = sk.calibrate.apply_calibration(self.cube, self.tables)
            st = sk.rx.compute_stats(rad)
            sc = sk.rx.rx_scores(rad, st)
        finally:
            sk._accel.mahalanobis_sq = keep
        return st, sc.values, self.O.topk_mask(sc.values)


def time_reference(raw, dark, coeff, B, steps, warmup, budget_s=None, numpy_scorer=False):
    """Mean seconds per call of ReferenceDetect on ``raw`` (warm-up untimed)."""
    fn = ReferenceDetect(raw, dark, coeff, B, numpy_scorer)
    for _ in range(max(warmup, 1)):
        fn()
    times = []
    t0 = time.perf_counter()
    for _ in range(max(steps, 1)):
        a = time.perf_counter()
        fn()
        times.append(time.perf_counter() - a)
        if budget_s is not None and time.perf_counter() - t0 > budget_s:
            break
    return float(np.mean(times)), len(times), fn


def cpu_sample_lines(cfg, lines):
    return min(lines, 512 if cfg["bands"] <= 128 else 96)


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    from oracle import synth as osynth

    lines = args.lines or cfg["lines"]
    sample_lines = cpu_sample_lines(cfg, lines)
    t = osynth.make_tables(cfg["seed"], cfg["samples"], cfg["bands"], cfg["components"])
    raw = osynth.generate_lines(t, 0, sample_lines)
    sec, reps, fn = time_reference(raw, t.dark, t.coeff, cfg["bands"], args.steps, args.warmup)
    px = sample_lines * cfg["samples"]
    value = px / sec
    hi = host_info()
    line = {
        "impl": "reference", "metric": "calibrated+RX-scored pixels/sec", "value": value,
        "unit": "pixels/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32 radiance, f64 stats and scores",
        "data": "synthetic (oracle/synth.py, seeded)",
        "config": config_key(args, cfg, world),
        "cpu_baseline": {"value": value, "unit": "pixels/s", "cores": hi["cpu_count"],
                         "kind": fn.kind,
                         "sample": f"{sample_lines} lines x {cfg['samples']} samples of strip 0 "
                                   f"(seed {cfg['seed']}) per step, {reps} steps; "
                                   + ("skyrx apply_calibration -> compute_stats -> rx_scores "
                                      f"[{fn.backend}] -> top-0.1% mask (baseline/_ref)"
                                      if fn.kind == "reference" else
                                      f"oracle detect [{fn.backend}]"),
                         "host": hi},
        "e2e": {"value": value, "unit": "pixels/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_key(args, cfg, world):
    lines = args.lines or cfg["lines"]
    strips = args.strips or cfg["strips"]
    return {"workload": {"c1": "single strip 2048x900x70", "c3": "high-band cube 8192x1024x270",
                         "c2": "streaming 60 x 249-line chunks of 900x70, forgetting 0.99",
                         "c4": "multi-strip batch 64 x (16384x900x70)",
                         "c5": "global mosaic 131072x2048x128"}[args.config]
            + ("" if (args.lines is None and args.strips is None) else " (resized)"),
            "config": args.config, "lines": lines, "samples": cfg["samples"],
            "bands": cfg["bands"], "strips": strips, "parallelism": f"strips/dp{world}",
            "l2": "inputs larger than L2 (no flush needed)"
            if strips * lines * cfg["samples"] * cfg["bands"] * 2 > 4 * 126e6 else
            "L2 flushed between steps"}


# ----------------------------------------------------------------------------- b200 arm
def free_port() -> int:
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def launch(args):
    """--gpus N without a torchrun environment: re-exec under torchrun with N
    ranks (one process per GPU, NCCL).  Under torchrun, WORLD_SIZE must equal
    --gpus.  Returns (rank, world, local)."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is None and args.gpus > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               f"--master-port={free_port()}", str(Path(__file__).resolve())] + sys.argv[1:]
        sys.stdout.flush()
        os.execv(sys.executable, cmd)
    world = int(ws or "1")
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; launch with "
                         f"torchrun --nproc-per-node {args.gpus} or without torchrun")
    return int(os.environ.get("RANK", "0")), world, int(os.environ.get("LOCAL_RANK", "0"))


def init_dist(local):
    """One NCCL process group whenever torchrun launched us (N = 1 included, so
    the collectives of the multi-GPU path run even on a one-GPU lease)."""
    import torch
    import torch.distributed as dist

    if torch.cuda.device_count() <= local:
        raise SystemExit(f"bench: LOCAL_RANK {local} but only {torch.cuda.device_count()} GPUs")
    torch.cuda.set_device(local)
    if "WORLD_SIZE" in os.environ and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return dist.is_initialized()


def main():
    args = parse()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        ws = os.environ.get("WORLD_SIZE")
        return run_reference(args, cfg, int(os.environ.get("RANK", "0")),
                             int(ws) if ws else args.gpus)
    rank, world, local = launch(args)
    if args.config == "c2":
        return run_stream(args, cfg, rank, world, local)
    if args.config == "c5":
        return run_global(args, cfg, rank, world, local)

    import torch
    import torch.distributed as dist

    distributed = init_dist(local)
    import paper_2602_13509_b200 as P
    from paper_2602_13509_b200 import _dev
    from paper_2602_13509_b200.strips import StripBatch, needs_redo, shard_strips
    from paper_2602_13509_b200.synth import Scene

    lines = args.lines or cfg["lines"]
    S, B = cfg["samples"], cfg["bands"]
    nstrips = args.strips or cfg["strips"]
    # the package's strip sharding (strips.shard_strips: strip i -> rank i % world)
    mine = shard_strips(nstrips, rank, world)
    if not mine:
        raise SystemExit(f"bench: {nstrips} strips leave rank {rank} of {world} without work")
    npix = lines * S
    scenes = [Scene(cfg["seed"] + i if nstrips > 1 else cfg["seed"], S, B, cfg["components"])
              for i in mine]
    raws = [sc.generate(0, lines) for sc in scenes]
    tabs = [(_dev.to_device(sc.dark), _dev.to_device(sc.coeff)) for sc in scenes]
    gains_t = _dev.to_device(np.ones(lines, np.float32))
    gains = [gains_t] * len(mine)
    gconst = [1.0] * len(mine)   # every line gain 1.0; tables are finite
    batch = StripBatch(lines, S, B, len(mine))
    plan = batch.plan
    stream = torch.cuda.current_stream()
    flush = None
    if len(mine) * npix * B * 2 <= 4 * 126e6:
        flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    ev = {"gram": [], "score": []}
    step_ev = []

    def pair():
        return (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))

    def step(instrument=False):
        if flush is not None:
            flush.zero_()  # outside the per-step events below
        if instrument:
            sa, sb = pair()
            sa.record(stream)
            gev = [pair() for _ in mine]
            kev = [pair() for _ in mine]
            ev["gram"] += gev
            ev["score"] += kev
        batch.enqueue(raws, tabs, gains, gconst,
                      moment_events=gev if instrument else None,
                      score_events=kev if instrument else None)
        if instrument:
            sb.record(stream)
            step_ev.append((sa, sb))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    batch.verify(raws, tabs, gains)
    # the step as one CUDA graph (every kernel of every strip, no host work between
    # launches); inputs larger than L2 only — the L2-flushed configs time eager steps
    graph = None
    if not args.no_graph and flush is None:
        launches0 = plan.launches
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                step()
            launches = plan.launches - launches0
            for _ in range(args.warmup):
                graph.replay()
            torch.cuda.synchronize()
        except Exception as e:  # capture refused: time eager steps instead
            print(f"bench: CUDA graph capture failed ({e}); eager steps", file=sys.stderr)
            graph = None
            torch.cuda.synchronize()
            step()
            torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = plan.launches
    with ClockSampler(local) as clocks:
        start.record(stream)
        for _ in range(args.steps):
            if graph is not None:
                graph.replay()
            else:
                step(instrument=True)
        end.record(stream)
        torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    ms = start.elapsed_time(end)
    if flush is not None:  # device time of the steps themselves, L2 flushes excluded
        ms = float(sum(a.elapsed_time(b) for a, b in step_ev))
    if graph is None:
        launches = (plan.launches - launches0) // args.steps
    # what the timed steps produced, checked before anything else runs: status and
    # flags of EVERY strip of this rank (a clamp, a counts >= 4096 or a missing
    # no-clamp proof would mean the timed kernels computed the wrong thing)
    st, fl = batch.flags()
    bad = int(sum(1 for a, f in zip(st, fl) if a != 0 or needs_redo(f) or f & 4))
    if graph is not None:
        # per-kernel events (roofline) from eager steps, outside the timed region
        for _ in range(max(1, min(args.steps, 2))):
            step(instrument=True)
        torch.cuda.synchronize()
    if distributed:
        t = torch.tensor([ms, float(bad)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0].item())
        tb = torch.tensor([bad], device="cuda", dtype=torch.int64)
        dist.all_reduce(tb, op=dist.ReduceOp.SUM)
        bad = int(tb.item())
    total_px = nstrips * npix * args.steps
    value = total_px / (ms / 1e3)

    # dominant kernel and its roofline: CUDA events on `stream` around each
    # kernel call alone (moments: 2B raw read per pixel; fused calibrate+score:
    # 2B raw read + 4 B f32 delta write per pixel)
    gram_k_ms = float(np.mean([a.elapsed_time(b) for a, b in ev["gram"]]))
    kern_ms = float(np.mean([a.elapsed_time(b) for a, b in ev["score"]]))
    peak, peak_kind = load_peaks()
    if B > 128:
        gname, sname = "raww_gram_kernel (+scan, per-pass)", "score_tcw_kernel"
    else:
        gname = "gram_raw_kernel (+reduce)"
        sname = ("score_tcs_kernel" if plan.tcs else
                 "score_tc_kernel" if plan.tc else "score_kernel")
    g_bytes, s_bytes = npix * 2 * B, npix * (2 * B + 4)
    if gram_k_ms > kern_ms:
        kname, dom_bytes, dom_ms, other = gname, g_bytes, gram_k_ms, (sname, kern_ms, s_bytes)
    else:
        kname, dom_bytes, dom_ms, other = sname, s_bytes, kern_ms, (gname, gram_k_ms, g_bytes)
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    traffic = ncu_traffic(kname, (lines, S, B))

    line = {
        "metric": "calibrated+RX-scored pixels/sec", "value": value, "unit": "pixels/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32 (fp64 stats accumulation, fp64 factorisation)",
        "data": "synthetic (seeded device generator, bit-identical to oracle/synth.py)",
        "config": config_key(args, cfg, world),
        "hbm_fraction_whole_path": value / world * bytes_per_pixel(B) / (peak * 1e9),
        "roofline": {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic,
                     "bytes_per_launch": dom_bytes, "ms_per_launch": dom_ms,
                     "other_pass": {"kernel": other[0], "ms_per_launch": other[1],
                                    "bytes_per_launch": other[2],
                                    "frac": other[2] / (other[1] / 1e3) / 1e9 / peak}},
        "gpu_launches": launches,
        "launch_mode": "cuda_graph (one captured step replayed)" if graph is not None else "eager",
        "clocks": clocks.summary(),
    }
    parity = {"strips_checked": nstrips, "strips_not_ok": bad,
              "check": "status == OK and flags & (2|4|16|32) == 0 (no clamp, no quantiser or "
                       "digit-range fallback) for every strip of every rank after the timed steps"}
    if bad:
        line["invalid"] = f"{bad} strips did not take the timed fast path"
    if rank == 0 and not args.no_parity:
        parity.update(strip_parity(batch, raws[0], scenes[0], lines, cfg, mine[0]))
    line["parity"] = parity
    if rank == 0 and not args.no_e2e:
        line["e2e"] = measure_e2e(args, P, cfg, lines, scenes[: max(1, args.e2e_strips)])
    if rank == 0 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(cfg, raws[0], scenes[0], lines)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()


def ncu_traffic(kname, geometry):
    """dram read+write bytes per launch of that kernel from the committed
    `ncu --set full` capture of this geometry (profiles/ncu_traffic.json)."""
    tp = ROOT / "profiles" / "ncu_traffic.json"
    if not tp.exists():
        return None
    try:
        tj = json.loads(tp.read_text())
        for entry in tj if isinstance(tj, list) else [tj]:
            if entry.get("geometry") == list(geometry):
                return entry.get(kname.split()[0])
    except Exception:
        return None
    return None


def strip_parity(batch, raw_dev, scene, lines, cfg, index):
    """The timed outputs of this rank's first strip against the CPU oracle on the
    same raw counts (BASELINE tolerances: stats 1e-5, scores 1e-4 per pixel, mask
    exact outside the 1e-4 band around the threshold), plus the Sigma^-1 error
    split into its two parts: ours vs the reference's algorithm
    on EXACT radiance, and the reference's own f32-radiance rounding."""
    from oracle import skyrx_oracle as O

    t0 = time.perf_counter()
    raw = raw_dev.cpu().numpy()
    det = batch.detection(0, host=True)
    gains = np.ones(lines)
    want_stats, want_sc, want_mask = O.detect(raw, scene.dark, scene.coeff, gains)
    exact = O.compute_stats_exact(raw, scene.dark, scene.coeff, gains)

    def nw(a, b):
        return float(np.abs(np.asarray(a) - np.asarray(b)).max() / np.abs(np.asarray(b)).max())

    rel = np.abs(det.scores - want_sc) / np.maximum(want_sc, 1e-12)
    thr = O.topk_threshold(want_sc)
    differ = det.mask != want_mask
    near = np.abs(want_sc - thr) <= 1e-4 * abs(thr)
    out = {
        "strip": index, "pixels": int(want_sc.size),
        "mu_rel": nw(det.stats.mu, want_stats.mu),
        "sigma_rel": nw(det.stats.sigma, want_stats.sigma),
        "sigma_inv_rel": nw(det.stats.sigma_inv, want_stats.sigma_inv),
        "sigma_inv_rel_vs_exact_radiance": nw(det.stats.sigma_inv, exact.sigma_inv),
        "reference_f32_rounding_sigma_inv_rel": nw(want_stats.sigma_inv, exact.sigma_inv),
        "ridge_equal": det.stats.ridge_used == want_stats.ridge_used,
        "score_max_rel": float(rel.max()),
        "threshold_rel": abs(det.threshold - thr) / abs(thr),
        "mask_differ": int(differ.sum()), "mask_differ_outside_band": int((differ & ~near).sum()),
        "tolerances": {"stats": 1e-5, "scores": 1e-4, "mask_band": 1e-4},
        "oracle_s": time.perf_counter() - t0,
    }
    out["pass"] = bool(out["mu_rel"] < 1e-5 and out["sigma_rel"] < 1e-5 and out["ridge_equal"]
                       and out["score_max_rel"] < 1e-4 and out["mask_differ_outside_band"] == 0)
    return out


# ----------------------------------------------------------------------------- c2: streaming
def run_stream(args, cfg, rank, world, local):
    """BASELINE config 2: per-chunk latency and sustained throughput of StreamingRX.

    Replicas only (streaming is single-GPU latency work); every
    rank runs its own stream, rank 0 reports.  `value` = chunk pixels per
    second with chunks resident in HBM (device events around K steps of the
    whole 60-chunk stream); `e2e` = the same through update() on pinned host
    chunks (H2D, graph replay, D2H of scores + mask, host sync per chunk)."""
    import torch

    init_dist(local)
    import paper_2602_13509_b200 as P
    from paper_2602_13509_b200.stream import StreamingRX
    from paper_2602_13509_b200.synth import Scene

    L, S, B, nch = cfg["lines"], cfg["samples"], cfg["bands"], cfg["chunks"]
    sc = Scene(cfg["seed"] + rank, S, B, cfg["components"])
    tabs = P.CalibrationTables(sc.dark, sc.coeff)
    raw = sc.generate(0, L * nch)
    chunks = [raw[i * L:(i + 1) * L] for i in range(nch)]
    stream = torch.cuda.current_stream()

    def one_pass(srx, src, lat=None):
        for c in src:
            if lat is not None:
                t0 = time.perf_counter()
            srx.update(c)
            if lat is not None:
                lat.append((time.perf_counter() - t0) * 1e3)

    srx = StreamingRX(tabs, L, cfg["forget"])
    l0 = srx.plan.launches
    srx.update(chunks[0])
    per_chunk = srx.plan.launches - l0 + 4  # + shift, accumulate, fold, flag reset
    srx.reset()
    for _ in range(args.warmup):
        srx.reset()
        one_pass(srx, chunks)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lat_dev = []
    with ClockSampler(local) as clocks:
        start.record(stream)
        for _ in range(args.steps):
            srx.reset()
            one_pass(srx, chunks, lat_dev)
        end.record(stream)
        torch.cuda.synchronize()
    ms = start.elapsed_time(end)
    px = L * S * nch * args.steps
    value = px / (ms / 1e3)
    # e2e: pinned host chunks through the public update()
    hosts = [c.cpu().pin_memory().numpy() for c in chunks]
    srx_h = StreamingRX(tabs, L, cfg["forget"])
    one_pass(srx_h, hosts[:3])
    lat = []
    srx_h.reset()
    t0 = time.perf_counter()
    one_pass(srx_h, hosts, lat)
    sec = time.perf_counter() - t0
    if rank != 0:
        return
    pct = lambda a, q: float(np.percentile(a, q))  # noqa: E731
    line = {
        "metric": "calibrated+RX-scored pixels/sec", "value": value, "unit": "pixels/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 (fp64 moments, fold and factorisation)",
        "data": "synthetic (seeded device generator, bit-identical to oracle/synth.py)",
        "config": config_key(args, cfg, world) | {"parallelism": f"replicas{world}"},
        "latency_ms_per_chunk": {"device_resident": {"p50": pct(lat_dev, 50),
                                                     "p99": pct(lat_dev, 99),
                                                     "max": max(lat_dev)},
                                 "host_e2e": {"p50": pct(lat, 50), "p99": pct(lat, 99),
                                              "max": max(lat)},
                                 "realtime_budget": 1000.0},
        "gpu_launches": per_chunk * nch,
        "clocks": clocks.summary(),
        "e2e": {"value": L * S * nch / sec, "unit": "pixels/s",
                "h2d_bytes_per_step": L * S * B * 2 * nch,
                "d2h_bytes_per_step": L * S * 5 * nch,
                "api": "paper_2602_13509_b200.StreamingRX.update(numpy chunk)"},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- c5: global mosaic
def run_global(args, cfg, rank, world, local):
    """BASELINE config 5: one background over line blocks, NCCL all-reduce of
    FP64 moments + radix histograms (paper_2602_13509_b200/distributed.py).
    Total work fixed (131072 lines split over the ranks): strong scaling."""
    import torch
    import torch.distributed as dist

    distributed = init_dist(local)
    import paper_2602_13509_b200 as P
    from paper_2602_13509_b200.distributed import GlobalRX
    from paper_2602_13509_b200.synth import Scene

    L = args.lines or cfg["lines"]
    S, B = cfg["samples"], cfg["bands"]
    per = L // world
    sc = Scene(cfg["seed"], S, B, cfg["components"])
    raw = sc.generate(rank * per, per)
    tabs = P.CalibrationTables(sc.dark, sc.coeff)
    g = GlobalRX(per, S, B, tabs, n_total=per * world * S)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        det = g.detect(raw)
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        start.record(stream)
        for _ in range(args.steps):
            det = g.detect(raw)
        end.record(stream)
        torch.cuda.synchronize()
    ms = start.elapsed_time(end)
    if distributed:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = per * world * S * args.steps / (ms / 1e3)
    if rank == 0:
        line = {
            "metric": "calibrated+RX-scored pixels/sec", "value": value, "unit": "pixels/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 (fp64 moments, all-reduce and factorisation)",
            "data": "synthetic (seeded device generator, bit-identical to oracle/synth.py)",
            "config": config_key(args, cfg, world) | {"parallelism": f"lineblocks/dp{world}"},
            "hbm_fraction_whole_path": value / world * bytes_per_pixel(B)
            / (load_peaks()[0] * 1e9),
            "global_threshold": det.threshold, "global_max": det.max_score,
            "gpu_launches": g.ops.plan.launches // max(1, args.steps + args.warmup),
            "clocks": clocks.summary(),
            "collectives": (f"{dist.get_backend()} (broadcast shift, SUM f64 moments, MAX flags "
                            "and max key, 3 x SUM radix histogram)") if distributed else
                           "none (single process: launch under torchrun for the NCCL path)",
        }
        if distributed and dist.get_backend() == "nccl":
            line["nccl_version"] = ".".join(map(str, torch.cuda.nccl.version()))
        print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()


def measure_e2e(args, P, cfg, lines, scenes):
    """Public API on host numpy cubes: H2D raw, D2H scores+mask+stats, per strip."""
    import torch

    S, B = cfg["samples"], cfg["bands"]
    hosts = []
    for sc in scenes:
        raw = sc.generate(0, lines).cpu().pin_memory().numpy()
        hosts.append((P.RawCube(raw, np.linspace(400, 1000, B), gains=np.ones(lines, np.float32)),
                      P.CalibrationTables(sc.dark, sc.coeff)))
    plan = P.DetectPlan(lines, S, B, batch=2)
    cubes, tabs = [h[0] for h in hosts], [h[1] for h in hosts]
    P.detect_batch(cubes, tabs, plan=plan)  # warm-up (pinned result buffers, graphs of nothing)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    steps = max(1, min(args.steps, 3))
    for _ in range(steps):
        det = P.detect_batch(cubes, tabs, plan=plan)[-1]
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    px = lines * S * len(hosts) * steps
    h2d = lines * S * B * 2 * len(hosts)
    d2h = lines * S * (4 + 1) * len(hosts)
    return {"value": px / sec, "unit": "pixels/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "strips_per_step": len(hosts),
            "api": "paper_2602_13509_b200.detect_batch([RawCube[numpy pinned]], tables): "
                   "H2D of strip i+1 and D2H of strip i-1 overlap the GPU work on strip i",
            "last_threshold": det.threshold}


def cpu_baseline(cfg, raw_dev, scene, lines):
    """The reference's own CPU path (baseline/_ref, numba default scorer) on a
    bounded sample of strip 0, on this box's host cores; the SKYRX_NO_NUMBA
    numpy scorer beside it (_accel.py:21-31)."""
    sample = cpu_sample_lines(cfg, lines)
    raw = raw_dev[:sample].cpu().numpy()
    sec, reps, fn = time_reference(raw, scene.dark, scene.coeff, cfg["bands"], 20, 1,
                                   budget_s=10.0)
    out = {"value": sample * cfg["samples"] / sec, "unit": "pixels/s",
           "cores": os.cpu_count(), "kind": fn.kind,
           "sample": f"{sample} lines x {cfg['samples']} samples of strip 0, {reps} reps; "
                     + ("skyrx apply_calibration -> compute_stats -> rx_scores "
                        f"[{fn.backend}] -> top-0.1% mask (baseline/_ref)"
                        if fn.kind == "reference" else f"oracle detect [{fn.backend}]"),
           "host": host_info()}
    if fn.kind == "reference":
        sec2, reps2, fn2 = time_reference(raw, scene.dark, scene.coeff, cfg["bands"], 5, 1,
                                          budget_s=5.0, numpy_scorer=True)
        out["numpy_scorer"] = {"value": sample * cfg["samples"] / sec2, "reps": reps2,
                               "backend": fn2.backend}
    return out


if __name__ == "__main__":
    main()
