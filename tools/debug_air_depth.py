"""Which cube / stage makes run_air's stream differ between queue depths on the GPU?

Runs the reference's test_pipeline small_config (baseline/_ref, through install())
several times per depth and reports, per run pair, the cubes whose frames, scores or
RGB differ and by how much."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT / "baseline" / "_ref"), str(ROOT / "baseline" / "_ref" / "tests"), str(ROOT)]

import skyrx  # noqa: E402

import paper_2602_13509_b200 as P  # noqa: E402

P.install(skyrx)
from skyrx.pipeline import synthesize  # noqa: E402
from test_pipeline import small_config  # noqa: E402

from paper_2602_13509_b200.air import run_air  # noqa: E402


def run(depth):
    cfg = small_config(queue_depth=depth)
    return run_air(cfg, synthesize(cfg))


def diff(a, b, tag):
    n = len(a.scores)
    per = len(a.frames) // max(n, 1)
    bad = []
    for c in range(n):
        fa, fb = a.frames[c * per:(c + 1) * per], b.frames[c * per:(c + 1) * per]
        sa, sb = np.asarray(a.scores[c].values), np.asarray(b.scores[c].values)
        ra, rb = np.asarray(a.rgb[c]), np.asarray(b.rgb[c])
        if fa != fb or not np.array_equal(sa, sb) or not np.array_equal(ra, rb):
            nf = sum(x != y for x, y in zip(fa, fb))
            ds = np.abs(sa.astype(np.float64) - sb) / np.maximum(np.abs(sa), 1e-30)
            bad.append(f"cube {c}: frames differ {nf}/{per}, scores differ "
                       f"{int((sa != sb).sum())} px (max rel {ds.max():.2e}), rgb differ "
                       f"{int((ra != rb).sum())}")
    print(f"{tag}: {len(bad)} cubes differ (of {n}); dropped {a.dropped} / {b.dropped}")
    for s in bad[:8]:
        print("   ", s)


ref = run(1)
for k in range(2):
    diff(ref, run(1), f"depth1 vs depth1 #{k}")
for k in range(2):
    diff(ref, run(3), f"depth1 vs depth3 #{k}")
r3 = run(3)
n = len(ref.rgb)
for c in range(n):
    m = [d for d in range(n) if np.array_equal(np.asarray(r3.rgb[c]), np.asarray(ref.rgb[d]))]
    a = np.asarray(r3.rgb[c])
    print(f"depth3 cube {c}: rgb equals depth1 cube(s) {m}; finite {np.isfinite(a).all()}, "
          f"mean {a.mean():.4g} vs {np.asarray(ref.rgb[c]).mean():.4g}")
for depth in (2, 4):
    diff(ref, run(depth), f"depth1 vs depth{depth}")
