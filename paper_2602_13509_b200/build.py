"""Build the in-tree CUDA library libskyrx_b200.so for sm_100a with nvcc.

    python -m paper_2602_13509_b200.build        (or __graft_entry__.build())

One shared object with a plain C ABI (include/skyrx_b200.h), cudart linked
statically so it loads next to torch's own runtime without version coupling.
Objects are rebuilt only when a source or header is newer than the .so.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "libskyrx_b200.so"
BUILD = ROOT / "build" / "obj"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-Xptxas", "-warn-spills",
    # numerics contract: IEEE division/sqrt, no flush-to-zero (1e-40 gains must
    # overflow to inf, test_pipeline.py:84-102); contraction only where written
    "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
]


def nvcc() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(cand).exists():
        raise RuntimeError("nvcc not found (CUDA 12.9 toolkit required to build)")
    return cand


def sources():
    return sorted(CSRC.glob("*.cu"))


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> Path:
    headers = list(CSRC.glob("*.cuh")) + list((ROOT / "include").glob("*.h"))
    srcs = sources()
    BUILD.mkdir(parents=True, exist_ok=True)
    objs = []
    jobs = []
    for s in srcs:
        o = BUILD / (s.stem + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            cmd = [nvcc(), *ARCH, *NVCC_FLAGS, "-I", str(ROOT / "include"), "-c", str(s),
                   "-o", str(o)]
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r.stderr

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        for log in ex.map(run, jobs):
            if verbose and log.strip():
                print(log, file=sys.stderr)
    if force or jobs or _stale(OUT, objs):
        cmd = [nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", str(OUT),
               *[str(o) for o in objs]]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return OUT


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
