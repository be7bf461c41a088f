"""Static SASS instruction census of the hot kernels in libskyrx_b200.so.

    python tools/sass_census.py > profiles/r02_sass_census.md

Counts the mnemonics that prove the Blackwell paths (B200_PROFILING.md: UTC*MMA =
tcgen05.mma, LDTM/STTM = tcgen05.ld/st, UTMALDG/UBLKCP = TMA / bulk copies) and the
CUDA-core work around them, per kernel (static instruction counts, not executed ones).
"""
import re
import subprocess
import sys
from collections import Counter, OrderedDict
from pathlib import Path

SO = Path(__file__).resolve().parent.parent / "paper_2602_13509_b200" / "libskyrx_b200.so"
HOT = ["score_tc_kernel", "score_tcs_kernel", "score_tcw_kernel", "gram_raw_kernel",
       "raww_gram_kernel", "raww_scan_kernel", "gram_tc_kernel", "finalize_small_kernel",
       "finalize_kernel", "topk_mask_pass_kernel", "calibrate_vec8_kernel", "gf_matmul_kernel"]
KEYS = ["UTCIMMA", "UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UBLKCP",
        "SYNCS", "HMMA", "DFMA", "DMUL", "DADD", "FFMA", "FFMA2", "FADD2", "FMUL2", "LDS",
        "STS", "LDG", "STG", "BAR", "SHFL"]


def main():
    out = subprocess.run(["cuobjdump", "-sass", str(SO)], capture_output=True, text=True).stdout
    funcs = OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
        if m:
            op = m.group(2)
            base = op.split(".")[0]
            funcs[cur][base] += 1
            funcs[cur]["_total"] += 1
    demangled = {}
    names = list(funcs)
    dm = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True,
                        text=True).stdout.splitlines()
    for n, d in zip(names, dm):
        demangled[n] = d
    print("| kernel | SASS total | " + " | ".join(KEYS) + " |")
    print("|---|---|" + "---|" * len(KEYS))
    for n, c in funcs.items():
        d = demangled[n]
        short = re.sub(r"\(.*", "", d).replace("skyrx::", "")
        if not any(h in short for h in HOT):
            continue
        print(f"| `{short}` | {c['_total']} | " + " | ".join(str(c.get(k, 0)) for k in KEYS)
              + " |")


if __name__ == "__main__":
    sys.exit(main())
