"""Summarise ncu outputs into profiles/.

  launches: python tools/ncu_summary.py launches <launches.csv> <out.md> [--from-id N]
  full:     python tools/ncu_summary.py full <report.ncu-rep> <out.json> [traffic.json]

The launch list comes from `ncu --metrics gpu__time_duration.sum --clock-control
none --csv`; per-launch times are cold-cache and serialised, so only each
kernel's SHARE of a step is comparable with the bench's live CUDA-event times.
"""
import csv, io, json, re, subprocess, sys
from collections import OrderedDict


def short(name):
    name = re.sub(r"\(.*", "", name)
    return name.replace("skyrx::", "")


def launches(path, out, from_id=0):
    text = open(path).read()
    rows = list(csv.reader(io.StringIO(text[text.index('"ID"'):])))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = OrderedDict()
    for r in rows[1:]:
        if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        if int(r[ix["ID"]]) < from_id:
            continue
        k = short(r[ix["Kernel Name"]])
        v = float(r[ix["Metric Value"]].replace(",", "")) / 1e3  # us
        a = agg.setdefault(k, [0, 0.0, r[ix["Grid Size"]], r[ix["Block Size"]]])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    lines = ["| kernel | launches | mean us | total us | share | grid | block |",
             "|---|---|---|---|---|---|---|"]
    for k, (n, t, g, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {k} | {n} | {t / n:.1f} | {t:.1f} | {100 * t / tot:.1f}% | {g} | {b} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
           "sm__cycles_elapsed.avg.per_second",
           # tensor pipe (tcgen05 UTC*MMA), TMEM and the shared-memory operand path
           "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
           "sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg",
           "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
           "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
           "smsp__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
           "sm__cycles_elapsed.avg"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
        "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "second": 1}


def full(rep, out, traffic_out=None):
    text = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                          text=True).stdout
    rows = list(csv.reader(io.StringIO(text)))
    hdr, units = rows[0], rows[1]
    res = OrderedDict()
    for r in rows[2:]:
        k = short(r[hdr.index("Kernel Name")])
        d = OrderedDict()
        for m in METRICS:
            # some Blackwell metrics carry a section prefix ("TPC.TriageCompute.<name>")
            cols = [j for j, h in enumerate(hdr) if h == m or h.endswith("." + m)]
            if cols:
                i = cols[0]
                try:
                    val = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if u in UNIT and u not in ("%",):
                    val *= UNIT[u]
                d[m] = val
        rd, wr = d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum")
        t = d.get("gpu__time_duration.sum")
        if rd is not None and wr is not None and t:
            d["dram_GBps"] = (rd + wr) / t / 1e9
        if k in res:   # several launches of one kernel: keep a list
            if not isinstance(res[k], list):
                res[k] = [res[k]]
            res[k].append(d)
        else:
            res[k] = d
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))
    if traffic_out:
        # keyed by the bare kernel name (bench.py looks them up that way)
        tr = {}
        for k, v in res.items():
            v = v[-1] if isinstance(v, list) else v
            if "dram__bytes_read.sum" in v:
                tr[re.sub(r"<.*", "", k.replace("void ", "")).strip()] = \
                    v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]
        json.dump(tr, open(traffic_out, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], int(sys.argv[5]) if len(sys.argv) > 5 else 0)
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
