"""Time skyrx_stats_raw_own_shift alone on one c4-shaped strip for each library given and
compare its moments with the first library's (tools/build_gr_var.sh builds variants).
  python tools/time_gr_direct.py [--bands B] lib0.so lib1.so ..."""
import os, sys, json, subprocess
args = sys.argv[1:]
bands, lines = 70, 16384
while args and args[0] in ("--bands", "--lines"):
    if args[0] == "--bands": bands = int(args[1])
    else: lines = int(args[1])
    args = args[2:]
if len(args) > 1:
    for l in args:
        subprocess.run([sys.executable, __file__, "--bands", str(bands), "--lines", str(lines), l])
    sys.exit(0)
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2602_13509_b200 import _lib
_lib.load(args[0])
import paper_2602_13509_b200 as P
from paper_2602_13509_b200.synth import Scene
L, S, B = lines, 900, bands
if (S * B * 2) % 16: S = 904
sc = Scene(4000, S, B, 5)
raws = [sc.generate(i, L) for i in range(4)]   # 4 strips: 8 GB cycled, larger than L2
d, c = torch.from_numpy(sc.dark).cuda(), torch.from_numpy(sc.coeff).cuda()
lib = _lib.load()
wsb = int(lib.skyrx_stats_raw_workspace_for(L, S, B))
ws = torch.empty(wsb, dtype=torch.uint8, device='cuda')
shift = torch.zeros(B, dtype=torch.float64, device='cuda')
mom = torch.zeros(B * B + B + 1, dtype=torch.float64, device='cuda')
flags = torch.zeros(1, dtype=torch.int32, device='cuda')
st = torch.cuda.current_stream().cuda_stream
def fn(i):
    _lib.call("skyrx_stats_raw_own_shift", raws[i % 4].data_ptr(), L, S, B, d.data_ptr(), c.data_ptr(),
              1.0, shift.data_ptr(), mom.data_ptr(), flags.data_ptr(), ws.data_ptr(), wsb, st)
fn(0); torch.cuda.synchronize()
m0 = mom.cpu().numpy().copy(); f0 = int(flags.item())
for i in range(4): fn(i)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for i in range(20): fn(i)
b.record(); torch.cuda.synchronize()
ref = f"gpurun_out/gr_direct_ref_{B}_{L}.npy"
os.makedirs("gpurun_out", exist_ok=True)
if not os.path.exists(ref):
    np.save(ref, m0); rel = None
else:
    r = np.load(ref); rel = float(np.abs(m0 - r).max() / np.abs(r).max())
    nz = np.abs(r) > 0
    relel = float((np.abs(m0 - r)[nz] / np.abs(r)[nz]).max())
print(json.dumps({"lib": args[0], "bands": B, "lines": L, "ms": a.elapsed_time(b) / 20, "flags": f0,
                  "rel_vs_first": rel, "rel_elementwise": None if rel is None else relel}), flush=True)
