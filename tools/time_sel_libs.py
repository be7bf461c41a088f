"""Time the select stage (top-k init + one-pass mask) of one c4 strip with each
library given (experiment variants: tools/build_sel_var.sh)."""
import json, subprocess, sys
libs = sys.argv[1:]
if len(libs) > 1:
    for l in libs:
        subprocess.run([sys.executable, __file__, l])
    sys.exit(0)
import torch
sys.path.insert(0, '.')
from paper_2602_13509_b200 import _lib, _dev
_lib.load(libs[0])
import paper_2602_13509_b200 as P
from paper_2602_13509_b200.synth import Scene
L, S, B = 16384, 900, 70
sc = Scene(4000, S, B, 5)
raw = sc.generate(0, L)
d, c = torch.from_numpy(sc.dark).cuda(), torch.from_numpy(sc.coeff).cuda()
g = torch.ones(L, dtype=torch.float32, device='cuda')
plan = P.DetectPlan(L, S, B)
plan.run(0, raw, d, c, g, gain_const=1.0).finalize().score(0, raw, d, c, g)
torch.cuda.synchronize()
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
full = t(lambda: plan.score(0, raw, d, c, g))
only = t(lambda: plan.score_only(0, raw, d, c, g, topk_hist0=True))
print(json.dumps({"lib": libs[0], "select_ms": full - only, "score_path_ms": full}), flush=True)
