"""Time the exact-digit score kernel (skyrx_score_tcs) on one c4 strip (B = 70)
and on a B = 128 cube of c5's width, with each library given (experiment
variants: tools/build_tcs_var.sh)."""
import json, os, subprocess, sys
libs = sys.argv[1:]
if len(libs) > 1:
    for l in libs:
        subprocess.run([sys.executable, __file__, l])
    sys.exit(0)
os.environ["SKYRX_B200_TCS"] = "1"
import torch
sys.path.insert(0, '.')
from paper_2602_13509_b200 import _lib, _dev
_lib.load(libs[0])
import paper_2602_13509_b200 as P
from paper_2602_13509_b200.synth import Scene
out = {"lib": libs[0]}
for L, S, B, K in ((16384, 900, 70, 5), (8192, 2048, 128, 5)):
    sc = Scene(4000, S, B, K)
    raw = sc.generate(0, L)
    d, c = torch.from_numpy(sc.dark).cuda(), torch.from_numpy(sc.coeff).cuda()
    g = torch.ones(L, dtype=torch.float32, device='cuda')
    plan = P.DetectPlan(L, S, B)
    plan.run(0, raw, d, c, g, gain_const=1.0).finalize()
    ds = plan.ds
    _lib.call("skyrx_score_prep", ds.w64[0].data_ptr(), ds.mu_hilo[0].data_ptr(), S, B,
              d.data_ptr(), c.data_ptr(), 1.0, 1, plan.records[0].data_ptr(), _dev.stream_ptr())
    def fn():
        _lib.call("skyrx_score_tcs", raw.data_ptr(), L, S, B, plan.records[0].data_ptr(),
                  ds.flags[0:1].data_ptr(), plan.scores[0].data_ptr(),
                  plan.max_key[0:1].data_ptr(), None, _dev.stream_ptr())
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): fn()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    out[f"B{B}_ms"] = ms
    out[f"B{B}_TBps_raw"] = L * S * B * 2 / ms / 1e9
    del raw, plan
print(json.dumps(out), flush=True)
