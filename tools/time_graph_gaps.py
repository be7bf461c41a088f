"""Where the c4 step's time goes beyond the two big kernels: CUDA-graph replays of 16 strips'
moments stage, score stage, and of each big kernel alone (events around the replays)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_2602_13509_b200 import _lib, _dev
import paper_2602_13509_b200 as P
from paper_2602_13509_b200.strips import StripBatch
from paper_2602_13509_b200.synth import Scene
L, S, B, N = 16384, 900, 70, 16
sc = Scene(4000, S, B, 5)
raws = [sc.generate(0, L) for _ in range(N)]
d, c = _dev.to_device(sc.dark), _dev.to_device(sc.coeff)
g = torch.ones(L, dtype=torch.float32, device="cuda")
batch = StripBatch(L, S, B, N)
plan = batch.plan
batch.enqueue(raws, [(d, c)] * N, [g] * N, [1.0] * N)
torch.cuda.synchronize()
ds = plan.ds
hist = _lib.load().skyrx_topk_histogram(plan.topk_ws.data_ptr())

def moments_stage():
    for j in range(N):
        plan.run(j, raws[j], d, c, g, gain_const=1.0)
def score_stage():
    for j in range(N):
        plan.score(j, raws[j], d, c, g)
def gram_only():
    for j in range(N):
        _lib.call("skyrx_stats_raw_own_shift", raws[j].data_ptr(), L, S, B, d.data_ptr(),
                  c.data_ptr(), 1.0, ds.shift[j].data_ptr(), ds.moments[j].data_ptr(),
                  ds.flags[j:j + 1].data_ptr(), plan.raw_ws.data_ptr(), plan.raw_ws_bytes,
                  _dev.stream_ptr())
def score_only():
    for j in range(N):
        _lib.call("skyrx_score_tc", raws[j].data_ptr(), L, S, B, d.data_ptr(), c.data_ptr(), None,
                  ds.mu_hilo[j].data_ptr(), plan.wpack[j].data_ptr(), ds.flags[j:j + 1].data_ptr(),
                  plan.scores[j].data_ptr(), plan.max_key[j:j + 1].data_ptr(), hist,
                  _dev.stream_ptr())
out = {}
side = torch.cuda.Stream()
for name, fn in (("moments_stage", moments_stage), ("stats_raw_calls", gram_only),
                 ("score_stage", score_stage), ("score_tc_calls", score_only)):
    side.wait_stream(torch.cuda.current_stream())
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=side):
        fn()
    torch.cuda.current_stream().wait_stream(side)
    gr.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        gr.replay()
    b.record(); torch.cuda.synchronize()
    out[name + "_us_per_strip"] = round(a.elapsed_time(b) / 3 / N * 1e3, 1)
print(json.dumps(out))
