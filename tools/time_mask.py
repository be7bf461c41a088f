"""The one-pass top-k mask on one c4 strip's scores (CUDA events, 20 launches after the
fused digit-0 histogram): python tools/time_mask.py lib.so ..."""
import json, os, subprocess, sys
if len(sys.argv) > 2 and sys.argv[1] == "--one":
    import torch
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
    from paper_2602_13509_b200 import _lib, _dev
    _lib.load(sys.argv[2])
    import paper_2602_13509_b200 as P
    from paper_2602_13509_b200.synth import Scene
    L, S, B = 16384, 900, 70
    sc = Scene(4000, S, B, 5)
    raw = sc.generate(0, L)
    d, c = torch.from_numpy(sc.dark).cuda(), torch.from_numpy(sc.coeff).cuda()
    g = torch.ones(L, dtype=torch.float32, device='cuda')
    plan = P.DetectPlan(L, S, B)
    plan.run(0, raw, d, c, g, gain_const=1.0).finalize().score(0, raw, d, c, g)
    n = L * S
    k = (n + 999) // 1000
    ws = plan.topk_ws.data_ptr()
    lib = _lib.load()
    hist = lib.skyrx_topk_histogram(ws)
    def setup():
        _lib.call("skyrx_topk_init", n, k, ws, _dev.stream_ptr())
        plan.score_only(0, raw, d, c, g, topk_hist0=True)
    setup(); torch.cuda.synchronize()
    def mask():
        _lib.call("skyrx_topk_mask", plan.scores[0].data_ptr(), n, 1, plan.thr[0:1].data_ptr(),
                  plan.mask[0].data_ptr(), ws, plan.cand.data_ptr(), plan.cand_cap,
                  _dev.stream_ptr())
    ms = 0.0
    for _ in range(10):
        setup()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); mask(); b.record(); torch.cuda.synchronize()
        ms += a.elapsed_time(b)
    print(json.dumps({"mask_ms": round(ms / 10, 4), "thr": float(plan.thr[0].item())}))
else:
    for lib in sys.argv[1:]:
        r = subprocess.run([sys.executable, __file__, "--one", lib], capture_output=True, text=True)
        print(lib, r.stdout.strip() or r.stderr[-400:], flush=True)
