"""A/B of score_tc_kernel builds on one c4 strip: python tools/time_sc_ab.py lib.so ...
(each lib in its own process; CUDA events over 20 launches, interleaved rounds)."""
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
    ds = plan.ds
    def tc_only():
        _lib.call("skyrx_score_tc", raw.data_ptr(), L, S, B, d.data_ptr(), c.data_ptr(), None,
                  ds.mu_hilo[0].data_ptr(), plan.wpack[0].data_ptr(), ds.flags[0:1].data_ptr(),
                  plan.scores[0].data_ptr(), plan.max_key[0:1].data_ptr(), None, _dev.stream_ptr())
    def stats():
        plan.run(0, raw, d, c, g, gain_const=1.0)
    out = {}
    for name, fn in (("score_tc", tc_only), ("moments", stats)):
        fn(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            fn()
        b.record(); torch.cuda.synchronize()
        out[name] = round(a.elapsed_time(b) / 20, 4)
    print(json.dumps(out))
else:
    for rnd in range(2):
        for lib in sys.argv[1:]:
            r = subprocess.run([sys.executable, __file__, "--one", lib], capture_output=True, text=True)
            print(rnd, lib, r.stdout.strip() or r.stderr[-300:], flush=True)
