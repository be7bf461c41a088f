"""A/B of library builds on COLD strips (the bench's situation: each strip last touched GBs
earlier): score_tc and moments over 16 distinct c4 strips, CUDA events, builds interleaved.
    python tools/time_cold_ab.py lib_a.so lib_b.so ..."""
import json, os, subprocess, sys
if len(sys.argv) > 2 and sys.argv[1] == "--one":
    import torch
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
    from paper_2602_13509_b200 import _lib, _dev
    _lib.load(sys.argv[2])
    import paper_2602_13509_b200 as P
    from paper_2602_13509_b200.synth import Scene
    L, S, B, N = 16384, 900, 70, 16
    sc = Scene(4000, S, B, 5)
    raws = [sc.generate(0, L) for _ in range(N)]
    d, c = torch.from_numpy(sc.dark).cuda(), torch.from_numpy(sc.coeff).cuda()
    g = torch.ones(L, dtype=torch.float32, device='cuda')
    plan = P.DetectPlan(L, S, B)
    plan.run(0, raws[0], d, c, g, gain_const=1.0).finalize().score(0, raws[0], d, c, g)
    ds = plan.ds
    def tc(raw):
        _lib.call("skyrx_score_tc", raw.data_ptr(), L, S, B, d.data_ptr(), c.data_ptr(), None,
                  ds.mu_hilo[0].data_ptr(), plan.wpack[0].data_ptr(), ds.flags[0:1].data_ptr(),
                  plan.scores[0].data_ptr(), plan.max_key[0:1].data_ptr(), None, _dev.stream_ptr())
    def gr(raw):
        plan.run(0, raw, d, c, g, gain_const=1.0)
    hist = _lib.load().skyrx_topk_histogram(plan.topk_ws.data_ptr())
    def tch(raw):  # with the fused digit-0 top-k histogram, as plan.score runs it
        _lib.call("skyrx_score_tc", raw.data_ptr(), L, S, B, d.data_ptr(), c.data_ptr(), None,
                  ds.mu_hilo[0].data_ptr(), plan.wpack[0].data_ptr(), ds.flags[0:1].data_ptr(),
                  plan.scores[0].data_ptr(), plan.max_key[0:1].data_ptr(), hist, _dev.stream_ptr())
    def full(raw):  # the whole score stage of the bench step (init, score + hist, mask pass)
        plan.score(0, raw, d, c, g)
    out = {}
    for name, fn in (("score_tc", tc), ("score_tc_hist", tch), ("score_stage", full), ("moments", gr)):
        fn(raws[0]); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(2 * N):
            fn(raws[i % N])
        b.record(); torch.cuda.synchronize()
        out[name] = round(a.elapsed_time(b) / (2 * N), 4)
    print(json.dumps(out))
else:
    for rnd in range(2):
        for lib in sys.argv[1:]:
            r = subprocess.run([sys.executable, __file__, "--one", lib], capture_output=True, text=True)
            print(rnd, lib, r.stdout.strip() or r.stderr[-300:], flush=True)
