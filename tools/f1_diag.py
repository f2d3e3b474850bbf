"""Diagnostic for §8(f) f1: trivial-loop cost per iteration with tile bodies skipped
(debug flag 1) and with 0 (= all SMs), 8 or 1 worker CTAs. Run on a GPU: python tools/f1_diag.py"""
import sys, json, torch
sys.path.insert(0, 'tools'); sys.path.insert(0, '.')
import control_overhead as co
from paper_1805_01772_b200 import cf
n = 5000
for nw in (0, 8, 1):
    for flags in (0, 1):
        g, fetches = co.build(1)
        st = torch.cuda.Stream(); torch.cuda.set_stream(st)
        s = cf.Session(g, fetches, precision=cf.F32, parallel_iterations=1, stream=st.cuda_stream,
                       max_iterations=n + 16, num_workers=nw)
        feeds = {"n": torch.tensor(n, dtype=torch.int64, device="cuda"), "a0": torch.zeros(1, device="cuda")}
        outs = s.alloc_outputs(); cf.debug_set_flags(flags)
        s.run(feeds, outs); torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st); s.run(feeds, outs); e1.record(st); torch.cuda.synchronize()
        _, _, tr = s.run(feeds, outs, trace=True); torch.cuda.synchronize()
        cf.debug_set_flags(0)
        print(json.dumps({"num_workers": nw, "flags": flags, "us_per_iter": e0.elapsed_time(e1) * 1e3 / n,
                          "instances_per_iter": tr["instances"] / n, "tiles_per_iter": tr["tiles"] / n}), flush=True)
