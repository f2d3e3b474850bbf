"""§8(f) f4: statically unrolled LSTM vs the device while_loop (§6.3).

(1) time: 1-layer LSTM, T=200, batch sweep (the paper reports dynamic 3-8% slower than static,
    shrinking with batch); (2) memory: H=2048, B=256, the device bytes a session of each
    program needs as T grows (the paper: dynamic_rnn fits T=256 where static unrolling ran out
    of memory at 128). One JSON line per measurement."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_1805_01772_b200 import cf  # noqa: E402
from paper_1805_01772_b200.models import dynamic_rnn_lstm, feeds_to_device, static_rnn_lstm  # noqa: E402
from synth import rnn_inputs  # noqa: E402


def device_bytes(s):
    for tok in s.describe().split():
        if tok.startswith("bytes="):
            return int(tok.split("=")[1])
    return None


def time_prog(p, f, reps, K=0):
    s = cf.Session(p.g, p.fetch_tensors(), precision=cf.BF16, parallel_iterations=K)
    dev = feeds_to_device(f, session=s)
    outs = s.alloc_outputs()
    for _ in range(3):
        s.run(dev, outs)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        _, _, tr = s.run(dev, outs, trace=True)
        ts.append(tr["wall_ms"])
    b = device_bytes(s)
    del s
    torch.cuda.empty_cache()
    return sorted(ts)[len(ts) // 2], b


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--H", type=int, default=512)
    ap.add_argument("--T", type=int, default=200)
    ap.add_argument("--batches", default="64,128,256,512")
    ap.add_argument("--mem-H", type=int, default=2048)
    ap.add_argument("--mem-B", type=int, default=256)
    ap.add_argument("--mem-T", default="32,64,128,256")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    H, T = a.H, a.T
    for B in [int(b) for b in a.batches.split(",")]:
        f = rnn_inputs(T, B, H, H, 1, seed=0, len_mode="full", bf16=True)
        ms_d, by_d = time_prog(dynamic_rnn_lstm(T, B, H, H, 1), f, a.reps)
        ms_s, by_s = time_prog(static_rnn_lstm(T, B, H, H, 1), f, a.reps)
        print(json.dumps({"kind": "time", "T": T, "H": H, "B": B, "dynamic_ms": ms_d, "static_ms": ms_s,
                          "dynamic_over_static": ms_d / ms_s, "dynamic_bytes": by_d, "static_bytes": by_s}),
              flush=True)
    H, B = a.mem_H, a.mem_B
    for T in [int(t) for t in a.mem_T.split(",")]:
        res = {"kind": "memory", "T": T, "H": H, "B": B}
        free, total = torch.cuda.mem_get_info()
        for name, mk in (("dynamic", dynamic_rnn_lstm), ("static", static_rnn_lstm)):
            p = mk(T, B, H, H, 1)
            # the compiled plan's device bytes (host-side compile; nothing allocated)
            lst = cf.debug_program_listing(p.g, p.fetch_tensors(), precision=cf.BF16)
            by = int(lst.split("device bytes=")[1].split()[0])
            res[name + "_bytes"] = by
            res[name + "_fits"] = by < free
        res["gpu_free_bytes"] = free
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
