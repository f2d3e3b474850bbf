"""SURVEY.md §8(f) row f1 (1 GPU): control-overhead microbenchmark.

The paper's E1 times a while-loop whose body does almost nothing, to isolate
the per-iteration cost of the control-flow machinery (>20,000 iterations/s on one machine).
Here the same loop runs as one persistent cf_run launch: the device driver evaluates
Merge -> Less -> Switch -> body -> NextIteration for every iteration with no host round trip.

Loop: i = 0; a = 0 (fp32 vector of width W); while i < n: i += 1; a += 1.
Closed form: trip count n, a == n elementwise (checked every run).
Timing: CUDA events on the session's stream, warm-up first, iterations/s = n / launch time.

    python tools/control_overhead.py [--n 100000] [--width 1] [--K 1] [--reps 5]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1805_01772_b200 import cf  # noqa: E402


def build(width: int):
    g = cf.Graph()
    n = g.placeholder("n", cf.I64, ())
    a0 = g.placeholder("a0", cf.F32, (width,))
    one_i = g.const(1, cf.I64)
    i_out, a_out = g.while_loop(
        lambda i, a: g.op1("Less", [i, n]),
        lambda i, a: [g.op1("Add", [i, one_i]), g.op1("Add", [a, g.const(1.0, cf.F32)])],
        [g.const(0, cf.I64), a0])
    return g, [i_out, a_out]


def run(n: int, width: int = 1, K: int = 1, reps: int = 5, warmup: int = 2):
    g, fetches = build(width)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    s = cf.Session(g, fetches, precision=cf.F32, parallel_iterations=K,
                   stream=stream.cuda_stream, max_iterations=n + 16)
    feeds = {"n": torch.tensor(n, dtype=torch.int64, device="cuda"),
             "a0": torch.zeros(width, dtype=torch.float32, device="cuda")}
    outs = s.alloc_outputs()
    for _ in range(warmup):
        s.run(feeds, outs)
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s.run(feeds, outs)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    _, dead, tr = s.run(feeds, outs, trace=True)
    torch.cuda.synchronize()
    i_v = int(outs[0].item())
    a_v = outs[1].cpu()
    ok = (i_v == n and bool(torch.all(a_v == float(n))) and not any(dead)
          and tr["trip_count"][0] == n)
    times.sort()
    ms = times[len(times) // 2]
    return {"n": n, "width": width, "parallel_iterations": K, "ms_median": ms,
            "ms_min": times[0], "iterations_per_s": n / (ms * 1e-3),
            "us_per_iteration": ms * 1e3 / max(n, 1), "trip_count": tr["trip_count"][0],
            "closed_form_ok": ok}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[1000, 10000, 100000])
    ap.add_argument("--width", type=int, default=1)
    ap.add_argument("--K", type=int, nargs="+", default=[1, 32])
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    for K in a.K:
        for n in a.n:
            print(json.dumps(run(n, a.width, K, a.reps)), flush=True)


if __name__ == "__main__":
    main()
