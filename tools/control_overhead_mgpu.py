"""SURVEY.md §8(f) row f1 on N GPUs: the trivial-body loop with a per-iteration exchange.

The paper's E1 measures the while-loop's control overhead across machines, with
and without a per-iteration barrier. Here every rank runs the same loop in one persistent
cf_run launch, and each iteration Sends its loop value to rank r+1 and Recvs rank r-1's value
over NVLink peer memory (PAPER.md:780-829 Send/Recv, keyed by iteration). Iteration t on any
rank therefore waits for iteration t of its neighbour; a chain of them is the barrier.

Loop on rank r: i = 0; a = 0; while i < n: i += 1; a = recv(i, from r-1) + 1, send(a, to r+1).
Closed form: a == n elementwise on every rank (checked every run).

--barrier: the per-iteration exchange is all-to-all instead (the paper's "with a barrier",
P:1253-1255): every rank Sends a to every other rank and the new value is the average of all
ranks' values plus one, a = (a + sum_p recv_p(a)) / N + 1, so iteration t on any rank waits
for iteration t of EVERY rank (a barrier plus an allreduce of the loop value). Closed form:
a == n on every rank.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port 29511 tools/control_overhead_mgpu.py [--iters 10000] [--K 1 32]
Without torchrun: one rank, no exchange (the 1-GPU loop of tools/control_overhead.py).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1805_01772_b200 import cf  # noqa: E402


def build(rank: int, world: int, width: int, barrier: bool = False):
    g = cf.Graph()
    n = g.placeholder("n", cf.I64, ())
    a0 = g.placeholder("a0", cf.F32, (width,))
    one_i = g.const(1, cf.I64)
    prev, nxt = (rank - 1) % world, (rank + 1) % world

    def body(i, a):
        if world > 1 and barrier:
            peers = [p for p in range(world) if p != rank]
            for p in peers:                               # channel = sender * N + receiver
                g.send(a, i, rank * world + p, p)
            s = a
            for p in peers:
                s = g.op1("Add", [s, g.recv(i, p * world + rank, p, cf.F32, (width,))])
            a = g.op1("Add", [g.op1("Mul", [s, g.const(1.0 / world, cf.F32)]), g.const(1.0, cf.F32)])
        elif world > 1:
            g.send(a, i, rank, nxt)                       # channel = sender's rank
            a = g.op1("Add", [g.recv(i, prev, prev, cf.F32, (width,)), g.const(1.0, cf.F32)])
        else:
            a = g.op1("Add", [a, g.const(1.0, cf.F32)])
        return [g.op1("Add", [i, one_i]), a]

    i_out, a_out = g.while_loop(lambda i, a: g.op1("Less", [i, n]), body,
                                [g.const(0, cf.I64), a0])
    return g, [i_out, a_out]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, nargs="+", default=[1000, 10000])
    ap.add_argument("--width", type=int, default=1)
    ap.add_argument("--K", type=int, nargs="+", default=[1, 32])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--barrier", action="store_true", help="all-to-all exchange every iteration")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")   # handles only; the data path is the device's
    torch.cuda.set_device(local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    for K in a.K:
        g, fetches = build(rank, world, a.width, a.barrier)
        nmax = max(a.iters)
        s = cf.Session(g, fetches, precision=cf.F32, parallel_iterations=K, device=local,
                       stream=stream.cuda_stream, max_iterations=nmax + 16, watchdog_ms=120000)
        if world > 1:
            s.connect_pipeline()
        outs = s.alloc_outputs(device=f"cuda:{local}")
        a0 = torch.zeros(a.width, dtype=torch.float32, device=f"cuda:{local}")
        for n in a.iters:
            feeds = {"n": torch.tensor(n, dtype=torch.int64, device=f"cuda:{local}"), "a0": a0}
            s.run(feeds, outs)          # warm-up
            torch.cuda.synchronize()
            times = []
            for _ in range(a.reps):
                if world > 1:
                    dist.barrier()
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                s.run(feeds, outs)
                e1.record(stream)
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1))
            ok = int(outs[0].item()) == n and bool(torch.all(outs[1] == float(n)))
            t = torch.tensor([sorted(times)[len(times) // 2], 0.0 if ok else 1.0])
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)   # max over ranks
            if rank == 0:
                ms = float(t[0])
                print(json.dumps({"n_gpus": world, "n": n, "width": a.width,
                                  "parallel_iterations": K,
                                  "exchange": ("all-to-all barrier" if a.barrier else "ring") if world > 1 else None,
                                  "ms_median_max_over_ranks": ms,
                                  "iterations_per_s": n / (ms * 1e-3),
                                  "us_per_iteration": ms * 1e3 / n,
                                  "closed_form_ok": float(t[1]) == 0.0}), flush=True)
        del s
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
