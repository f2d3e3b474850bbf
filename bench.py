#!/usr/bin/env python
"""Benchmark: LSTM fwd+bwd sequence-steps/s through the dynamic-control-flow engine.

One "step" = one cf_run: the whole hot path (while_loop forward with StackPush, gradient
loop with StackPop, TensorArray reads/writes, length conds) over one batch of synthetic
input, ONE launch of the persistent driver kernel. Workload (--config, default cfg3):

  cfg3  8-layer LSTM, hidden 1024, batch 512, seq_len 200, full lengths (BASELINE.json
        configs[2]; the metric's 1/2/4/8-B200 configuration)
  cfg2  1 layer, hidden 512, batch 64, seq_len 100, variable lengths (configs[1])
  cfg4  1 layer, hidden 2048, batch 256, seq_len 4000 (configs[3])

sequence-steps/s = sum_b len_b (live sample-timesteps) / step time.
--impl reference times the fp64 CPU oracle (the only reference that exists: the paper ships
no code) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "cfg3": dict(T=200, B=512, I=1024, H=1024, L=8, len_mode="full"),
    "cfg2": dict(T=100, B=64, I=512, H=512, L=1, len_mode="uniform"),
    "cfg4": dict(T=4000, B=256, I=2048, H=2048, L=1, len_mode="full"),
    "tiny": dict(T=5, B=2, I=4, H=8, L=1, len_mode="full"),
    # BASELINE.json configs[4]: nested MoE-style gated cond in the body, bf16, PI sweep via --K
    # (tanh experts: DESIGN.md reading R21; the bf16 parity tests run the same workload)
    "cfg5": dict(T=200, B=128, I=1024, H=1024, L=8, len_mode="uniform", moe=True, moe_act="tanh"),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0, "_fallback": True}


class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev=0):
        self.dev, self.rows, self.proc = dev, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].lower() == "active":
                    reasons.add(nm)
        mx = float(self.rows[0][2]) if self.rows and self.rows[0][2].replace(".", "").isdigit() else None
        pw = []
        for r in self.rows:
            try:
                pw.append(float(r[3]))
            except (IndexError, ValueError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w": statistics.median(pw) if pw else None}


def flops_per_step(c, lens_sum):
    """Algorithmic FLOPs: 24*H*(I_l+H) per live sample-step per layer (fwd 8, bwd 16)."""
    H, I, L = c["H"], c["I"], c["L"]
    per = 0
    for l in range(L):
        il = I if l == 0 else H
        per += 24 * H * (il + H)
        if c.get("moe"):
            per += 3 * 2 * H * H   # the taken expert's matmul: forward + two gradient matmuls
    return per * lens_sum


def model_kw(c):
    """Builder options of a config beyond its sizes (the MoE-style gated branch)."""
    return {"moe": c.get("moe", False), "moe_act": c.get("moe_act", "relu")}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def run_reference(args, c, cfg_name):
    """The fp64 oracle on the host cores, each step a bounded sample (truncated T)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import numpy as np
    from oracle.models import dynamic_rnn_lstm, run_program
    from synth import rnn_inputs
    T_s = max(2, min(c["T"], args.ref_T))
    p = dynamic_rnn_lstm(T_s, c["B"], c["I"], c["H"], c["L"], **model_kw(c))
    f = rnn_inputs(T_s, c["B"], c["I"], c["H"], c["L"], seed=0, len_mode=c["len_mode"],
                   moe=c.get("moe", False))
    lens_sum = int(np.minimum(f["len"], T_s).sum())
    # the driver's --steps / --warmup; each step is one bounded sample (truncated T)
    n_steps = max(1, args.steps if args.steps else args.steps_ref)
    n_warm = args.warmup if args.warmup is not None else args.warmup_ref
    for _ in range(n_warm):
        run_program(p, f)
    ts = []
    for _ in range(n_steps):
        t0 = time.perf_counter()
        run_program(p, f)
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    v = lens_sum / t
    line = {"impl": "reference", "metric": "LSTM fwd+bwd sequence-steps/sec", "value": v,
            "unit": "sequence-steps/s", "n_gpus": max(world, args.gpus), "steps": n_steps,
            "warmup": n_warm, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg_name, **{k: c[k] for k in ("T", "B", "I", "H", "L")},
                       "sample_T": T_s},
            "cpu_baseline": {"value": v, "unit": "sequence-steps/s", "cores": cores, "kind": "oracle",
                             "sample": f"{cfg_name} truncated to T={T_s} (full B/H/L), median of "
                                       f"{n_steps} steps"},
            "e2e": {"value": v, "unit": "sequence-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(c, cfg_name, T_s, T_1=2):
    """The fp64 oracle as it stands on the host cores (all BLAS threads), plus a 1-thread
    sample: each a bounded, truncated-T run of the same workload."""
    import numpy as np
    from threadpoolctl import threadpool_limits
    from oracle.models import dynamic_rnn_lstm, run_program
    from synth import rnn_inputs

    def one(T):
        p = dynamic_rnn_lstm(T, c["B"], c["I"], c["H"], c["L"], **model_kw(c))
        f = rnn_inputs(T, c["B"], c["I"], c["H"], c["L"], seed=0, len_mode=c["len_mode"],
                       moe=c.get("moe", False))
        lens_sum = int(np.minimum(f["len"], T).sum())
        t0 = time.perf_counter()
        run_program(p, f)
        return lens_sum, time.perf_counter() - t0

    n, t = one(T_s)
    with threadpool_limits(limits=1):
        n1, t1 = one(min(T_1, T_s))
    return {"value": n / t, "unit": "sequence-steps/s", "cores": os.cpu_count(),
            "kind": "oracle", "sample": f"{cfg_name} truncated to T={T_s} (full B/H/L), one run, "
                                        f"{t:.1f} s",
            "one_thread": {"value": n1 / t1, "cores": 1,
                           "sample": f"{cfg_name} truncated to T={min(T_1, T_s)}, one run, {t1:.1f} s"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3", choices=list(CONFIGS))
    ap.add_argument("--precision", default="bf16", choices=["f32", "bf16"])
    ap.add_argument("--K", type=int, default=0, help="parallel_iterations override (0 = 32)")
    ap.add_argument("--T", type=int, default=0, help="override the config's sequence length")
    ap.add_argument("--watchdog-ms", type=int, default=0, help="device watchdog (0: 300 s multi-GPU)")
    ap.add_argument("--ref-T", type=int, default=8)
    ap.add_argument("--steps-ref", type=int, default=3)
    ap.add_argument("--warmup-ref", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-T", type=int, default=12)
    ap.add_argument("--stack-budget", type=int, default=0,
                    help="device bytes for stacked activations; beyond it stacks swap to pinned "
                         "host memory (0 = no swapping, 1 = swap every eligible value)")
    ap.add_argument("--swap-smallest-first", action="store_true",
                    help="with --stack-budget: swap the smallest stacked values first")
    ap.add_argument("--parallel", default="pipeline", choices=["pipeline", "dp", "replicas"],
                    help="N>1: layer-partitioned pipeline (strong scaling, SURVEY.md a14), batch "
                         "data parallelism with the in-graph weight-gradient allreduce (weak "
                         "scaling, f3), or independent replicas (weak scaling, no exchange)")
    args = ap.parse_args()
    c = dict(CONFIGS[args.config])
    if args.T:
        c["T"] = args.T
    if args.impl == "reference":
        return run_reference(args, c, args.config)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torchrun (the driver's own launch
        # sets WORLD_SIZE and lands below directly)
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))

    import numpy as np
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_1805_01772_b200 import cf
    from paper_1805_01772_b200.models import dynamic_rnn_lstm, feeds_to_device
    from synth import rnn_inputs

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    W = max(args.warmup, 3)
    prec = cf.F32 if args.precision == "f32" else cf.BF16
    pipe = world > 1 and args.parallel == "pipeline"
    if pipe and world > c["L"]:
        raise SystemExit(f"pipeline over {world} GPUs needs >= {world} layers")
    stage = (rank, world) if pipe else None
    dp = (rank, world) if world > 1 and args.parallel == "dp" else None
    p = dynamic_rnn_lstm(c["T"], c["B"], c["I"], c["H"], c["L"], stage=stage, dp=dp, **model_kw(c))
    # a dedicated stream, current for torch too: the input copies of the end-to-end loop and
    # the cf_run launches are ordered on it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sess = cf.Session(p.g, p.fetch_tensors(), precision=prec, parallel_iterations=args.K,
                      device=local, stream=stream.cuda_stream,
                      watchdog_ms=args.watchdog_ms or (300000 if (pipe or dp) else 0), stack_budget_bytes=args.stack_budget,
                      swap_smallest_first=args.swap_smallest_first)
    if pipe or dp:
        sess.connect_pipeline()
    # pipeline: one model split over the ranks (same inputs everywhere); dp: the same weights
    # (and, for timing, the same batch) on every rank; replicas: own inputs
    f = rnn_inputs(c["T"], c["B"], c["I"], c["H"], c["L"], seed=0 if (pipe or dp) else rank,
                   moe=c.get("moe", False),
                   len_mode=c["len_mode"], bf16=prec == cf.BF16)
    lens_sum = int(f["len"].sum())
    dev = feeds_to_device(f, device=f"cuda:{local}", session=sess)
    outs = sess.alloc_outputs(device=f"cuda:{local}")
    for _ in range(W):
        sess.run(dev, outs)
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed():
        kms = []
        with Clocks(local) as ck:
            torch.cuda.synchronize()
            ev0.record(stream)
            for _ in range(args.steps):
                _, _, t = sess.run(dev, outs, trace=True)
                kms.append(t["wall_ms"])
            ev1.record(stream)
            torch.cuda.synchronize()
        return kms, t, ck

    kernel_ms, tr, clk = timed()
    # the timing rules: a run that saw a hardware / thermal slowdown, or SM clocks well below
    # max with no reason, is re-measured once (sw_power_cap is kept and noted)
    cs = clk.summary()
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(cs["reasons"])
    low = (cs["sm_mhz"] and cs["sm_max_mhz"] and cs["sm_mhz"] < 0.8 * cs["sm_max_mhz"]
           and not cs["reasons"])
    remeasured = False
    flag = torch.tensor([1.0 if (bad or low) else 0.0], device=f"cuda:{local}")
    if pg:
        pg.all_reduce(flag, op=pg.ReduceOp.MAX)
        pg.barrier()
    if float(flag.item()) > 0:
        kernel_ms, tr, clk = timed()
        remeasured = True
    swap = {"stack_budget_bytes": args.stack_budget, "smallest_first": args.swap_smallest_first,
            "swap_out": tr["swap_out"],
            "swap_in": tr["swap_in"], "bytes_d2h": tr["bytes_d2h"], "bytes_h2d": tr["bytes_h2d"]}
    if pg:
        pg.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    if pg:
        t = torch.tensor([ms], device=f"cuda:{local}")
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        ms = float(t.item())
    # ---- end to end through the public API with HOST buffers (pinned), per step:
    #      H2D of the step's data (x, lengths, loss projections) + D2H of the loss
    data_names = ["x", "len", "R_out", "route"] + [f"R_h{l}" for l in range(c["L"])] + \
        [f"R_c{l}" for l in range(c["L"])]
    host = {k: v.cpu().pin_memory() for k, v in dev.items() if k in data_names}
    h2d = sum(v.numel() * v.element_size() for v in host.values())
    y_host = torch.empty(outs[0].shape, dtype=outs[0].dtype).pin_memory()
    d2h = y_host.numel() * y_host.element_size()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_steps = max(2, args.steps)   # the same step count as the device-timed value
    # the step's inputs are copied on a copy stream into one of two device input sets while
    # the previous step computes (double buffering, as a data loader would); every copy is
    # inside the timed region and each cf_run waits for its own inputs
    sets = [dev, dict(dev)]
    for k in host:
        sets[1][k] = torch.empty_like(dev[k])
    copy_stream = torch.cuda.Stream()
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    cev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(e2e_steps)]
    # the step itself (after its inputs arrived), to see what the copies cost the kernel
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(e2e_steps)]

    # diagnostics only: "oneset" runs every step on set 0 while the copies still stream in
    # (separates the copies' cost from the alternation of the input sets)
    e2e_ab = os.environ.get("BENCH_E2E_AB", "")

    def issue_copy(i):
        with torch.cuda.stream(copy_stream):
            cev[i][0].record(copy_stream)
            for k, v in host.items():
                sets[i % 2][k].copy_(v, non_blocking=True)
            cev[i][1].record(copy_stream)
            copied[i % 2].record(copy_stream)

    torch.cuda.synchronize()
    if pg:
        pg.barrier()   # every rank has its pinned inputs ready before the clock starts
        torch.cuda.synchronize()
    ck_e2e = Clocks(local).__enter__()
    e0.record(stream)
    copy_stream.wait_event(e0)
    issue_copy(0)
    for i in range(e2e_steps):
        stream.wait_event(copied[i % 2])
        if i + 1 < e2e_steps:
            issue_copy(i + 1)   # the set it overwrites was used by step i - 1 (finished)
        kev[i][0].record(stream)
        sess.run(sets[0 if e2e_ab == "oneset" else i % 2], outs)
        kev[i][1].record(stream)
        y_host.copy_(outs[0], non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    ck_e2e.__exit__(None, None, None)
    copy_ms = sum(a.elapsed_time(b) for a, b in cev)
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    copy_ms /= e2e_steps
    run_ms = sum(a.elapsed_time(b) for a, b in kev) / e2e_steps
    if os.environ.get("BENCH_DEBUG"):
        print(f"[rank {rank}] ms={ms:.2f} e2e_ms={e2e_ms:.2f} copy_ms={copy_ms:.2f} "
              f"kernel_ms={statistics.mean(kernel_ms):.2f}", file=sys.stderr, flush=True)
    if pg:
        t = torch.tensor([e2e_ms], device=f"cuda:{local}")
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        e2e_ms = float(t.item())
        b = torch.tensor([h2d, d2h], device=f"cuda:{local}", dtype=torch.float64)
        pg.all_reduce(b, op=pg.ReduceOp.SUM)   # whole job: every rank's copies
        h2d, d2h = int(b[0].item()), int(b[1].item())
    if rank != 0:
        if pg:
            pg.destroy_process_group()
        return
    pk = peaks()
    fl = flops_per_step(c, lens_sum)
    if pipe:   # rank 0's stage: its share of the layers
        from paper_1805_01772_b200.models import layer_partition
        l0, l1 = layer_partition(c["L"], world, 0)
        fl = fl * (l1 - l0) / c["L"]
    kms = statistics.mean(kernel_ms)
    if prec == cf.F32:
        mhz = pk.get("sm_max_mhz", 1965.0)
        peak = 148 * 128 * 2 * mhz * 1e6 / 1e12       # fp32 FFMA lanes x 2 flop x clock
        roof = {"bound": "alu", "achieved": fl / (kms * 1e-3) / 1e12, "peak": peak,
                "unit": "TFLOP/s", "frac": None, "traffic": None,
                "peak_source": "derived: 148 SM x 128 FP32 lanes x 2 x sm_max_mhz (DESIGN.md)",
                "kernel": "cf_driver_kernel (persistent; all heavy work)"}
    else:
        peak = pk.get("bf16_tflops_sustained", 1360.6)
        roof = {"bound": "tensor", "achieved": fl / (kms * 1e-3) / 1e12, "peak": peak,
                "unit": "TFLOP/s", "frac": None, "traffic": None,
                "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained",
                "kernel": "cf_driver_kernel (persistent; all heavy work)"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    traffic_file = os.path.join(ROOT, "profiles", f"traffic_{args.config}_{args.precision}.json")
    if os.path.exists(traffic_file):
        try:
            roof["traffic"] = json.load(open(traffic_file)).get("bytes_per_launch")
        except Exception:
            pass
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline(c, args.config, min(args.cpu_T, c["T"]))
    line = {
        "metric": "LSTM fwd+bwd sequence-steps/sec",
        "value": lens_sum * (1 if pipe else world) / (ms * 1e-3),
        "unit": "sequence-steps/s",
        "n_gpus": world, "steps": args.steps, "warmup": W, "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong" if pipe else "weak",
        "vs_baseline": None,
        "dtype": args.precision,
        "data": "synthetic (seeded; synth.rnn_inputs)",
        "config": {"workload": args.config, **{k: c[k] for k in ("T", "B", "I", "H", "L")},
                   "lengths": c["len_mode"], "parallel_iterations": args.K or 32,
                   "parallelism": (f"layer-pipeline{world}" if pipe else f"dp{world}" if dp
                                   else f"replicas{world}") if world > 1 else "single",
                   "l2": "inputs/activations > L2 (no flush needed)"},
        "loop_iterations_per_s": c["T"] / (ms * 1e-3),
        "kernel_ms": kms,
        "tflops": fl / (ms * 1e-3) / 1e12,
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": dict(clk.summary(), remeasured=remeasured),
        "e2e": {"value": lens_sum * (1 if pipe else world) / (e2e_ms * 1e-3),
                "unit": "sequence-steps/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "h2d_ms_per_step": copy_ms,
                "run_ms_per_step": run_ms,
                "clocks": ck_e2e.summary()},
        "gpu_launches": 2 * args.steps,   # per cf_run: cf_stage_kernel + cf_driver_kernel
        "stack_swap": swap,
    }
    print(json.dumps(line), flush=True)
    if pg:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
