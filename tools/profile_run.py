"""Run one workload with the device-side instance profiler and summarise where time goes."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

# the profiler is compiled into libcf_prof.so only: build it and select it before cf loads
os.environ["CF_LIB"] = "libcf_prof.so"
__graft_entry__.build(profile=True)
from bench import CONFIGS  # noqa: E402
from paper_1805_01772_b200 import cf  # noqa: E402
from paper_1805_01772_b200.models import dynamic_rnn_lstm, feeds_to_device  # noqa: E402
from synth import rnn_inputs  # noqa: E402

KINDS = ["NOP", "EW", "FILL", "COPY", "REDUCE_SUM", "REDUCE_SUM0", "MATMUL", "LSTM_FWD",
         "LSTM_BWD_EW", "LSTM_BWD_MM", "ACC", "PREP_WP", "PREP_WT", "LSTM_FWD_TC",
         "LSTM_BWD_EW_BF", "LSTM_DXH_TC", "LSTM_DW_TC", "SWAP", "WAIT", "LSTM_XPROJ_TC", "MATMUL_TC"]

OPS = ["NOP", "PLACEHOLDER", "CONST", "PASS", "SWITCH", "MERGE", "MERGE_LOOP", "ENTER", "EXIT",
       "NEXTITER", "SCALAR", "REDUCE_I", "SLICE_I", "FLOW", "TA_CREATE", "TA_READ", "TA_WRITE",
       "TA_STACK", "TA_UNSTACK", "TA_GRAD", "STACK_CREATE", "STACK_PUSH", "STACK_POP", "HEAVY", "ACC",
       "SEND", "RECV"]
OPS = OPS + ["RING_FULL_WAIT", "BL_WAKE", "BL_CHECK", "BL_RESERVE"] + ["SMEM_MASK"]
OPS += ["R_RUN_BODY", "R_NEW_INST", "R_PUBLISH", "R_RESOLVE", "R_DRAIN", "R_ADD_DEP", "R_PLACE",
        "R_PREP", "R_FLUSH_DW", "R_EVAL_LSTM_TC", "R_EVAL_HEAVY", "R_DRAIN_IO", "R_COMPLETE",
        "R_WAVE", "F_PREP_RESOLVE", "F_NEW_INST", "F_FIELDS", "F_ADD_DEPS", "F_OUT_SUBMIT",
        "H_PLACES", "W_WAIT", "W_WAIT_DRAIN", "W_HELPER_BUSY(n=leftovers)", "R_BATCH",
        "B_DRV_RESERVE", "BL_PLACE", "BL_BUILD", "BL_SUBMIT_TAIL", "B_DRV_SUBMIT", "B_F_RECORD"]
OPS = OPS + ["?%d" % k for k in range(len(OPS), 62)] + ["R_SWITCH_FAST", "B_F_DEPS"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--precision", default="bf16")
    ap.add_argument("--T", type=int, default=0)
    ap.add_argument("--K", type=int, default=0)
    ap.add_argument("--stack-budget", type=int, default=0)
    ap.add_argument("--swap-smallest-first", action="store_true")
    ap.add_argument("--out", default="gpurun_out/profile.json")
    ap.add_argument("--no-tiles", action="store_true", help="workers skip tile bodies (driver alone)")
    ap.add_argument("--fwd-only", action="store_true", help="the forward loop alone (no gradients)")
    ap.add_argument("--workers", type=int, default=0, help="worker CTAs (0: one per SM but the driver's)")
    a = ap.parse_args()
    c = dict(CONFIGS[a.config])
    if a.T:
        c["T"] = a.T
    prec = cf.BF16 if a.precision == "bf16" else cf.F32
    if a.no_tiles:
        cf.debug_set_flags(1)
    kw = {"moe": True, "moe_act": c.get("moe_act", "relu")} if c.get("moe") else {}
    p = dynamic_rnn_lstm(c["T"], c["B"], c["I"], c["H"], c["L"], with_grads=not a.fwd_only, **kw)
    s = cf.Session(p.g, p.fetch_tensors(), precision=prec, parallel_iterations=a.K, profile=True,
                   num_workers=a.workers,
                   stack_budget_bytes=a.stack_budget, swap_smallest_first=a.swap_smallest_first)
    f = rnn_inputs(c["T"], c["B"], c["I"], c["H"], c["L"], seed=0, len_mode=c["len_mode"], bf16=prec == cf.BF16,
                   moe=c.get("moe", False))
    dev = feeds_to_device(f, session=s)
    outs = s.alloc_outputs()
    for _ in range(2):
        s.run(dev, outs)
    _, _, tr = s.run(dev, outs, trace=True)
    torch.cuda.synchronize()
    rows, (t0, t1) = s.profile()
    rows = rows[rows[:, 0] > 0]
    wall = (t1 - t0) * 1e-6
    workers = torch.cuda.get_device_properties(0).multi_processor_count - 1
    res = {"config": c, "wall_ms": wall, "kernel_ms": tr["wall_ms"], "instances": int(rows.shape[0]),
           "busy_frac": float(rows[:, 4].sum() * 1e-6 / (workers * wall)), "kinds": {}}
    for k in np.unique(rows[:, 5]).astype(int):
        r = rows[rows[:, 5] == k]
        tiles = r[:, 6].sum()
        res["kinds"][KINDS[k]] = {
            "n": int(r.shape[0]), "tiles": int(tiles),
            "busy_ms": float(r[:, 4].sum() * 1e-6),
            "us_per_tile": float(r[:, 4].sum() * 1e-3 / max(tiles, 1)),
            "dep_wait_us_mean": float(np.mean(r[:, 1] - r[:, 0]) * 1e-3),
            "queue_wait_us_mean": float(np.mean(r[:, 2] - r[:, 1]) * 1e-3),
            "span_us_mean": float(np.mean(r[:, 3] - r[:, 2]) * 1e-3),
        }
    # timeline: active instances over time (coarse)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    res["driver"] = {OPS[k]: {"n": n, "us": cyc / 1965.0}
                     for k, (n, cyc) in enumerate(s.driver_ops) if n}
    res["describe"] = s.describe()
    json.dump(res, open(a.out, "w"), indent=1)
    rel = rows.copy()
    rel[:, :4] = np.where(rel[:, :4] > 1.8e19, np.nan, rel[:, :4] - t0)
    np.save(a.out.replace(".json", ".npy"), rel)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
