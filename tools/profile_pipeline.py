"""Device-side instance/driver profile of every stage of the layer pipeline (torchrun, one rank
per GPU): writes gpurun_out/pipe_prof_r{rank}.json with wall time, worker busy fraction, per
kind tiles/busy and the driver's per-opcode / per-region cycles."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import __graft_entry__  # noqa: E402

# the profiler is compiled into libcf_prof.so only: build it and select it before cf loads
os.environ["CF_LIB"] = "libcf_prof.so"
__graft_entry__.build(profile=True)
from bench import CONFIGS  # noqa: E402
from paper_1805_01772_b200 import cf  # noqa: E402
from paper_1805_01772_b200.models import dynamic_rnn_lstm, feeds_to_device  # noqa: E402
from synth import rnn_inputs  # noqa: E402
from tools.profile_run import KINDS, OPS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--T", type=int, default=50)
a = ap.parse_args()
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("gloo")
c = dict(CONFIGS[a.config])
c["T"] = a.T
p = dynamic_rnn_lstm(c["T"], c["B"], c["I"], c["H"], c["L"], stage=(rank, world))
s = cf.Session(p.g, p.fetch_tensors(), precision=cf.BF16, device=local, profile=True, watchdog_ms=120000)
s.connect_pipeline()
f = rnn_inputs(c["T"], c["B"], c["I"], c["H"], c["L"], seed=0, len_mode=c["len_mode"], bf16=True)
dev = feeds_to_device(f, device=f"cuda:{local}", session=s)
outs = s.alloc_outputs(device=f"cuda:{local}")
for _ in range(3):
    dist.barrier()
    s.run(dev, outs)
rows, (t0, t1) = s.profile()
rows = rows[rows[:, 0] > 0]
wall = (t1 - t0) * 1e-6
workers = torch.cuda.get_device_properties(local).multi_processor_count - 1
res = {"rank": rank, "world": world, "wall_ms": wall,
       "busy_frac": float(rows[:, 4].sum() * 1e-6 / (workers * wall)), "kinds": {}}
for k in np.unique(rows[:, 5]).astype(int):
    r = rows[rows[:, 5] == k]
    res["kinds"][KINDS[k]] = {"n": int(r.shape[0]), "tiles": int(r[:, 6].sum()),
                              "busy_ms": float(r[:, 4].sum() * 1e-6),
                              "first_start_ms": float(np.nanmin(np.where(r[:, 2] > 1.8e19, np.nan, r[:, 2] - t0)) * 1e-6),
                              "last_end_ms": float(np.nanmax(r[:, 3] - t0) * 1e-6)}
res["driver"] = {OPS[k]: {"n": n, "us": cyc / 1965.0} for k, (n, cyc) in enumerate(s.driver_ops) if n}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open(f"gpurun_out/pipe_prof_r{rank}.json", "w"), indent=1)
dist.barrier()
