"""One cf_run (after warm-up) of a workload, for ncu captures."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
from bench import CONFIGS  # noqa: E402
from paper_1805_01772_b200 import cf  # noqa: E402
from paper_1805_01772_b200.models import dynamic_rnn_lstm, feeds_to_device  # noqa: E402
from synth import rnn_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3")
ap.add_argument("--precision", default="bf16")
ap.add_argument("--T", type=int, default=0)
ap.add_argument("--runs", type=int, default=2)
ap.add_argument("--no-tiles", action="store_true", help="workers skip tile bodies (driver alone)")
a = ap.parse_args()
c = dict(CONFIGS[a.config])
if a.T:
    c["T"] = a.T
prec = cf.BF16 if a.precision == "bf16" else cf.F32
if a.no_tiles:
    cf.debug_set_flags(1)
p = dynamic_rnn_lstm(c["T"], c["B"], c["I"], c["H"], c["L"])
s = cf.Session(p.g, p.fetch_tensors(), precision=prec)
f = rnn_inputs(c["T"], c["B"], c["I"], c["H"], c["L"], seed=0, len_mode=c["len_mode"], bf16=prec == cf.BF16)
dev = feeds_to_device(f, session=s)
outs = s.alloc_outputs()
for _ in range(a.runs):
    _, _, tr = s.run(dev, outs, trace=True)
torch.cuda.synchronize()
print("ok", tr["wall_ms"])
