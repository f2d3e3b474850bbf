"""A/B of worker roles for the dW chunks (cf_debug_set_worker_roles) on cfg3: ms per run."""
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

c = dict(CONFIGS["cfg3"])
p = dynamic_rnn_lstm(c["T"], c["B"], c["I"], c["H"], c["L"])
s = cf.Session(p.g, p.fetch_tensors(), precision=cf.BF16)
f = rnn_inputs(c["T"], c["B"], c["I"], c["H"], c["L"], seed=0, len_mode=c["len_mode"], bf16=True)
dev = feeds_to_device(f, session=s)
outs = s.alloc_outputs()
for _ in range(2):
    s.run(dev, outs)
for rep in range(2):
    for (n, strict) in [(0, 0), (32, 0), (48, 0), (64, 0), (32, 1), (48, 1), (64, 1)]:
        cf.debug_set_worker_roles(n, strict)
        ts = []
        for _ in range(3):
            _, _, tr = s.run(dev, outs, trace=True)
            ts.append(tr["wall_ms"])
        torch.cuda.synchronize()
        print(f"low_first={n} strict={strict}: {sorted(ts)[1]:.2f} ms", flush=True)
cf.debug_set_worker_roles(0, 0)
