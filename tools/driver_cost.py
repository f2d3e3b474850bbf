"""Driver cost in isolation: cfg3 cf_run with the workers skipping tile bodies
(cf_debug_set_flags(1)) vs normal, same session. Prints ms per run for both."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

if not os.environ.get("CF_LIB"):
    __graft_entry__.build()
from bench import CONFIGS  # noqa: E402
from paper_1805_01772_b200 import cf  # noqa: E402
from paper_1805_01772_b200.models import dynamic_rnn_lstm, feeds_to_device  # noqa: E402
from synth import rnn_inputs  # noqa: E402

c = dict(CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"])
p = dynamic_rnn_lstm(c["T"], c["B"], c["I"], c["H"], c["L"])
s = cf.Session(p.g, p.fetch_tensors(), precision=cf.BF16, num_workers=int(os.environ.get("NW", "0")))
f = rnn_inputs(c["T"], c["B"], c["I"], c["H"], c["L"], seed=0, len_mode=c["len_mode"], bf16=True)
dev = feeds_to_device(f, session=s)
outs = s.alloc_outputs()
if os.environ.get("M2"):
    cf.debug_set_m2_rows(int(os.environ["M2"]))
    print("m2 rows", os.environ["M2"])
for flags in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else '0,1,0').split(',')]:
    cf.debug_set_flags(flags)
    ts = []
    for _ in range(4):
        _, _, tr = s.run(dev, outs, trace=True)
        ts.append(tr["wall_ms"])
    torch.cuda.synchronize()
    print(f"flags={flags}: ms per run {sorted(ts)[1:]}")
cf.debug_set_flags(0)
