"""A/B of the dW chunk length (debug flag bits 24-27; 0 = 8 steps) on cfg3: ms per run.

Also checks the fetched gradients against the default chunk (fp32 accumulation order is the
only difference, so they agree to rounding)."""
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

c = dict(CONFIGS[os.environ.get("CFG", "cfg3")])
p = dynamic_rnn_lstm(c["T"], c["B"], c["I"], c["H"], c["L"])
s = cf.Session(p.g, p.fetch_tensors(), precision=cf.BF16)
f = rnn_inputs(c["T"], c["B"], c["I"], c["H"], c["L"], seed=0, len_mode=c["len_mode"], bf16=True)
dev = feeds_to_device(f, session=s)
outs = s.alloc_outputs()
for _ in range(2):
    s.run(dev, outs)
torch.cuda.synchronize()
ref = [o.clone() for o in outs]
chunks = [int(x) for x in os.environ.get("CHUNKS", "8 1 2 4 6").split()]
for rep in range(2):
    for ch in chunks:
        cf.debug_set_flags((ch & 15) << 24)
        ts = []
        for _ in range(3):
            _, _, tr = s.run(dev, outs, trace=True)
            ts.append(tr["wall_ms"])
        torch.cuda.synchronize()
        err = max(float(((a.double() - b.double()).abs().max() /
                         (b.double().abs().max() + 1e-30))) for a, b in zip(outs, ref))
        print(f"dw_chunk={ch}: {sorted(ts)[1]:.2f} ms  max rel diff vs chunk 8 {err:.2e}", flush=True)
cf.debug_set_flags(0)
