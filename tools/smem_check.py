"""Which driver arrays the device driver could stage in shared memory (st->smem_mask) and how
many bytes it used, for one cfg run."""
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
c["T"] = 8
p = dynamic_rnn_lstm(c["T"], c["B"], c["I"], c["H"], c["L"])
s = cf.Session(p.g, p.fetch_tensors(), precision=cf.BF16)
f = rnn_inputs(c["T"], c["B"], c["I"], c["H"], c["L"], seed=0, len_mode=c["len_mode"], bf16=True)
dev = feeds_to_device(f, session=s)
outs = s.alloc_outputs()
s.run(dev, outs)
torch.cuda.synchronize()
s.profile()
n, cyc = s.driver_ops[31]
print(f"smem_mask={n:#x} smem_used={cyc} bytes")
