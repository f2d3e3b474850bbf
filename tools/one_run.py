"""cf_run of a bench config a few times (for ncu captures of one launch: -k regex:cf_driver -s 2 -c 1).

    python tools/one_run.py [cfg3] [runs]     env FLAGS: cf_debug_set_flags value"""
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

c = dict(CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"])
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
p = dynamic_rnn_lstm(c["T"], c["B"], c["I"], c["H"], c["L"])
s = cf.Session(p.g, p.fetch_tensors(), precision=cf.BF16)
f = rnn_inputs(c["T"], c["B"], c["I"], c["H"], c["L"], seed=0, len_mode=c["len_mode"], bf16=True)
dev = feeds_to_device(f, session=s)
outs = s.alloc_outputs()
cf.debug_set_flags(int(os.environ.get("FLAGS", "0")))
for _ in range(runs):
    _, _, tr = s.run(dev, outs, trace=True)
    torch.cuda.synchronize()
    print(f"{tr['wall_ms']:.2f} ms", flush=True)
