"""One cf_run of the cfg3 forward loop alone (no gradient loop): for ncu captures of the
forward gate-GEMM tile in isolation (tensor-pipe, L2 and DRAM throughput of that phase)."""
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
for k in ("B", "T", "L", "H", "I"):   # overrides, e.g. B=1024
    if os.environ.get(k):
        c[k] = int(os.environ[k])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p = dynamic_rnn_lstm(c["T"], c["B"], c["I"], c["H"], c["L"], with_grads=False)
s = cf.Session(p.g, p.fetch_tensors(), precision=cf.BF16)
f = rnn_inputs(c["T"], c["B"], c["I"], c["H"], c["L"], seed=0, len_mode=c["len_mode"], bf16=True)
dev = feeds_to_device(f, session=s)
outs = s.alloc_outputs()
flags = [int(x) for x in os.environ.get("FLAGS", "0").split(",")]
for fl in flags:
    cf.debug_set_flags(fl)
    ts = []
    for _ in range(reps):
        _, _, tr = s.run(dev, outs, trace=True)
        ts.append(tr["wall_ms"])
    torch.cuda.synchronize()
    print(f"forward only (flags {fl}, B={c['B']} T={c['T']} L={c['L']}): {sorted(ts)[len(ts) // 2]:.2f} ms "
          f"median of {reps}, {tr['instances']} instances")
    if fl & (1 << 22):   # tile phase clocks (cf_debug.h), averaged over the reps
        ph = cf.debug_tile_phases(reset=True)
        n = max(ph[0], 1)
        print(f"  fwd tile phases: {ph[0]} tiles, setup {ph[1] / n / 1.95e3:.2f} us, mainloop "
              f"{ph[2] / n / 1.95e3:.2f} us, epilogue {ph[3] / n / 1.95e3:.2f} us (1.95 GHz)")
cf.debug_set_flags(0)
