"""Debug runs of the nested ponder RNN on the device (f2): variants and env switches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_1805_01772_b200 import cf  # noqa: E402
from paper_1805_01772_b200.models import feeds_to_device, ponder_rnn  # noqa: E402

T, B, D = int(sys.argv[1]), 3, 64
counts = [int(c) for c in sys.argv[2].split(",")]
K = int(sys.argv[3])
rng = np.random.default_rng(3)
f = {"x": rng.standard_normal((T, B, D)), "n": np.asarray(counts, dtype=np.int64),
     "W": rng.uniform(-0.2, 0.2, (D, D)), "c": 0.1 * rng.standard_normal((B, D)),
     "a0": 0.1 * rng.standard_normal((B, D)), "R": rng.standard_normal((B, D))}
p = ponder_rnn(T, B, D, K=K)
s = cf.Session(p.g, p.fetch_tensors(), precision=cf.F32, max_iterations=8)
try:
    outs, dead, tr = s.run(feeds_to_device(f, session=s), trace=True)
    torch.cuda.synchronize()
    print("OK", {k: tr[k] for k in ("trip_count", "pushes", "pops", "exit_fires", "instances")})
except cf.CfError as e:
    print("ERR", e)
