"""f2 debug: per-output error vs the oracle for several parallel_iterations values."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_1805_01772_b200 import cf  # noqa: E402
from paper_1805_01772_b200.models import feeds_to_device, ponder_rnn  # noqa: E402
from oracle.models import ponder_rnn as oracle_ponder, run_program  # noqa: E402

T, B, D = 5, 4, 64
counts = [int(c) for c in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 3, 2, 0, 3]
T = len(counts)
rng = np.random.default_rng(5)
k = 1.0 / np.sqrt(D)
f = {"x": rng.standard_normal((T, B, D)), "n": np.asarray(counts, dtype=np.int64),
     "W": rng.uniform(-k, k, (D, D)) * 2.0, "c": 0.1 * rng.standard_normal((B, D)),
     "a0": 0.1 * rng.standard_normal((B, D)), "R": rng.standard_normal((B, D))}
ref = run_program(oracle_ponder(T, B, D), f)
for K in (1, 2, 3, 4, 32):
    p = ponder_rnn(T, B, D, K=K)
    s = cf.Session(p.g, p.fetch_tensors(), precision=cf.F32, max_iterations=8)
    outs, dead, tr = s.run(feeds_to_device(f, session=s), trace=True)
    torch.cuda.synchronize()
    errs = {}
    for n, o in zip(p.fetch_names(), outs):
        r = np.asarray(ref[n], dtype=np.float64)
        errs[n] = float(np.abs(o.double().cpu().numpy() - r).max() / max(np.abs(r).max(), 1e-30))
    print("K", K, "trips", tr["trip_count"], " ".join(f"{n}:{e:.1e}" for n, e in errs.items()), flush=True)
