"""Race check: the results must not depend on the order and timing in which the
workers run the tiles. With cf_run_opts.sched_seed != 0 every claim attempt sleeps a
pseudo-random 0-4 us and picks the high / low-priority ring order at random
(runtime.cu worker_loop try_claim), so instances complete in other orders and the driver sees
other completion interleavings. The runtime's reductions have fixed orders (dW chunks in step
order behind the accumulator's last writer, db partials summed in row-tile order, ReduceSum's
two levels), so every fetched tensor must be bit-identical to the FIFO schedule's, and the
control trace identical.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import __graft_entry__  # noqa: E402

__graft_entry__.build()

from paper_1805_01772_b200 import cf  # noqa: E402
from paper_1805_01772_b200.models import dynamic_rnn_lstm, feeds_to_device  # noqa: E402
from synth import rnn_inputs  # noqa: E402


def run(p, f, precision, seed, T, K=0):
    s = cf.Session(p.g, p.fetch_tensors(), precision=precision, parallel_iterations=K,
                   sched_seed=seed)
    outs, dead, tr = s.run(feeds_to_device(f, session=s), trace=True, branch_cap=64 * (T + 1))
    torch.cuda.synchronize()
    return [o.cpu() for o in outs], tr


@pytest.mark.parametrize("case", ["f32_ragged", "bf16_256row", "bf16_moe", "bf16_cfg3_shape"])
def test_schedule_perturbation_bit_identical(case):
    if case == "bf16_cfg3_shape":   # 8-member heavy batches: the lanes' edges race the routing after them
        T, B, I, H, L, prec, kw, mode = 9, 512, 1024, 1024, 8, cf.BF16, {}, "uniform"
    elif case == "f32_ragged":
        T, B, I, H, L, prec, kw, mode = 7, 40, 24, 32, 3, cf.F32, {}, "uniform"
    elif case == "bf16_256row":   # 256-row tiles, chunked dW (T > 8), ragged lengths
        T, B, I, H, L, prec, kw, mode = 19, 512, 256, 256, 2, cf.BF16, {}, "uniform"
    else:
        T, B, I, H, L, prec, kw, mode = 9, 96, 256, 256, 2, cf.BF16, {"moe": True, "moe_act": "tanh"}, "uniform"
    p = dynamic_rnn_lstm(T, B, I, H, L, **kw)
    f = rnn_inputs(T, B, I, H, L, seed=3, len_mode=mode, moe=kw.get("moe", False), bf16=prec == cf.BF16)
    base, btr = run(p, f, prec, 0, T)
    for seed in (1, 2, 3):
        got, tr = run(p, f, prec, seed, T)
        for name, a, b in zip(p.fetch_names(), base, got):
            assert torch.equal(a, b), (seed, name)
        for k in ("trip_count", "pushes", "pops", "exit_fires"):
            assert tr[k] == btr[k], (seed, k)
        assert tr["branch_bits"] == btr["branch_bits"]
