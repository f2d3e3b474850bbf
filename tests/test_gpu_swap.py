"""GPU: stack swapping to pinned host memory.

A stack budget of 1 byte swaps every stacked value of at least swap_min_bytes: its device
storage shrinks to a (K + 1)-slot ring, every push copies the entry to pinned host memory on
the D2H copy stream and every pop whose ring slot was reused brings it back on the H2D stream.
Swapping moves bytes, never changes them: results must be bit-identical to the unswapped run
(and within the parity bar of the oracle), control traces identical, and the swap counters
consistent with the ring size (entries of the last K + 1 iterations are never brought back).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import __graft_entry__  # noqa: E402

__graft_entry__.build()

from paper_1805_01772_b200 import cf  # noqa: E402
from paper_1805_01772_b200.models import dynamic_rnn_lstm, feeds_to_device  # noqa: E402

from oracle.models import dynamic_rnn_lstm as oracle_rnn  # noqa: E402
from oracle.models import run_program  # noqa: E402
from synth import rnn_inputs  # noqa: E402


def run(T, B, I, H, L, f, precision, K, budget, swap_min=0):
    p = dynamic_rnn_lstm(T, B, I, H, L)
    s = cf.Session(p.g, p.fetch_tensors(), precision=precision, parallel_iterations=K,
                   stack_budget_bytes=budget, swap_min_bytes=swap_min)
    outs, dead, tr = s.run(feeds_to_device(f, session=s), trace=True)
    torch.cuda.synchronize()
    assert not any(dead)
    return {n: o.double().cpu().numpy() for n, o in zip(p.fetch_names(), outs)}, tr, s.describe()


@pytest.mark.parametrize("prec,shape,mode,K,tol,smin", [
    ("f32", (9, 70, 40, 72, 2), "uniform", 2, 1e-5, 0),
    ("f32", (12, 5, 12, 16, 1), "full", 1, 1e-5, 64),     # small values: lowered threshold
    ("bf16", (8, 130, 256, 512, 2), "capped", 3, 2e-2, 0),
    # T >= 2 (K + 1) + 8: the swap-in ring wraps while a chunked dW (8 gradient steps) still
    # reads popped x / h (the swap-in ring needs K + 9 slots in bf16 mode)
    ("bf16", (24, 64, 256, 256, 2), "full", 3, 2e-2, 0),
])
def test_swap_bit_identical_and_parity(prec, shape, mode, K, tol, smin):
    T, B, I, H, L = shape
    precision = cf.BF16 if prec == "bf16" else cf.F32
    f = rnn_inputs(T, B, I, H, L, seed=6, len_mode=mode, bf16=prec == "bf16")
    base, btr, _ = run(T, B, I, H, L, f, precision, K, 0)
    sw, tr, desc = run(T, B, I, H, L, f, precision, K, 1, smin)
    assert "swapped arenas=0" not in desc, desc
    assert btr["swap_out"] == 0 and btr["swap_in"] == 0
    for k in base:
        assert np.array_equal(base[k], sw[k]), k
    for key in ("trip_count", "pushes", "pops", "exit_fires"):
        assert tr[key] == btr[key], key
    assert tr["swap_out"] > 0
    # entries of the last K + 1 forward iterations are still in their ring slot at the pop
    assert 0 < tr["swap_in"] < tr["swap_out"]
    assert tr["bytes_d2h"] > tr["bytes_h2d"] > 0
    ref = run_program(oracle_rnn(T, B, I, H, L), f)
    for k in ref:
        r = np.asarray(ref[k], dtype=np.float64)
        err = np.abs(sw[k] - r).max() / max(np.abs(r).max(), 1e-30)
        assert err <= tol, (k, err)


def test_swap_without_wrap_never_swaps_in():
    """T <= K + 1: the ring holds every iteration, so nothing comes back from the host."""
    T, B, I, H, L = 5, 4, 8, 8, 1
    f = rnn_inputs(T, B, I, H, L, seed=1, len_mode="full")
    base, _, _ = run(T, B, I, H, L, f, cf.F32, 32, 0)
    sw, tr, _ = run(T, B, I, H, L, f, cf.F32, 32, 1, 64)
    for k in base:
        assert np.array_equal(base[k], sw[k]), k
    assert tr["swap_out"] > 0 and tr["swap_in"] == 0
