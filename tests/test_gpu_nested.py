"""GPU: a while_loop nested in a while_loop and its recursive gradient on the device driver
("for nested loops, we apply our techniques recursively",
PAPER.md:1094-1098). The ponder RNN: per step t the state takes x[t] and then runs an inner
loop of n[t] (fed, ragged) tanh(a W + c) updates. Values and gradients against the fp64 oracle
(fp32 path, 1e-5 normwise), trip counts per frame (summed over a nested frame's instances) and
push/pop counts bit-exact, results bit-identical across parallel_iterations."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import __graft_entry__  # noqa: E402

__graft_entry__.build()

from paper_1805_01772_b200 import cf  # noqa: E402
from paper_1805_01772_b200.models import feeds_to_device, ponder_rnn  # noqa: E402

from oracle.models import ponder_rnn as oracle_ponder  # noqa: E402
from oracle.models import run_program  # noqa: E402


def _feeds(T, B, D, seed, counts):
    rng = np.random.default_rng(seed)
    k = 1.0 / np.sqrt(D)
    return {"x": rng.standard_normal((T, B, D)), "n": np.asarray(counts, dtype=np.int64),
            "W": rng.uniform(-k, k, (D, D)) * 2.0, "c": 0.1 * rng.standard_normal((B, D)),
            "a0": 0.1 * rng.standard_normal((B, D)), "R": rng.standard_normal((B, D))}


def _device(T, B, D, f, K):
    p = ponder_rnn(T, B, D, K=K)
    s = cf.Session(p.g, p.fetch_tensors(), precision=cf.F32, max_iterations=8)
    outs, dead, tr = s.run(feeds_to_device(f, session=s), trace=True)
    torch.cuda.synchronize()
    assert not any(dead)
    return {n: o.double().cpu().numpy() for n, o in zip(p.fetch_names(), outs)}, tr


@pytest.mark.parametrize("K", [2, 32])
@pytest.mark.parametrize("counts", [[2, 2, 2, 2, 2], [1, 3, 0, 2, 4], [0, 0, 1, 0, 0]])
def test_ponder_rnn_matches_oracle(counts, K):
    """K = 2: the enclosing loop's ring wraps (5 steps, 3 slots); a loop variable's initial
    value enters the inner frame from that ring and is pushed there: it must be pinned."""
    T, B, D = 5, 3, 64
    f = _feeds(T, B, D, 3, counts)
    dev, tr = _device(T, B, D, f, K)
    ref, otr = run_program(oracle_ponder(T, B, D), f, return_trace=True)
    for k, v in ref.items():
        r = np.asarray(v, dtype=np.float64)
        err = np.abs(dev[k] - r).max() / max(np.abs(r).max(), 1e-30)
        assert err <= 1e-5, (k, err)
    # trip counts summed over the instances of each frame (the ponder frames run once per
    # outer iteration, plus a dead instance in the exiting one: 0 trips)
    want = {}
    for (tag, name), v in otr.trip_counts.items():
        want[name] = want.get(name, 0) + v
    assert sorted(tr["trip_count"]) == sorted(want.values()), (tr["trip_count"], want)
    assert want["ponder"] == sum(counts) and want["steps"] == T
    assert tr["pushes"] == sum(otr.pushes.values()) == tr["pops"]
    assert tr["exit_fires"] == sum(otr.exit_fires.values())


@pytest.mark.parametrize("K", [1, 2, 32])
def test_ponder_rnn_parallel_iterations_bit_identical(K):
    T, B, D = 5, 4, 64
    f = _feeds(T, B, D, 5, [1, 3, 2, 0, 3])
    a, _ = _device(T, B, D, f, 1)
    b, tr = _device(T, B, D, f, K)
    for k in a:
        assert np.array_equal(a[k], b[k]), k
