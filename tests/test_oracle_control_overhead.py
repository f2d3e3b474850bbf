"""§8(f) f1 on CPU: the paper's trivial-body loop in the oracle.

Pins: the closed form (trip count n, a == n elementwise) from the oracle interpreter for
n = 0, 1 and a ragged width, for K 1 and 32. The C-ABI builder lowers tools/control_overhead.py's
graph to the same primitive counts as the oracle builder (host logic only; no GPU call)."""
import os
import sys

import numpy as np
import pytest

from oracle import interp
from oracle.graph import FLOAT, INT, Builder

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


def _oracle_loop(width):
    b = Builder()
    n = b.placeholder("n", INT, ())
    a0 = b.placeholder("a0", FLOAT, (width,))
    one_i = b.const(1, INT)
    i_out, a_out = b.while_loop(lambda i, a: b.less(i, n),
                                lambda i, a: [b.add(i, one_i), b.add(a, b.const(1.0, FLOAT))],
                                [b.const(0, INT), a0])
    return b, i_out, a_out


@pytest.mark.parametrize("n,width,K", [(0, 1, 1), (1, 1, 32), (37, 3, 1), (37, 3, 32)])
def test_trivial_loop_closed_form_oracle(n, width, K):
    b, i_out, a_out = _oracle_loop(width)
    (iv, av), tr = interp.run(b.g, {"n": n, "a0": np.zeros(width)}, [i_out, a_out],
                              return_trace=True, K_override=K)
    assert int(iv) == n
    assert np.array_equal(np.asarray(av), np.full(width, float(n)))
    assert list(tr.trip_counts.values()) == [n]


def test_capi_lowers_like_oracle():
    import control_overhead as co
    g, _ = co.build(3)
    b, _, _ = _oracle_loop(3)
    assert g.count_ops() == b.g.count_ops()
    assert g.validate() == []
