"""the trivial-body loop of the paper's E1 on the device
driver. Closed form: trip count n and a == n elementwise, for any parallel_iterations K, including a loop
longer than the 16-bit iteration field of the driver's in-flight ring (n = 70000)."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,width,K", [(0, 1, 1), (1, 1, 1), (257, 3, 1), (2000, 1, 32), (1500, 64, 8), (70000, 2, 32)])
def test_trivial_loop_closed_form(n, width, K):
    import control_overhead as co
    r = co.run(n, width=width, K=K, reps=1, warmup=0)
    assert r["trip_count"] == n
    assert r["closed_form_ok"], r
