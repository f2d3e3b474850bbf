import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running")


import pytest  # noqa: E402


@pytest.fixture(autouse=True, scope="session")
def _debug_knobs():
    """CF_TEST_KNOBS="0=4,1=1" runs the GPU tests with cf_debug_set_knob A/B knobs set (knob 0:
    claim-ahead lead in k-blocks, knob 1: no batch/routing overlap)."""
    spec = os.environ.get("CF_TEST_KNOBS")
    if spec:
        from paper_1805_01772_b200 import cf
        for kv in spec.split(","):
            k, v = kv.split("=")
            cf.debug_set_knob(int(k), int(v))
    yield
