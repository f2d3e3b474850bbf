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


@pytest.mark.parametrize("barrier", [False, True])
def test_exchange_two_gpus(barrier):
    """Each iteration Sends the loop value to the next rank and Recvs the previous rank's
    (PAPER.md:780-829), or (barrier) exchanges it with every rank and averages (the paper's
    loop "with a barrier"); closed form a == n on every rank, K 1 and 8."""
    import json
    import subprocess

    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517",
           os.path.join(root, "tools", "control_overhead_mgpu.py"),
           "--iters", "1", "300", "--K", "1", "8", "--reps", "1"] + (["--barrier"] if barrier else [])
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=240, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    rows = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(rows) == 4
    assert all(r["closed_form_ok"] and r["n_gpus"] == 2 for r in rows), rows
