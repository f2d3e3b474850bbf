"""GPU: batch data parallelism with the in-graph gradient allreduce.

Two ranks, one GPU each, each running the whole model on half of a batch; the weight
gradients are exchanged over NVLink peer memory by root-level Send/Recv and summed (AddN).
Every rank's summed dW / db must equal the full batch's gradient from the fp64 oracle (the
loss is a sum over samples); per-sample gradients (dx, dh0, dc0) equal the oracle's rows of
that rank. Needs 2 GPUs."""
import os
import socket
import tempfile

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import __graft_entry__  # noqa: E402

__graft_entry__.build()

from oracle.models import dynamic_rnn_lstm as oracle_rnn  # noqa: E402
from oracle.models import run_program  # noqa: E402
from synth import rnn_inputs  # noqa: E402


def _worker(rank, world, port, cfg, outdir):
    import torch.distributed as dist

    from paper_1805_01772_b200 import cf
    from paper_1805_01772_b200.models import dynamic_rnn_lstm, feeds_to_device
    from synth import shard_inputs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    T, B, I, H, L, mode, prec = cfg
    precision = cf.BF16 if prec == "bf16" else cf.F32
    f = shard_inputs(rnn_inputs(T, B, I, H, L, seed=4, len_mode=mode, bf16=prec == "bf16"), rank, world)
    p = dynamic_rnn_lstm(T, B // world, I, H, L, dp=(rank, world))
    s = cf.Session(p.g, p.fetch_tensors(), precision=precision, device=rank, watchdog_ms=120000)
    s.connect_pipeline()
    dev = feeds_to_device(f, device=f"cuda:{rank}", session=s)
    res = []
    for _ in range(2):   # run epochs keep the exchanges of consecutive runs apart
        outs, dead, tr = s.run(dev, trace=True)
        torch.cuda.synchronize()
        assert not any(dead)
        res.append({n: o.double().cpu().numpy() for n, o in zip(p.fetch_names(), outs)})
    for k in res[0]:
        assert np.array_equal(res[0][k], res[1][k]), f"rank {rank}: second run differs in {k}"
    np.savez(os.path.join(outdir, f"r{rank}.npz"), **res[0])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("cfg,tol", [((6, 10, 12, 16, 2, "uniform", "f32"), 1e-5),
                                     ((6, 128, 256, 256, 2, "uniform", "bf16"), 2e-2)])
def test_dp_two_gpus_matches_full_batch(cfg, tol):
    import torch.multiprocessing as mp
    world = 2
    T, B, I, H, L, mode, prec = cfg
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, port, cfg, d), nprocs=world, join=True)
        vals = [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(world)]
    f = rnn_inputs(T, B, I, H, L, seed=4, len_mode=mode, bf16=prec == "bf16")
    ref = run_program(oracle_rnn(T, B, I, H, L), f)   # the full batch, fp64
    b = B // world
    for r in range(world):
        for k, v in vals[r].items():
            rr = np.asarray(ref[k], dtype=np.float64)
            if k.startswith(("dW", "db")):
                pass                                   # summed over the ranks: full batch
            elif k in ("dx", "out"):
                rr = rr[:, r * b:(r + 1) * b]
            elif k.startswith(("dh0", "dc0", "hT", "cT")):
                rr = rr[r * b:(r + 1) * b]
            else:
                continue                               # y: this rank's part of the loss
            err = np.abs(v - rr).max() / max(np.abs(rr).max(), 1e-30)
            assert err <= tol, (r, k, err)
    for k in vals[0]:   # the summed gradients are the same on every rank
        if k.startswith(("dW", "db")):
            assert np.array_equal(vals[0][k], vals[1][k]), k
