"""GPU parity of the layer-partitioned pipeline.

One process per GPU (torch.multiprocessing, gloo for the channel-handle exchange only); the
data path is the driver kernels' Send/Recv over NVLink peer memory. Each stage's outputs and
gradients are compared with the unpartitioned fp64 oracle (same bar as tests/test_gpu_parity),
its control trace with the oracle's per-stage trace (bit-exact, including the T + 1 messages
per edge and direction), and a second run checks that run epochs keep messages apart
(results bit-identical to the first run). Needs >= 2 GPUs; skipped otherwise.
"""
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
from oracle.models import run_pipeline_threads, run_program  # noqa: E402
from synth import rnn_inputs  # noqa: E402

BF16_TOL = 2e-2
needs2 = pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                            reason="needs 2 GPUs")


def _worker(rank, world, port, cfg, outdir):
    import torch.distributed as dist

    from paper_1805_01772_b200 import cf
    from paper_1805_01772_b200.models import dynamic_rnn_lstm, feeds_to_device
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    T, B, I, H, L, mode, prec = cfg
    precision = cf.BF16 if prec == "bf16" else cf.F32
    f = rnn_inputs(T, B, I, H, L, seed=3, len_mode=mode, bf16=prec == "bf16")
    p = dynamic_rnn_lstm(T, B, I, H, L, stage=(rank, world))
    s = cf.Session(p.g, p.fetch_tensors(), precision=precision, device=rank, watchdog_ms=120000)
    s.connect_pipeline()
    dev = feeds_to_device(f, device=f"cuda:{rank}", session=s)
    res = []
    for _ in range(2):
        outs, dead, tr = s.run(dev, trace=True, branch_cap=64 * (T + 1))
        torch.cuda.synchronize()
        assert not any(dead)
        res.append(({n: o.double().cpu().numpy() for n, o in zip(p.fetch_names(), outs)}, tr))
    (v0, tr), (v1, _) = res
    for k in v0:
        assert np.array_equal(v0[k], v1[k]), f"rank {rank}: second run differs in {k}"
    np.savez(os.path.join(outdir, f"r{rank}.npz"), **v0)
    np.savez(os.path.join(outdir, f"t{rank}.npz"), trip=np.array(tr["trip_count"]),
             pushes=tr["pushes"], pops=tr["pops"], sends=tr["sends"], recvs=tr["recvs"],
             exit_fires=tr["exit_fires"])
    dist.barrier()
    dist.destroy_process_group()


def _run(cfg, world=2):
    import torch.multiprocessing as mp
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, port, cfg, d), nprocs=world, join=True)
        vals = [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(world)]
        trs = [dict(np.load(os.path.join(d, f"t{r}.npz"))) for r in range(world)]
    return vals, trs


def _check(cfg, tol, world=2):
    T, B, I, H, L, mode, prec = cfg
    vals, trs = _run(cfg, world)
    f = rnn_inputs(T, B, I, H, L, seed=3, len_mode=mode, bf16=prec == "bf16")
    ref = run_program(oracle_rnn(T, B, I, H, L), f)   # plain fp64 (reading R16)
    stages = run_pipeline_threads(T, B, I, H, L, world, f)
    y = 0.0
    for r in range(world):
        y += float(vals[r]["y"])
        for k, v in vals[r].items():
            if k == "y":
                continue
            rr = np.asarray(ref[k], dtype=np.float64)
            err = np.abs(v - rr).max() / max(np.abs(rr).max(), 1e-30)
            assert err <= tol, (r, k, err)
        _, otr = stages[r]
        t = trs[r]
        assert list(t["trip"][:2]) == [otr.trip_counts[((), "rnn")], otr.trip_counts[((), "rnn_grad")]]
        assert int(t["pushes"]) == sum(otr.pushes.values()) == int(t["pops"])
        assert int(t["sends"]) == otr.sends and int(t["recvs"]) == otr.recvs
        assert int(t["exit_fires"]) == sum(otr.exit_fires.values())
        ys = float(stages[r][0]["y"])   # the stage's part of the loss (oracle, same stage graph)
        assert abs(float(vals[r]["y"]) - ys) <= tol * abs(ys), (r, float(vals[r]["y"]), ys)
    # the stage losses sum to the full model's loss (oracle identity, fp64)
    assert abs(sum(float(st[0]["y"]) for st in stages) - float(ref["y"])) <= 1e-9 * abs(float(ref["y"]))


@needs2
@pytest.mark.parametrize("mode", ["uniform", "full"])
def test_pipeline_fp32_two_gpus(mode):
    _check((6, 5, 12, 16, 4, mode, "f32"), 1e-5)


@needs2
def test_pipeline_bf16_two_gpus():
    _check((5, 40, 256, 256, 2, "uniform", "bf16"), BF16_TOL)


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 4,
                    reason="needs 4 GPUs")
def test_pipeline_fp32_four_gpus():
    _check((5, 3, 8, 16, 4, "capped", "f32"), 1e-5, world=4)


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 4,
                    reason="needs 4 GPUs")
def test_pipeline_bf16_four_gpus():
    """cfg3's stage layout in small: 8 layers over 4 stages on the tcgen05 path."""
    _check((6, 256, 256, 256, 8, "upper_half", "bf16"), BF16_TOL, world=4)
