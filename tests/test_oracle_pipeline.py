"""Oracle: the layer-partitioned pipeline (§4.4).

Pins: the partitioned program is the full program cut at layer boundaries, so every stage's
outputs and gradients must equal the unpartitioned oracle's exactly (the same fp64 operations
in the same order), and the stage losses must sum to the full loss. The Send/Recv message
count per edge and direction is T + 1: T live iterations plus the dead signal of the exiting
iteration. The gloo test runs the stages as separate processes over
torch.distributed point-to-point, the transport of the N>1 path's host side."""
import os
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle.models import dynamic_rnn_lstm, layer_partition, run_program, run_pipeline_threads
from synth import rnn_inputs


def test_layer_partition():
    for L in range(1, 9):
        for w in range(1, L + 1):
            parts = [layer_partition(L, w, r) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == L
            for (a0, a1), (b0, b1) in zip(parts, parts[1:]):
                assert a1 == b0
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 1
    with pytest.raises(ValueError):
        layer_partition(2, 3, 0)


@pytest.mark.parametrize("mode,world", [("full", 2), ("uniform", 2), ("with_zero", 3), ("capped", 4)])
def test_pipeline_equals_full(mode, world):
    T, B, I, H, L = 5, 3, 4, 6, 4
    f = rnn_inputs(T, B, I, H, L, seed=7, len_mode=mode)
    full, ftr = run_program(dynamic_rnn_lstm(T, B, I, H, L), f, return_trace=True)
    res = run_pipeline_threads(T, B, I, H, L, world, f, sched_seed=11)
    y = 0.0
    seen = set()
    for r, (out, tr) in enumerate(res):
        y += out["y"]
        for k, v in out.items():
            if k == "y":
                continue
            assert k not in seen
            seen.add(k)
            np.testing.assert_array_equal(np.asarray(v), np.asarray(full[k]), err_msg=k)
        # control replicated per stage: same trip counts as the full program
        assert sorted(tr.trip_counts.values()) == sorted(ftr.trip_counts.values())
        edges = (r > 0) + (r < world - 1)
        assert tr.sends == tr.recvs == edges * (T + 1)
    assert seen == set(full) - {"y"}
    assert abs(y - full["y"]) <= 1e-12 * max(1.0, abs(full["y"]))


def test_pipeline_moe_and_k1():
    T, B, I, H, L = 4, 2, 3, 4, 2
    f = rnn_inputs(T, B, I, H, L, seed=3, len_mode="uniform", moe=True)
    full = run_program(dynamic_rnn_lstm(T, B, I, H, L, moe=True), f)
    res = run_pipeline_threads(T, B, I, H, L, 2, f, K=1, moe=True)
    for out, _ in res:
        for k, v in out.items():
            if k != "y":
                np.testing.assert_array_equal(np.asarray(v), np.asarray(full[k]), err_msg=k)


def _gloo_stage(rank, world, port, outdir):
    import torch.distributed as dist

    from oracle.transport import DistTransport
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    T, B, I, H, L = 4, 2, 3, 5, 3
    f = rnn_inputs(T, B, I, H, L, seed=5, len_mode="uniform")
    tp = DistTransport()
    out = run_program(dynamic_rnn_lstm(T, B, I, H, L, stage=(rank, world)), f, transport=tp)
    tp.finish()
    dist.barrier()
    np.savez(os.path.join(outdir, f"r{rank}.npz"), **{k: np.asarray(v) for k, v in out.items()})
    dist.destroy_process_group()


def test_pipeline_gloo_world2():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gloo_stage, args=(2, port, d), nprocs=2, join=True)
        T, B, I, H, L = 4, 2, 3, 5, 3
        f = rnn_inputs(T, B, I, H, L, seed=5, len_mode="uniform")
        full = run_program(dynamic_rnn_lstm(T, B, I, H, L), f)
        y = 0.0
        for r in range(2):
            z = np.load(os.path.join(d, f"r{r}.npz"))
            y += float(z["y"])
            for k in z.files:
                if k != "y":
                    np.testing.assert_array_equal(z[k], np.asarray(full[k]), err_msg=k)
        assert abs(y - full["y"]) <= 1e-12 * max(1.0, abs(full["y"]))
