"""CPU pins of batch data parallelism in the oracle: the loss is a sum
over samples (reading R11), so the weight gradients of the batch shards sum to the full
batch's and the per-sample values of a shard are the full batch's rows. This is the identity
the device's in-graph allreduce relies on."""
import numpy as np
import pytest

from oracle.models import dynamic_rnn_lstm, run_program
from synth import rnn_inputs, shard_inputs


@pytest.mark.parametrize("world", [2, 4])
def test_shard_gradients_sum_to_full_batch(world):
    T, B, I, H, L = 5, 8, 3, 6, 2
    f = rnn_inputs(T, B, I, H, L, seed=4, len_mode="uniform")
    full = run_program(dynamic_rnn_lstm(T, B, I, H, L), f)
    b = B // world
    parts = [run_program(dynamic_rnn_lstm(T, b, I, H, L), shard_inputs(f, r, world)) for r in range(world)]
    for k, v in full.items():
        v = np.asarray(v, dtype=np.float64)
        if k.startswith(("dW", "db")) or k == "y":
            got = sum(np.asarray(p[k], dtype=np.float64) for p in parts)
        elif k in ("dx", "out"):
            got = np.concatenate([p[k] for p in parts], axis=1)
        else:
            got = np.concatenate([p[k] for p in parts], axis=0)
        assert np.abs(got - v).max() <= 1e-12 * max(1.0, np.abs(v).max()), k
