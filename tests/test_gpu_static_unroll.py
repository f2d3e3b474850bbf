"""GPU: the statically unrolled LSTM (§6.3) through the
same C-ABI and kernels, no control-flow primitive in the graph. Values against the fp64 oracle
of the dynamic program (same math, reading R11 loss), and the static and dynamic device paths
against each other."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import __graft_entry__  # noqa: E402

__graft_entry__.build()

from paper_1805_01772_b200 import cf  # noqa: E402
from paper_1805_01772_b200.models import dynamic_rnn_lstm, feeds_to_device, static_rnn_lstm  # noqa: E402

from oracle.models import dynamic_rnn_lstm as oracle_rnn  # noqa: E402
from oracle.models import run_program  # noqa: E402
from synth import rnn_inputs  # noqa: E402


def _run(p, f, precision):
    s = cf.Session(p.g, p.fetch_tensors(), precision=precision)
    outs, dead, tr = s.run(feeds_to_device(f, session=s), trace=True)
    torch.cuda.synchronize()
    assert not any(dead)
    return {n: o.double().cpu().numpy() for n, o in zip(p.fetch_names(), outs)}, tr


@pytest.mark.parametrize("prec,tol,shape", [("f32", 1e-5, (7, 5, 12, 16, 2)),
                                            ("bf16", 2e-2, (12, 64, 256, 256, 2))])
def test_static_unroll_matches_oracle(prec, tol, shape):
    T, B, I, H, L = shape
    precision = cf.BF16 if prec == "bf16" else cf.F32
    f = rnn_inputs(T, B, I, H, L, seed=2, len_mode="full", bf16=prec == "bf16")
    st, tr = _run(static_rnn_lstm(T, B, I, H, L), f, precision)
    assert tr["n_frames"] == 0 and tr["pushes"] == 0   # no loop, no stack
    ref = run_program(oracle_rnn(T, B, I, H, L), f)
    for k in st:
        r = np.asarray(ref[k], dtype=np.float64)
        err = np.abs(st[k] - r).max() / max(np.abs(r).max(), 1e-30)
        assert err <= tol, (k, err)
    dy, _ = _run(dynamic_rnn_lstm(T, B, I, H, L), f, precision)
    for k in st:   # the two device paths agree (forward values bit-identical: same tiles)
        if k in ("out",) or k.startswith(("hT", "cT")):
            assert np.array_equal(st[k], dy[k]), k
