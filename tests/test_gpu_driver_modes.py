"""The device driver's scheduling optimisations change WHEN things are evaluated, never WHAT:
every A/B switch of cf_debug_set_flags (include/cf_debug.h) must give bit-identical outputs
and an identical control trace (trip counts, pushes/pops, branch bits) on the bf16
tensor-core path, with variable lengths (dead cond branches) and 3 layers."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import __graft_entry__  # noqa: E402

__graft_entry__.build()

from paper_1805_01772_b200 import cf  # noqa: E402
from paper_1805_01772_b200.models import dynamic_rnn_lstm, feeds_to_device  # noqa: E402
from synth import rnn_inputs  # noqa: E402

# A/B switches (results must not change): poll after every node, helpers spin, release after
# every publication, driver-side LSTM preparation, short poll interval, no prep chaining,
# no wave fusion, poll before heavy nodes, no overlap of the next wave with a forward node /
# a backward node
FLAGS = [4, 8, 16, 128, 1 << 8, 1 << 24, 1 << 25, 1 << 26, 1 << 27, 1 << 29,
         128 | (1 << 24) | (1 << 25) | (1 << 27) | (1 << 29)]


def _run(s, p, dev):
    outs, dead, tr = s.run(dev, trace=True, branch_cap=64 * 13)
    torch.cuda.synchronize()
    return [o.clone() for o in outs], dead, tr


def test_driver_modes_bit_identical():
    T, B, I, H, L = 12, 130, 256, 256, 3
    f = rnn_inputs(T, B, I, H, L, seed=7, len_mode="capped", bf16=True)
    p = dynamic_rnn_lstm(T, B, I, H, L)
    s = cf.Session(p.g, p.fetch_tensors(), precision=cf.BF16)
    dev = feeds_to_device(f, session=s)
    try:
        cf.debug_set_flags(0)
        ref, dead0, tr0 = _run(s, p, dev)
        assert not any(dead0)
        for fl in FLAGS:
            cf.debug_set_flags(fl)
            outs, dead, tr = _run(s, p, dev)
            assert dead == dead0, fl
            for name, a, b in zip(p.fetch_names(), ref, outs):
                assert torch.equal(a, b), (fl, name, float((a.double() - b.double()).abs().max()))
            for key in ("trip_count", "pushes", "pops", "exit_fires", "max_depth"):
                assert tr[key] == tr0[key], (fl, key)
            assert np.array_equal(np.asarray(tr["branch_bits"]), np.asarray(tr0["branch_bits"])), fl
    finally:
        cf.debug_set_flags(0)
