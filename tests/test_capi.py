"""C-ABI host tests (no GPU): the library loads, exports every symbol include/cf.h declares,
and its builder + autodiff (independent C++ code) produce the same graph structure as the
oracle for the same programs. Execution itself has no CPU fallback."""
import os
import re

import numpy as np
import pytest

import __graft_entry__

__graft_entry__.build()

from paper_1805_01772_b200 import cf  # noqa: E402
from paper_1805_01772_b200.models import dynamic_rnn_lstm as dev_rnn  # noqa: E402

from oracle.graph import Builder  # noqa: E402
from oracle.autodiff import gradients as oracle_gradients  # noqa: E402
from oracle.models import dynamic_rnn_lstm as oracle_rnn  # noqa: E402

HDRS = [os.path.join(os.path.dirname(__file__), "..", "include", h) for h in ("cf.h", "cf_debug.h")]


def declared_functions():
    src = "".join(open(h).read() for h in HDRS)
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cf_[a-z_0-9]+)\s*\(", src)) -
                  {"cf_pred_fn", "cf_body_fn", "cf_branch_fn", "cf_status"})


def test_exports_every_declared_symbol():
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(cf._lib, n), n
    assert set(names) == set(cf.EXPORTED)
    assert "sm_100a" in cf.version()


@pytest.mark.parametrize("args,kw", [((5, 2, 4, 8, 1), {}), ((5, 3, 4, 8, 2), {}),
                                     ((4, 2, 3, 4, 1), {"moe": True}),
                                     ((6, 4, 4, 4, 3), {"length_conds": False}),
                                     ((5, 2, 4, 8, 4), {"stage": (0, 2)}),
                                     ((5, 2, 4, 8, 4), {"stage": (1, 2)}),
                                     ((5, 2, 4, 8, 3), {"stage": (1, 3)}),
                                     ((4, 2, 3, 4, 2), {"moe": True, "stage": (1, 2)})])
def test_structure_matches_oracle(args, kw):
    p = dev_rnn(*args, **kw)
    q = oracle_rnn(*args, **kw)
    assert p.g.count_ops() == q.b.g.count_ops()
    assert p.g.validate() == []


def test_nested_loop_structure_matches_oracle():
    """f2: a while_loop nested in a while_loop with its recursive gradient (the ponder RNN):
    same op counts as the oracle's builder + autodiff, and the device compiler lowers it (the
    inner loop is one step, OP_FRAME, of the outer body; nested gradient loops likewise)."""
    from paper_1805_01772_b200.models import ponder_rnn as dev_ponder
    from oracle.models import ponder_rnn as oracle_ponder
    p = dev_ponder(5, 3, 8)
    q = oracle_ponder(5, 3, 8)
    assert p.g.count_ops() == q.b.g.count_ops()
    assert p.g.validate() == []
    os.environ["CF_DEBUG_MAX_ITERATIONS"] = "8"
    try:
        lst = cf.debug_program_listing(p.g, p.fetch_tensors())
    finally:
        del os.environ["CF_DEBUG_MAX_ITERATIONS"]
    assert "nested_frames=1" in lst
    assert lst.count("FRAME ponder") == 2   # forward: ponder in steps; gradient: ponder_grad step
    assert "FRAME ponder_grad" in lst


def test_loop_example_structure_and_validate():
    g = cf.Graph()
    x = g.placeholder("x", cf.F32, (1, 1))
    w = g.placeholder("w", cf.F32, (1, 1))
    n3 = g.const(3, cf.I64)
    _, a = g.while_loop(lambda i, a: g.op1("Less", [i, n3]),
                        lambda i, a: [g.op1("Add", [i, g.const(1, cf.I64)]), g.op1("MatMul", [a, w])],
                        [g.const(0, cf.I64), x])
    y = g.op1("ReduceSum", [a])
    g.gradients(y, [w, x])
    c = g.count_ops()
    assert c["StackPush"] == 1 and c["StackPop"] == 1 and c["StackCreate"] == 1
    assert g.validate() == []
    js = g.json()
    assert js["version"] == 1 and len(js["nodes"]) == g.num_nodes()
    # the oracle builds the same structure
    b = Builder()
    from oracle.graph import FLOAT, INT
    xo, wo = b.placeholder("x", FLOAT, (1, 1)), b.placeholder("w", FLOAT, (1, 1))
    n3o = b.const(3, INT)
    _, ao = b.while_loop(lambda i, a: b.less(i, n3o),
                         lambda i, a: (b.add(i, b.const(1, INT)), b.matmul(a, wo)),
                         [b.const(0, INT), xo])
    oracle_gradients(b, b.reduce_sum(ao), [wo, xo])
    assert b.g.count_ops() == c


def test_errors_match_spec_names():
    g = cf.Graph()
    x = g.placeholder("x", cf.F32, ())
    p = g.placeholder("p", cf.BOOL, ())
    with pytest.raises(cf.CfError) as e:
        g.cond(x, lambda: [x], lambda: [x], 1)
    assert e.value.code == "CF_E_NONBOOL_PRED"
    with pytest.raises(cf.CfError) as e:
        g.cond(p, lambda: [x, x], lambda: [x], 1)
    assert e.value.code == "CF_E_BRANCH_MISMATCH"
    v = g.placeholder("v", cf.F32, (2,))
    with pytest.raises(cf.CfError) as e:
        g.gradients(v, [x])
    assert e.value.code == "CF_E_NONSCALAR_OBJECTIVE"
    with pytest.raises(cf.CfError) as e:
        g.op1("MatMul", [x, x])
    assert e.value.code == "CF_E_SHAPE"
    with pytest.raises(cf.CfError) as e:
        g.placeholder("x", cf.F32, ())
    assert e.value.code == "CF_E_INVALID_GRAPH"


def test_no_cpu_fallback():
    """Without a CUDA device session creation fails loudly (CF_E_CUDA), never falls back."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = dev_rnn(3, 2, 2, 4, 1)
    with pytest.raises(cf.CfError) as e:
        cf.Session(p.g, p.fetch_tensors())
    assert e.value.code == "CF_E_CUDA"


def test_unsupported_is_loud():
    """Graphs the device compiler cannot lower are rejected before any device work."""
    g = cf.Graph()
    x = g.placeholder("x", cf.F32, (2, 2))
    y = g.op1("Transpose", [x])
    with pytest.raises(cf.CfError) as e:
        cf.Session(g, [y])
    assert e.value.code in ("CF_E_UNSUPPORTED", "CF_E_CUDA")


def test_send_recv_graph_errors_and_channels_api():
    g = cf.Graph()
    x = g.placeholder("x", cf.F32, (2, 2))
    f = g.placeholder("f", cf.F32, ())
    with pytest.raises(cf.CfError) as e:
        g.send(x, f, 0, 1)          # index must be an int64 scalar
    assert e.value.code == "CF_E_DTYPE"
    i = g.const(0, cf.I64)
    with pytest.raises(cf.CfError) as e:
        g.op("Recv", [i], {"dtype": cf.F32, "shape": [2, 2]})   # no channel / peer
    assert e.value.code == "CF_E_ARITY"
    r = g.recv(i, 3, 1, cf.F32, (2, 2))
    assert r.shape == (2, 2)
    assert g.count_ops()["Recv"] == 1
