"""Pins for the oracle's control-flow core (CPU only).

Each test checks the oracle against something other than itself: the evaluation-rule table
of PAPER.md:712-735, the closed forms of the paper's loop example, the scan
definition, static unrolling, and invariants the paper
fixes (at most once per frame PAPER.md:584; the window of PAPER.md:757-764; push/pop counts).
"""
import json
import os

import numpy as np
import pytest

from oracle import interp
from oracle.autodiff import gradients
from oracle.graph import BOOL, FLOAT, INT, Builder, GraphError, T, validate

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------------------ rules
def _dead_or_live(b, x, dead):
    """A tensor that is live, or dead via the untaken port of a root Switch."""
    p = b.const(True)
    sw = b._add("Switch", [x, p])
    return T(sw.id, 0 if dead else 1)


@pytest.mark.parametrize("case", gold("eval_rules.json")["switch"])
def test_switch_rule(case):
    b = Builder()
    d = _dead_or_live(b, b.const([5.0]), case["d_dead"])
    p = b.const(case["p"])
    sw = b._add("Switch", [d, p])
    vals = interp.run(b.g, {}, [T(sw.id, 0), T(sw.id, 1)])
    assert (vals[0] is interp.DEAD) == case["false_dead"]
    assert (vals[1] is interp.DEAD) == case["true_dead"]
    for v, dead in zip(vals, (case["false_dead"], case["true_dead"])):
        if not dead:
            assert v.tolist() == [5.0]


@pytest.mark.parametrize("case", gold("eval_rules.json")["op"])
def test_op_dead_propagation(case):
    b = Builder()
    a = _dead_or_live(b, b.const(2.0), case["a_dead"])
    c = _dead_or_live(b, b.const(3.0), case["b_dead"])
    s = b._add("Add", [a, c])
    (v,) = interp.run(b.g, {}, [T(s.id, 0)])
    assert (v is interp.DEAD) == case["out_dead"]
    if not case["out_dead"]:
        assert float(v) == 5.0


@pytest.mark.parametrize("d1_dead,d2_dead", [(False, True), (True, False), (True, True)])
def test_merge_rule(d1_dead, d2_dead):
    b = Builder()
    d1 = _dead_or_live(b, b.const(1.0), d1_dead)
    d2 = _dead_or_live(b, b.const(2.0), d2_dead)
    m = b._add("Merge", [d1, d2], {"cond_id": -1})
    (v,) = interp.run(b.g, {}, [T(m.id, 0)])
    if d1_dead and d2_dead:
        assert v is interp.DEAD
    else:       # r = if is_dead(d1) then d2 else d1
        assert float(v) == (2.0 if d1_dead else 1.0)


def test_enter_nextiteration_exit_tags():
    """Enter -> tag/name/0, NextIteration -> tag/name/(n+1), Exit -> parent tag."""
    b = Builder()
    n3 = b.const(3, INT)
    res = b.while_loop(lambda i: b.less(i, n3), lambda i: [b.add(i, b.const(1, INT))],
                       [b.const(0, INT)], name="L")
    # push the loop variable each iteration to observe the tags it carries
    ctx = b.g.whiles["L"]
    h = b.op1("StackCreate", [], {"frame": "L", "dtype": INT, "elem_shape": ()})
    with b.in_ctx(ctx):
        b.op("StackPush", [h, T(ctx.loop_vars[1]["switch"], 1)])
    (v,), tr = interp.run(b.g, {}, [res[0]], return_trace=True)
    assert int(v) == 3
    assert [tag for _, tag in tr.push_log] == [(("L", 0),), (("L", 1),), (("L", 2),)]
    assert tr.trip_counts == {((), "L"): 3}


# ------------------------------------------------------------------------------ loops
def _loop_1x1(n, K=32):
    b = Builder()
    nn = b.const(n, INT)
    x = b.placeholder("x", FLOAT, (1, 1))
    w = b.placeholder("w", FLOAT, (1, 1))
    _, a = b.while_loop(lambda i, a: b.less(i, nn),
                        lambda i, a: (b.add(i, b.const(1, INT)), b.matmul(a, w)),
                        [b.const(0, INT), x], parallel_iterations=K)
    y = b.reduce_sum(a)
    gw, gx = gradients(b, y, [w, x])
    return b, a, y, gw, gx


def test_paper_loop_example_closed_form():
    G = gold("loop_1x1.json")
    b, a, y, gw, gx = _loop_1x1(G["n"])
    assert validate(b.g) == []
    (av, yv, gwv, gxv), tr = interp.run(b.g, {"x": [[G["x"]]], "w": [[G["w"]]]},
                                        [a, y, gw, gx], return_trace=True)
    assert float(av[0, 0]) == G["a"] and float(yv) == G["a"]
    assert float(gwv[0, 0]) == G["dy_dw"] and float(gxv[0, 0]) == G["dy_dx"]
    assert len(tr.pushes) == G["stacks"]
    assert list(tr.pushes.values()) == [G["pushes"]] and list(tr.pops.values()) == [G["pops"]]


@pytest.mark.parametrize("n", range(0, 9))
def test_loop_matches_static_unrolling(n):
    """Loop gradient == MatMulGrad applied to the statically unrolled chain (Fig. 'Computing
    the gradient of a loop by unrolling'), for random 3x3 x, w."""
    rng = np.random.default_rng(n)
    b = Builder()
    nn = b.const(n, INT)
    x = b.placeholder("x", FLOAT, (3, 3))
    w = b.placeholder("w", FLOAT, (3, 3))
    _, a = b.while_loop(lambda i, a: b.less(i, nn),
                        lambda i, a: (b.add(i, b.const(1, INT)), b.matmul(a, w)),
                        [b.const(0, INT), x])
    y = b.reduce_sum(a)
    gw, gx = gradients(b, y, [w, x])
    xv, wv = rng.uniform(0.5, 1.5, (3, 3)), rng.uniform(0.5, 1.5, (3, 3))
    av, gwv, gxv = interp.run(b.g, {"x": xv, "w": wv}, [a, gw, gx])
    # hand-unrolled (figure): a_{k+1} = a_k w; g_a_n = ones; g_w += a_k^T g_{a_{k+1}}
    acts = [xv]
    for _ in range(n):
        acts.append(acts[-1] @ wv)
    g = np.ones_like(xv)
    g_w = np.zeros_like(wv)
    for k in reversed(range(n)):
        g_w += acts[k].T @ g
        g = g @ wv.T
    np.testing.assert_allclose(av, acts[-1], rtol=1e-12)
    np.testing.assert_allclose(gwv, g_w, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(gxv, g, rtol=1e-12)


def test_zero_trip_loop():
    b, a, y, gw, gx = _loop_1x1(0)
    av, gwv, gxv = interp.run(b.g, {"x": [[2.0]], "w": [[3.0]]}, [a, gw, gx])
    assert av.item() == 2.0 and gwv.item() == 0.0 and gxv.item() == 1.0


@pytest.mark.parametrize("K", [1, 2, 8, 32])
def test_parallel_iterations_invariance_and_window(K):
    b, a, y, gw, gx = _loop_1x1(6, K=K)
    vals, tr = interp.run(b.g, {"x": [[0.9]], "w": [[1.1]]}, [a, gw, gx], sched_seed=K,
                          return_trace=True)
    ref = interp.run(b.g, {"x": [[0.9]], "w": [[1.1]]}, [a, gw, gx], K_override=1)
    for v, r in zip(vals, ref):
        assert np.array_equal(v, r)
    assert all(m <= K for m in tr.max_inflight.values())
    if K == 1:
        assert max(tr.max_inflight.values()) == 1


def test_counter_and_dead_fetch():
    b = Builder()
    n3 = b.const(3, INT)
    (i,) = b.while_loop(lambda i: b.less(i, n3), lambda i: [b.add(i, b.const(1, INT))],
                        [b.const(0, INT)])
    p = b.placeholder("p", BOOL, ())
    x = b.placeholder("x", FLOAT, ())
    sw = b._add("Switch", [x, p])
    m = b.cond(p, lambda: [b.add(x, b.const(1.0))], lambda: [b.mul(x, b.const(2.0))])
    vi, pre_true, merged = interp.run(b.g, {"p": False, "x": 3.0}, [i, T(sw.id, 1), m[0]])
    assert int(vi) == 3
    assert pre_true is interp.DEAD          # fetched untaken branch -> DeadMarker
    assert float(merged) == 6.0


def test_cond_one_switch_per_captured_tensor():
    """"we use one Switch for each external tensor"."""
    b = Builder()
    p = b.placeholder("p", BOOL, ())
    xs = [b.placeholder(f"x{k}", FLOAT, ()) for k in range(3)]
    before = b.g.count_ops().get("Switch", 0)
    b.cond(p, lambda: [b.add(b.add(xs[0], xs[1]), xs[2])], lambda: [xs[0]])
    assert b.g.count_ops()["Switch"] - before == 3 + 1
    assert b.g.count_ops()["Merge"] == 1


def test_while_structure_and_validate():
    b = Builder()
    n = b.const(4, INT)
    x = b.placeholder("x", FLOAT, (2,))
    w = b.placeholder("w", FLOAT, (2,))
    b.while_loop(lambda i, a: b.less(i, n), lambda i, a: (b.add(i, b.const(1, INT)), b.mul(a, w)),
                 [b.const(0, INT), x])
    c = b.g.count_ops()
    # 2 user loop vars + hidden counter -> 3 x (Enter, Merge, Switch, NextIteration, Exit)
    # plus one Enter(is_constant) for w (and for the bound n used in the predicate)
    assert c["Merge"] == 3 and c["Switch"] == 3 and c["NextIteration"] == 3 and c["Exit"] == 3
    assert c["Enter"] == 3 + 2
    assert validate(b.g) == []
    # removing a NextIteration leaves an illegal cycle
    ni = next(nd for nd in b.g.nodes if nd.op == "NextIteration")
    ni.op = "Identity"
    assert any("cycle" in e for e in validate(b.g))


def test_errors():
    b = Builder()
    x = b.placeholder("x", FLOAT, ())
    with pytest.raises(GraphError) as e:
        b.cond(x, lambda: [x], lambda: [x])
    assert e.value.code == "CF_E_NONBOOL_PRED"
    p = b.placeholder("p", BOOL, ())
    with pytest.raises(GraphError) as e:
        b.cond(p, lambda: [x, x], lambda: [x])
    assert e.value.code == "CF_E_BRANCH_MISMATCH"
    with pytest.raises(GraphError) as e:
        gradients(b, b.placeholder("v", FLOAT, (2,)), [x])
    assert e.value.code == "CF_E_NONSCALAR_OBJECTIVE"
    with pytest.raises(interp.InterpError) as e:
        interp.run(b.g, {}, [x])
    assert e.value.code == "CF_E_MISSING_FEED"


# ------------------------------------------------------------------------------ TensorArray
@pytest.mark.parametrize("case", gold("scan.json")["cases"])
def test_scan(case):
    b = Builder()
    el = np.asarray(case["elems"], dtype=np.float64)
    e = b.placeholder("e", FLOAT, el.shape)
    i0 = b.placeholder("i0", FLOAT, ())
    fn = {"add": b.add, "mul": b.mul}[case["fn"]]
    out = b.scan(fn, e, i0)
    (v,) = interp.run(b.g, {"e": el, "i0": float(case["init"])}, [out])
    assert v.shape == (len(case["out"]),)
    assert v.tolist() == [float(o) for o in case["out"]]


def test_tensor_array_double_write_and_multi_read_gradient():
    b = Builder()
    v = b.placeholder("v", FLOAT, ())
    ta = b.tensor_array(2, FLOAT, ())
    ta = ta.write(b.const(0, INT), v)
    with pytest.raises(interp.InterpError) as e:
        ta2 = ta.write(b.const(0, INT), v)
        interp.run(b.g, {"v": 1.0}, [ta2.flow])
    assert e.value.code == "CF_E_DOUBLE_WRITE"
    b = Builder()
    v = b.placeholder("v", FLOAT, ())
    ta = b.tensor_array(2, FLOAT, ()).write(b.const(0, INT), v)
    r1, r2 = ta.read(b.const(0, INT)), ta.read(b.const(0, INT))
    y = b.add(r1, r2)
    (gv,) = gradients(b, y, [v])
    # the grad TensorArray holds the sum of the partial gradients
    assert float(interp.run(b.g, {"v": 0.7}, [gv])[0]) == 2.0


def test_scan_gradient_finite_difference():
    b = Builder()
    e = b.placeholder("e", FLOAT, (4,))
    i0 = b.placeholder("i0", FLOAT, ())
    y = b.reduce_sum(b.scan(lambda a, x: b.mul(b.add(a, x), x), e, i0))
    ge, gi = gradients(b, y, [e, i0])
    rng = np.random.default_rng(3)
    ev, iv = rng.uniform(0.5, 1.5, 4), 0.8
    gev, giv = interp.run(b.g, {"e": ev, "i0": iv}, [ge, gi])
    f = lambda ee, ii: float(interp.run(b.g, {"e": ee, "i0": ii}, [y])[0])
    h = 1e-6
    fd = [(f(ev + h * np.eye(4)[k], iv) - f(ev - h * np.eye(4)[k], iv)) / (2 * h) for k in range(4)]
    np.testing.assert_allclose(gev, fd, rtol=1e-5)
    np.testing.assert_allclose(giv, (f(ev, iv + h) - f(ev, iv - h)) / (2 * h), rtol=1e-5)
