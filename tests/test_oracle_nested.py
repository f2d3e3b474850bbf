"""CPU pins of a while_loop nested in a while_loop and its recursive gradient (SURVEY.md §8(f)
f2; "for nested loops, we apply our techniques recursively"):
the inner loop's saved values go on a stack created once per outer iteration, whose handle is
itself saved for the outer gradient loop. Pinned by closed forms (a scalar product loop, an
inner trip count that depends on the outer counter), by torch autograd of the statically
unrolled computation, and by the trace invariants, for parallel_iterations 1 / 2 / 32 and
shuffled schedules."""
import numpy as np
import pytest
import torch

from oracle import interp
from oracle.autodiff import gradients
from oracle.graph import FLOAT, INT, Builder


def _power_loop(n_out, inner_of_i, K):
    """a = x; for i < n_out: for j < inner(i): a = a * w. y = a."""
    b = Builder()
    x = b.placeholder("x", FLOAT, ())
    w = b.placeholder("w", FLOAT, ())
    nb = b.const(n_out, INT)

    def obody(i, a):
        m = inner_of_i(b, i)
        r = b.while_loop(lambda j, c: b.less(j, m),
                         lambda j, c: [b.add(j, b.const(1, INT)), b.mul(c, w)],
                         [b.const(0, INT), a], parallel_iterations=K, name="inner")
        return [b.add(i, b.const(1, INT)), r[1]]
    res = b.while_loop(lambda i, a: b.less(i, nb), obody, [b.const(0, INT), x],
                       parallel_iterations=K, name="outer")
    y = res[1]
    return b, y, gradients(b, y, [x, w])


@pytest.mark.parametrize("K", [1, 2, 32])
@pytest.mark.parametrize("seed", [None, 1, 2])
def test_nested_power_closed_form(K, seed):
    b, y, gs = _power_loop(3, lambda b, i: b.const(2, INT), K)
    x, w = 1.5, 1.25
    out, tr = interp.run(b.g, {"x": np.array(x), "w": np.array(w)}, [y] + gs, sched_seed=seed,
                         return_trace=True)
    n = 6
    assert abs(out[0] - x * w ** n) <= 1e-12 * abs(x * w ** n)
    assert abs(out[1] - w ** n) <= 1e-12 * w ** n
    assert abs(out[2] - n * x * w ** (n - 1)) <= 1e-12 * n * x * w ** (n - 1)
    assert sum(tr.pushes.values()) == sum(tr.pops.values())


@pytest.mark.parametrize("K", [1, 32])
def test_nested_inner_trip_count_depends_on_outer_counter(K):
    """inner(i) = i + 1: an ACT-style ragged inner loop; exponent sum_i (i + 1)."""
    n_out = 4
    b, y, gs = _power_loop(n_out, lambda b, i: b.add(i, b.const(1, INT)), K)
    x, w = 0.75, 1.1
    out, tr = interp.run(b.g, {"x": np.array(x), "w": np.array(w)}, [y] + gs, return_trace=True)
    n = sum(i + 1 for i in range(n_out))
    assert abs(out[0] - x * w ** n) <= 1e-12 * abs(x * w ** n)
    assert abs(out[2] - n * x * w ** (n - 1)) <= 1e-12 * abs(n * x * w ** (n - 1))
    # the inner forward frame ran once per outer iteration with i + 1 trips, plus once dead
    # (0 trips) in the outer loop's exiting iteration (reading R2: a dead frame's Exits fire
    # once, dead); its gradient frames replay the live counts
    inner = sorted(v for (pt, f), v in tr.trip_counts.items() if f == "inner")
    assert inner == [0, 1, 2, 3, 4]
    inner_g = sorted(v for (pt, f), v in tr.trip_counts.items() if f == "inner_grad")
    assert inner_g[-4:] == [1, 2, 3, 4] and all(v == 0 for v in inner_g[:-4]), inner_g
    assert sum(tr.exit_fires.values()) > 0


def test_nested_vector_recurrence_vs_torch_unrolled():
    """outer t < T: a = a + x[t]; inner k < 1 + t % 3: a = tanh(a W + c); loss sum(R * a)."""
    T, D = 5, 4
    rng = np.random.default_rng(3)
    xv, Wv, cv, Rv, a0 = (rng.standard_normal((T, 1, D)), rng.standard_normal((D, D)) * 0.5,
                          rng.standard_normal((1, D)), rng.standard_normal((1, D)),
                          rng.standard_normal((1, D)))
    b = Builder()
    x = b.placeholder("x", FLOAT, (T, 1, D))
    W = b.placeholder("W", FLOAT, (D, D))
    c = b.placeholder("c", FLOAT, (1, D))
    R = b.placeholder("R", FLOAT, (1, D))
    A0 = b.placeholder("a0", FLOAT, (1, D))
    xta = b.tensor_array(T, FLOAT, (1, D)).unstack(x)
    Tb = b.const(T, INT)

    def obody(t, a):
        a = b.add(a, xta.read(t))
        m = cnt_ta.read(t)   # inner trip count 1 + t % 3, from a table (a TensorArray)
        r = b.while_loop(lambda k, s: b.less(k, m),
                         lambda k, s: [b.add(k, b.const(1, INT)),
                                       b.op1("Tanh", [b.add(b.matmul(s, W), c)])],
                         [b.const(0, INT), a], name="ponder")
        return [b.add(t, b.const(1, INT)), r[1]]
    cnt_ta = b.tensor_array(T, INT, ()).unstack(b.const(np.array([1 + t % 3 for t in range(T)]), INT))
    res = b.while_loop(lambda t, a: b.less(t, Tb), obody, [b.const(0, INT), A0], name="steps")
    y = b.reduce_sum(b.mul(R, res[1]))
    gs = gradients(b, y, [x, W, c, A0])
    out = interp.run(b.g, {"x": xv, "W": Wv, "c": cv, "R": Rv, "a0": a0}, [y] + gs)
    tx, tW, tc, ta0 = (torch.tensor(v, requires_grad=True) for v in (xv, Wv, cv, a0))
    a = ta0
    for t in range(T):
        a = a + tx[t]
        for _ in range(1 + t % 3):
            a = torch.tanh(a @ tW + tc)
    ty = (torch.tensor(Rv) * a).sum()
    ty.backward()
    ref = [ty.item(), tx.grad.numpy(), tW.grad.numpy(), tc.grad.numpy(), ta0.grad.numpy()]
    for got, want in zip(out, ref):
        want = np.asarray(want)
        assert np.abs(np.asarray(got) - want).max() <= 1e-12 * max(1.0, np.abs(want).max())
