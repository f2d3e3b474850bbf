"""The north-star workload built with the oracle's own builder (test infrastructure only).

``dynamic_rnn`` "is based on our work" and is "while-loops and TensorArray objects"
(PAPER.md:410-411, 1310-1313); the LSTM experiments use it. The paper does
not spell out its variable-length semantics, so DESIGN.md reading R10 fixes TF's: the loop runs
``t < T`` (padded length); inside the body ``cond(t < max_len, cell_branch, empty_update)`` and,
in the cell branch, ``cond(t < min_len, cells, masked_cells)``; finished rows (t >= len_b) copy
their state through and emit zeros. The loss is the random projection of reading R11:
``y = sum(R_out * out_top) + sum_l (sum(R_h[l] * h_T[l]) + sum(R_c[l] * c_T[l]))``.

The optional MoE-style gated branch (BASELINE.json configs[4]) adds after every layer
``y_l = out_l + cond(route[t, l], act(out_l @ WA_l), act(out_l @ WB_l))`` with seeded, exact
route bits (reading R12); act = relu (default) or tanh (``moe_act="tanh"``, reading R21: the
bf16 parity workload, whose expert has no float-decided mask).
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List

import numpy as np

from .autodiff import gradients
from .graph import BOOL, FLOAT, INT, Builder, T


@dataclasses.dataclass
class RNNProgram:
    b: Builder
    fetch: Dict[str, T]
    grads: Dict[str, T]
    T: int
    B: int
    I: int
    H: int
    L: int


def layer_partition(L: int, world: int, rank: int):
    """Layers of pipeline stage `rank` (contiguous, balanced; reading R18 of DESIGN.md)."""
    if not 1 <= world <= L:
        raise ValueError(f"cannot split {L} layers over {world} stages")
    base, extra = divmod(L, world)
    l0 = rank * base + min(rank, extra)
    return l0, l0 + base + (1 if rank < extra else 0)


def dynamic_rnn_lstm(T_: int, B: int, I: int, H: int, L: int = 1, parallel_iterations: int = 32,
                     length_conds: bool = True, moe: bool = False, forget_bias: float = 0.0,
                     with_grads: bool = True, stage=None, moe_act: str = "relu") -> RNNProgram:
    """The full model, or with ``stage=(rank, world)`` the partition of pipeline stage `rank`
    (layers ``layer_partition(L, world, rank)``): the layer input of a later stage is a Recv of
    the previous stage's top output and a non-final stage Sends its top output on, inside the
    loop at every iteration (§4.4). Each stage keeps its
    own copy of the loop control: the loop and cond predicates depend only on the counter and
    the fed lengths, so every partition computes them itself (reading R18). The stage loss is
    the part of y owned by the stage; the stage losses sum to the full model's y."""
    rank, world = stage if stage is not None else (0, 1)
    act = {"relu": "Relu", "tanh": "Tanh"}[moe_act]   # expert activation (reading R21)
    l0, l1 = layer_partition(L, world, rank)
    first, last = rank == 0, rank == world - 1
    Ls = list(range(l0, l1))
    n = len(Ls)
    b = Builder()
    x = b.placeholder("x", FLOAT, (T_, B, I)) if first else None
    lens = b.placeholder("len", INT, (B,))
    Ws, bs, h0, c0, WA, WB = {}, {}, {}, {}, {}, {}
    for l in Ls:
        il = I if l == 0 else H
        Ws[l] = b.placeholder(f"W{l}", FLOAT, (4 * H, il + H))
        bs[l] = b.placeholder(f"b{l}", FLOAT, (4 * H,))
        h0[l] = b.placeholder(f"h0_{l}", FLOAT, (B, H))
        c0[l] = b.placeholder(f"c0_{l}", FLOAT, (B, H))
        if moe:
            WA[l] = b.placeholder(f"WA{l}", FLOAT, (H, H))
            WB[l] = b.placeholder(f"WB{l}", FLOAT, (H, H))
    route_ta = None
    if moe:
        route = b.placeholder("route", BOOL, (T_, L))
        route_ta = b.tensor_array(T_, BOOL, (L,)).unstack(route)
    x_ta = b.tensor_array(T_, FLOAT, (B, I)).unstack(x) if first else None
    out_tas = [b.tensor_array(T_, FLOAT, (B, H)) for _ in Ls]
    max_len = b.op1("ReduceMax", [lens])
    min_len = b.op1("ReduceMin", [lens])
    t_bound = b.const(T_, INT)

    def pred(t, *rest):
        return b.less(t, t_bound)

    def body(t, *vs):
        hs, cs, flows = vs[:n], vs[n:2 * n], vs[2 * n:3 * n]
        x_t = x_ta.read(t) if first else b.recv(t, rank - 1, rank - 1, FLOAT, (B, H))
        r_t = route_ta.read(t) if moe else None

        def cells(masked):
            inp, outs, nh, nc = x_t, [], [], []
            for k, l in enumerate(Ls):
                ins = [inp, hs[k], cs[k], Ws[l], bs[l]] + ([t, lens] if masked else [])
                hn, cn, o, _g = b.op("LSTMCell", ins, {"masked": masked, "forget_bias": forget_bias})
                if moe:
                    r = b.op1("Reshape", [b.op1("Slice", [r_t], {"begin": (l,), "size": (1,)})],
                              {"shape": ()})
                    oo = o
                    e = b.cond(r, lambda: [b.op1(act, [b.matmul(oo, WA[l])])],
                               lambda: [b.op1(act, [b.matmul(oo, WB[l])])])[0]
                    o = b.add(o, e)
                outs.append(o)
                nh.append(hn)
                nc.append(cn)
                inp = o
            return outs + nh + nc

        if length_conds:
            def cell_branch():
                return b.cond(b.less(t, min_len), lambda: cells(False), lambda: cells(True))

            def empty_update():
                return [b.zeros((B, H)) for _ in Ls] + list(hs) + list(cs)
            res = b.cond(b.less(t, max_len), cell_branch, empty_update)
        else:
            res = cells(True)
        outs, nh, nc = res[:n], res[n:2 * n], res[2 * n:]
        if not last:
            b.send(outs[-1], t, rank, rank + 1)
        nf = [out_tas[k].with_flow(flows[k]).write(t, outs[k]).flow for k in range(n)]
        return [b.add(t, b.const(1, INT))] + nh + nc + nf

    res = b.while_loop(pred, body, [b.const(0, INT)] + [h0[l] for l in Ls] + [c0[l] for l in Ls]
                       + [ta.flow for ta in out_tas], parallel_iterations, name="rnn")
    hT, cT, fT = res[1:1 + n], res[1 + n:1 + 2 * n], res[1 + 2 * n:]
    y = None
    fetch = {}
    if last:
        out_top = out_tas[n - 1].with_flow(fT[n - 1]).stack()
        R_out = b.placeholder("R_out", FLOAT, (T_, B, H))
        y = b.reduce_sum(b.mul(R_out, out_top))
        fetch["out"] = out_top
    for k, l in enumerate(Ls):
        Rh = b.placeholder(f"R_h{l}", FLOAT, (B, H))
        Rc = b.placeholder(f"R_c{l}", FLOAT, (B, H))
        yl = b.add(b.reduce_sum(b.mul(Rh, hT[k])), b.reduce_sum(b.mul(Rc, cT[k])))
        y = yl if y is None else b.add(y, yl)
    fetch = {"y": y, **fetch}
    for k, l in enumerate(Ls):
        fetch[f"hT{l}"] = hT[k]
        fetch[f"cT{l}"] = cT[k]
    grads = {}
    if with_grads:
        names, xs = (["x"], [x]) if first else ([], [])
        for l in Ls:
            names += [f"W{l}", f"b{l}", f"h0_{l}", f"c0_{l}"]
            xs += [Ws[l], bs[l], h0[l], c0[l]]
            if moe:
                names += [f"WA{l}", f"WB{l}"]
                xs += [WA[l], WB[l]]
        for nm, gt in zip(names, gradients(b, y, xs)):
            grads["d" + nm] = gt
    return RNNProgram(b, fetch, grads, T_, B, I, H, L)


def run_program(p: RNNProgram, feeds: Dict[str, np.ndarray], K=None, sched_seed=None,
                return_trace=False, transport=None):
    """Run the program in the fp64 interpreter; every value stays float64 (the bf16 parity
    tests feed bf16-rounded inputs, reading R16)."""
    from . import interp
    names = list(p.fetch) + list(p.grads)
    tensors = [p.fetch[n] for n in p.fetch] + [p.grads[n] for n in p.grads]
    feeds = {k: v for k, v in feeds.items() if k in p.b.g.placeholders}
    r = interp.run(p.b.g, feeds, tensors, K_override=K, sched_seed=sched_seed,
                   return_trace=return_trace, transport=transport)
    vals, tr = (r if return_trace else (r, None))
    out = dict(zip(names, vals))
    return (out, tr) if return_trace else out


def run_pipeline_threads(T_, B, I, H, L, world, feeds, K=None, sched_seed=None, **kw):
    """All stages of the layer pipeline in one process, one thread per stage, Send/Recv through
    an in-process mailbox (test helper). Returns per-stage (results, trace)."""
    import threading

    from .transport import Mailbox
    mb = Mailbox()
    res = [None] * world
    errs = []

    def work(r):
        try:
            p = dynamic_rnn_lstm(T_, B, I, H, L, stage=(r, world), **kw)
            res[r] = run_program(p, feeds, K=K, sched_seed=sched_seed, return_trace=True,
                                 transport=mb.port(r))
        except Exception as e:  # noqa: BLE001 -- surfaced to the caller below
            errs.append(e)
    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return res


def ponder_rnn(T_: int, B: int, D: int, K: int = 32) -> RNNProgram:
    """A while_loop nested in a while_loop (the adaptive-
    computation RNN shape): for every step t the state takes x[t] and then ponders n[t] times,
    ``a = tanh(a W + c)``; n[t] is fed (ragged inner trip counts). Loss sum(R * a_T)."""
    b = Builder()
    x = b.placeholder("x", FLOAT, (T_, B, D))
    n = b.placeholder("n", INT, (T_,))
    W = b.placeholder("W", FLOAT, (D, D))
    c = b.placeholder("c", FLOAT, (B, D))
    a0 = b.placeholder("a0", FLOAT, (B, D))
    R = b.placeholder("R", FLOAT, (B, D))
    x_ta = b.tensor_array(T_, FLOAT, (B, D)).unstack(x)
    n_ta = b.tensor_array(T_, INT, ()).unstack(n)
    t_bound = b.const(T_, INT)

    def step(t, a):
        a = b.add(a, x_ta.read(t))
        m = n_ta.read(t)
        r = b.while_loop(lambda k, s: b.less(k, m),
                         lambda k, s: [b.add(k, b.const(1, INT)),
                                       b.op1("Tanh", [b.add(b.matmul(s, W), c)])],
                         [b.const(0, INT), a], parallel_iterations=K, name="ponder")
        return [b.add(t, b.const(1, INT)), r[1]]
    res = b.while_loop(lambda t, a: b.less(t, t_bound), step, [b.const(0, INT), a0],
                       parallel_iterations=K, name="steps")
    y = b.reduce_sum(b.mul(R, res[1]))
    names = ["x", "W", "c", "a0"]
    grads = {"d" + k: gt for k, gt in zip(names, gradients(b, y, [x, W, c, a0]))}
    return RNNProgram(b, {"y": y, "aT": res[1]}, grads, T_, B, D, D, 1)
