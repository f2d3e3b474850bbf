"""The north-star workload built with the oracle's own builder (test infrastructure only).

``dynamic_rnn`` "is based on our work" and is "while-loops and TensorArray objects"
(PAPER.md:410-411, 1310-1313); the LSTM experiments use it. The paper does
not spell out its variable-length semantics, so DESIGN.md reading R10 fixes TF's: the loop runs
``t < T`` (padded length); inside the body ``cond(t < max_len, cell_branch, empty_update)`` and,
in the cell branch, ``cond(t < min_len, cells, masked_cells)``; finished rows (t >= len_b) copy
their state through and emit zeros. The loss is the random projection of reading R11:
``y = sum(R_out * out_top) + sum_l (sum(R_h[l] * h_T[l]) + sum(R_c[l] * c_T[l]))``.

The optional MoE-style gated branch (BASELINE.json configs[4]) adds after every layer
``y_l = out_l + cond(route[t, l], relu(out_l @ WA_l), relu(out_l @ WB_l))`` with seeded, exact
route bits (reading R12).
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


def dynamic_rnn_lstm(T_: int, B: int, I: int, H: int, L: int = 1, parallel_iterations: int = 32,
                     length_conds: bool = True, moe: bool = False, forget_bias: float = 0.0,
                     with_grads: bool = True) -> RNNProgram:
    b = Builder()
    x = b.placeholder("x", FLOAT, (T_, B, I))
    lens = b.placeholder("len", INT, (B,))
    Ws, bs, h0, c0, WA, WB = [], [], [], [], [], []
    for l in range(L):
        il = I if l == 0 else H
        Ws.append(b.placeholder(f"W{l}", FLOAT, (4 * H, il + H)))
        bs.append(b.placeholder(f"b{l}", FLOAT, (4 * H,)))
        h0.append(b.placeholder(f"h0_{l}", FLOAT, (B, H)))
        c0.append(b.placeholder(f"c0_{l}", FLOAT, (B, H)))
        if moe:
            WA.append(b.placeholder(f"WA{l}", FLOAT, (H, H)))
            WB.append(b.placeholder(f"WB{l}", FLOAT, (H, H)))
    route_ta = None
    if moe:
        route = b.placeholder("route", BOOL, (T_, L))
        route_ta = b.tensor_array(T_, BOOL, (L,)).unstack(route)
    x_ta = b.tensor_array(T_, FLOAT, (B, I)).unstack(x)
    out_tas = [b.tensor_array(T_, FLOAT, (B, H)) for _ in range(L)]
    max_len = b.op1("ReduceMax", [lens])
    min_len = b.op1("ReduceMin", [lens])
    t_bound = b.const(T_, INT)

    def pred(t, *rest):
        return b.less(t, t_bound)

    def body(t, *vs):
        hs, cs, flows = vs[:L], vs[L:2 * L], vs[2 * L:3 * L]
        x_t = x_ta.read(t)
        r_t = route_ta.read(t) if moe else None

        def cells(masked):
            inp, outs, nh, nc = x_t, [], [], []
            for l in range(L):
                ins = [inp, hs[l], cs[l], Ws[l], bs[l]] + ([t, lens] if masked else [])
                hn, cn, o, _g = b.op("LSTMCell", ins, {"masked": masked, "forget_bias": forget_bias})
                if moe:
                    r = b.op1("Reshape", [b.op1("Slice", [r_t], {"begin": (l,), "size": (1,)})],
                              {"shape": ()})
                    oo = o
                    e = b.cond(r, lambda: [b.op1("Relu", [b.matmul(oo, WA[l])])],
                               lambda: [b.op1("Relu", [b.matmul(oo, WB[l])])])[0]
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
                return [b.zeros((B, H)) for _ in range(L)] + list(hs) + list(cs)
            res = b.cond(b.less(t, max_len), cell_branch, empty_update)
        else:
            res = cells(True)
        outs, nh, nc = res[:L], res[L:2 * L], res[2 * L:]
        nf = [out_tas[l].with_flow(flows[l]).write(t, outs[l]).flow for l in range(L)]
        return [b.add(t, b.const(1, INT))] + nh + nc + nf

    res = b.while_loop(pred, body, [b.const(0, INT)] + h0 + c0 + [ta.flow for ta in out_tas],
                       parallel_iterations, name="rnn")
    hT, cT, fT = res[1:1 + L], res[1 + L:1 + 2 * L], res[1 + 2 * L:]
    out_top = out_tas[L - 1].with_flow(fT[L - 1]).stack()
    R_out = b.placeholder("R_out", FLOAT, (T_, B, H))
    y = b.reduce_sum(b.mul(R_out, out_top))
    for l in range(L):
        Rh = b.placeholder(f"R_h{l}", FLOAT, (B, H))
        Rc = b.placeholder(f"R_c{l}", FLOAT, (B, H))
        y = b.add(y, b.add(b.reduce_sum(b.mul(Rh, hT[l])), b.reduce_sum(b.mul(Rc, cT[l]))))
    fetch = {"y": y, "out": out_top}
    for l in range(L):
        fetch[f"hT{l}"] = hT[l]
        fetch[f"cT{l}"] = cT[l]
    grads = {}
    if with_grads:
        names, xs = ["x"], [x]
        for l in range(L):
            names += [f"W{l}", f"b{l}", f"h0_{l}", f"c0_{l}"]
            xs += [Ws[l], bs[l], h0[l], c0[l]]
            if moe:
                names += [f"WA{l}", f"WB{l}"]
                xs += [WA[l], WB[l]]
        for nm, gt in zip(names, gradients(b, y, xs)):
            grads["d" + nm] = gt
    return RNNProgram(b, fetch, grads, T_, B, I, H, L)


def run_program(p: RNNProgram, feeds: Dict[str, np.ndarray], K=None, sched_seed=None,
                return_trace=False):
    from . import interp
    names = list(p.fetch) + list(p.grads)
    tensors = [p.fetch[n] for n in p.fetch] + [p.grads[n] for n in p.grads]
    r = interp.run(p.b.g, feeds, tensors, K_override=K, sched_seed=sched_seed,
                   return_trace=return_trace)
    vals, tr = (r if return_trace else (r, None))
    out = dict(zip(names, vals))
    return (out, tr) if return_trace else out
