"""dynamic_rnn LSTM built on the C-ABI ("We implemented the dynamic_rnn
operator in TensorFlow using while-loops and TensorArray objects").

Variable-length semantics (reading R10, TF dynamic_rnn): the loop runs t < T;
the body is ``cond(t < max_len, cell_branch, empty_update)`` and inside the cell branch
``cond(t < min_len, cells, masked_cells)``; a finished row keeps its state and emits zeros.
The loss is the random projection of reading R11. The optional MoE-style gated branch
(BASELINE.json configs[4]) adds ``y_l = out_l + cond(route[t, l], relu(out_l WA_l),
relu(out_l WB_l))`` after every layer.

Graph structure is the same as the oracle's builder produces for the same program
(tests/test_structure.py compares op counts), so the device's control trace can be compared
with the oracle's bit for bit.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List

from . import cf
from .cf import BOOL, F32, I64, Graph, Tensor


@dataclasses.dataclass
class RNNProgram:
    g: Graph
    fetch: Dict[str, Tensor]
    grads: Dict[str, Tensor]
    T: int
    B: int
    I: int
    H: int
    L: int

    def fetch_names(self) -> List[str]:
        return list(self.fetch) + list(self.grads)

    def fetch_tensors(self) -> List[Tensor]:
        return [self.fetch[n] for n in self.fetch] + [self.grads[n] for n in self.grads]


def layer_partition(L: int, world: int, rank: int):
    """Layers [l0, l1) of pipeline stage `rank`: contiguous, balanced (reading R18)."""
    if not 1 <= world <= L:
        raise ValueError(f"cannot split {L} layers over {world} stages")
    base, extra = divmod(L, world)
    l0 = rank * base + min(rank, extra)
    return l0, l0 + base + (1 if rank < extra else 0)


def dynamic_rnn_lstm(T: int, B: int, I: int, H: int, L: int = 1, parallel_iterations: int = 32,
                     length_conds: bool = True, moe: bool = False, forget_bias: float = 0.0,
                     with_grads: bool = True, stage=None, moe_act: str = "relu", dp=None) -> RNNProgram:
    """The full model, or with ``stage=(rank, world)`` the partition of layer-pipeline stage
    `rank`: a later stage Recvs its layer input from
    the previous stage and a non-final stage Sends its top output on, inside the loop, every
    iteration; each stage runs its own copy of the loop control (reading R18). The stage loss
    is the part of y owned by the stage (the stage losses sum to y)."""
    rank, world = stage if stage is not None else (0, 1)
    act = {"relu": "Relu", "tanh": "Tanh"}[moe_act]   # expert activation (reading R21)
    l0, l1 = layer_partition(L, world, rank)
    first, last = rank == 0, rank == world - 1
    Ls = list(range(l0, l1))
    n = len(Ls)
    g = Graph()
    x = g.placeholder("x", F32, (T, B, I)) if first else None
    lens = g.placeholder("len", I64, (B,))
    Ws, bs, h0, c0, WA, WB = {}, {}, {}, {}, {}, {}
    for l in Ls:
        il = I if l == 0 else H
        Ws[l] = g.placeholder(f"W{l}", F32, (4 * H, il + H))
        bs[l] = g.placeholder(f"b{l}", F32, (4 * H,))
        h0[l] = g.placeholder(f"h0_{l}", F32, (B, H))
        c0[l] = g.placeholder(f"c0_{l}", F32, (B, H))
        if moe:
            WA[l] = g.placeholder(f"WA{l}", F32, (H, H))
            WB[l] = g.placeholder(f"WB{l}", F32, (H, H))
    route_ta = None
    if moe:
        route = g.placeholder("route", BOOL, (T, L))
        route_ta = g.tensor_array(T, BOOL, (L,)).unstack(route)
    x_ta = g.tensor_array(T, F32, (B, I)).unstack(x) if first else None
    out_tas = [g.tensor_array(T, F32, (B, H)) for _ in Ls]
    max_len = g.op1("ReduceMax", [lens])
    min_len = g.op1("ReduceMin", [lens])
    t_bound = g.const(T, I64)

    def pred(t, *rest):
        return g.op1("Less", [t, t_bound])

    def body(t, *vs):
        hs, cs, flows = vs[:n], vs[n:2 * n], vs[2 * n:3 * n]
        x_t = x_ta.read(t) if first else g.recv(t, rank - 1, rank - 1, F32, (B, H))
        r_t = route_ta.read(t) if moe else None

        def cells(masked):
            inp, outs, nh, nc = x_t, [], [], []
            for k, l in enumerate(Ls):
                ins = [inp, hs[k], cs[k], Ws[l], bs[l]] + ([t, lens] if masked else [])
                hn, cn, o, _g = g.op("LSTMCell", ins, {"masked": masked, "forget_bias": forget_bias})
                if moe:
                    r = g.op1("Reshape", [g.op1("Slice", [r_t], {"begin": (l,), "size": (1,)})],
                              {"shape": ()})
                    oo, wa, wb = o, WA[l], WB[l]
                    e = g.cond(r, lambda: [g.op1(act, [g.op1("MatMul", [oo, wa])])],
                               lambda: [g.op1(act, [g.op1("MatMul", [oo, wb])])], 1)[0]
                    o = g.op1("Add", [o, e])
                outs.append(o)
                nh.append(hn)
                nc.append(cn)
                inp = o
            return outs + nh + nc

        if length_conds:
            def cell_branch():
                return g.cond(g.op1("Less", [t, min_len]), lambda: cells(False),
                              lambda: cells(True), 3 * n)

            def empty_update():
                return [g.const([[0.0] * H] * B, F32) for _ in Ls] + list(hs) + list(cs)
            res = g.cond(g.op1("Less", [t, max_len]), cell_branch, empty_update, 3 * n)
        else:
            res = cells(True)
        outs, nh, nc = res[:n], res[n:2 * n], res[2 * n:]
        if not last:
            g.send(outs[-1], t, rank, rank + 1)
        nf = [out_tas[k].with_flow(flows[k]).write(t, outs[k]).flow for k in range(n)]
        return [g.op1("Add", [t, g.const(1, I64)])] + nh + nc + nf

    res = g.while_loop(pred, body, [g.const(0, I64)] + [h0[l] for l in Ls] + [c0[l] for l in Ls]
                       + [ta.flow for ta in out_tas], parallel_iterations, name="rnn")
    hT, cT, fT = res[1:1 + n], res[1 + n:1 + 2 * n], res[1 + 2 * n:]
    y = None
    fetch = {}
    if last:
        out_top = out_tas[n - 1].with_flow(fT[n - 1]).stack()
        R_out = g.placeholder("R_out", F32, (T, B, H))
        y = g.op1("ReduceSum", [g.op1("Mul", [R_out, out_top])])
        fetch["out"] = out_top
    for k, l in enumerate(Ls):
        Rh = g.placeholder(f"R_h{l}", F32, (B, H))
        Rc = g.placeholder(f"R_c{l}", F32, (B, H))
        yl = g.op1("Add", [g.op1("ReduceSum", [g.op1("Mul", [Rh, hT[k]])]),
                           g.op1("ReduceSum", [g.op1("Mul", [Rc, cT[k]])])])
        y = yl if y is None else g.op1("Add", [y, yl])
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
        for nm, gt in zip(names, g.gradients(y, xs)):
            grads["d" + nm] = gt
        if dp is not None and dp[1] > 1:
            grads = _allreduce_weight_grads(g, grads, *dp)
    return RNNProgram(g, fetch, grads, T, B, I, H, L)


def _allreduce_weight_grads(g: Graph, grads: Dict[str, Tensor], rank: int, world: int):
    """Batch data parallelism: every rank runs the whole model on its own
    batch shard; the weight gradients (W, b and the experts') are summed over the ranks. The
    loss is a sum over samples, so the sum of the shards' gradients is the full batch's.
    In-graph, at the root: each rank Sends its gradient to every other rank (NVLink peer
    stores, PAPER.md:780-829 Send/Recv) and adds what it receives (AddN). The Send of a layer's
    gradient depends only on that layer's last dW chunk, so the exchange of the upper layers
    (whose backward finishes first) overlaps the lower layers' backward. Channel id =
    (tensor * world + sender) * world + receiver."""
    zero = g.const(0, I64)
    out = dict(grads)
    k = 0
    for nm, gt in grads.items():
        if not nm.startswith(("dW", "db", "dWA", "dWB")):
            continue   # dx, dh0, dc0 are per-sample: nothing to sum
        peers = [p for p in range(world) if p != rank]
        for p in peers:
            g.send(gt, zero, (k * world + rank) * world + p, p)
        terms = [gt] + [g.recv(zero, (k * world + p) * world + rank, p, gt.dtype, gt.shape)
                        for p in peers]
        out[nm] = g.op1("AddN", terms)
        k += 1
    return out


def feeds_to_device(feeds, device="cuda", session=None):
    """numpy feeds (synth.rnn_inputs) -> contiguous CUDA tensors in the session's feed dtypes
    (bf16 for the LSTM GEMM operands on the CF_BF16 path, fp32 / int64 / bool otherwise)."""
    import numpy as np
    import torch
    tdt = {cf.F32: torch.float32, cf.BF16: torch.bfloat16}
    out = {}
    for k, v in feeds.items():
        if session is not None and not session.has_feed(k):
            continue   # e.g. a pipeline stage without this placeholder
        v = np.asarray(v)
        if v.dtype == np.float64:
            dt = torch.float32
            if session is not None:
                dt = tdt.get(session.feed_dtype(k), torch.float32)
            out[k] = torch.from_numpy(v).to(device=device, dtype=torch.float32).to(dt).contiguous()
        elif v.dtype == np.bool_:
            out[k] = torch.from_numpy(v).to(device=device).contiguous()
        else:
            out[k] = torch.from_numpy(v.astype(np.int64)).to(device=device).contiguous()
    return out


def static_rnn_lstm(T: int, B: int, I: int, H: int, L: int = 1, forget_bias: float = 0.0,
                    with_grads: bool = True) -> RNNProgram:
    """The same LSTM statically unrolled: no while_loop, no cond, T x L LSTMCell nodes in the
    root context (§6.3 "Static vs. Dynamic": the paper
    compares dynamic_rnn with a statically unrolled graph). Full-length sequences only. The loss
    and the fetches are the dynamic program's (reading R11), so the two are checked against
    each other value by value."""
    g = Graph()
    x = g.placeholder("x", F32, (T, B, I))
    Ws, bs, hs, cs = {}, {}, [], []
    for l in range(L):
        il = I if l == 0 else H
        Ws[l] = g.placeholder(f"W{l}", F32, (4 * H, il + H))
        bs[l] = g.placeholder(f"b{l}", F32, (4 * H,))
        hs.append(g.placeholder(f"h0_{l}", F32, (B, H)))
        cs.append(g.placeholder(f"c0_{l}", F32, (B, H)))
    h0 = list(hs)
    c0 = list(cs)
    x_ta = g.tensor_array(T, F32, (B, I)).unstack(x)
    out_ta = g.tensor_array(T, F32, (B, H))
    for t in range(T):
        inp = x_ta.read(g.const(t, I64))
        for l in range(L):
            hn, cn, o, _g = g.op("LSTMCell", [inp, hs[l], cs[l], Ws[l], bs[l]],
                                 {"masked": False, "forget_bias": forget_bias})
            hs[l], cs[l], inp = hn, cn, o
        out_ta = out_ta.write(g.const(t, I64), inp)
    out_top = out_ta.stack()
    R_out = g.placeholder("R_out", F32, (T, B, H))
    y = g.op1("ReduceSum", [g.op1("Mul", [R_out, out_top])])
    fetch = {}
    for l in range(L):
        Rh = g.placeholder(f"R_h{l}", F32, (B, H))
        Rc = g.placeholder(f"R_c{l}", F32, (B, H))
        y = g.op1("Add", [y, g.op1("Add", [g.op1("ReduceSum", [g.op1("Mul", [Rh, hs[l]])]),
                                           g.op1("ReduceSum", [g.op1("Mul", [Rc, cs[l]])])])])
    fetch = {"y": y, "out": out_top}
    for l in range(L):
        fetch[f"hT{l}"] = hs[l]
        fetch[f"cT{l}"] = cs[l]
    grads = {}
    if with_grads:
        names, xs = ["x"], [x]
        for l in range(L):
            names += [f"W{l}", f"b{l}", f"h0_{l}", f"c0_{l}"]
            xs += [Ws[l], bs[l], h0[l], c0[l]]
        for nm, gt in zip(names, g.gradients(y, xs)):
            grads["d" + nm] = gt
    return RNNProgram(g, fetch, grads, T, B, I, H, L)


def ponder_rnn(T: int, B: int, D: int, K: int = 32) -> RNNProgram:
    """A while_loop nested in a while_loop (the adaptive-
    computation RNN shape) through the C-ABI: for every step t the state takes x[t] and then
    ponders n[t] times, ``a = tanh(a W + c)``; n[t] is fed (ragged inner trip counts). The
    device runs the inner loop as a nested frame of the outer body and differentiates it with
    nested gradient loops whose stacks are created once per outer iteration (their handles
    saved on a stack of the outer loop). Loss sum(R * a_T)."""
    g = Graph()
    x = g.placeholder("x", F32, (T, B, D))
    n = g.placeholder("n", I64, (T,))
    W = g.placeholder("W", F32, (D, D))
    c = g.placeholder("c", F32, (B, D))
    a0 = g.placeholder("a0", F32, (B, D))
    R = g.placeholder("R", F32, (B, D))
    x_ta = g.tensor_array(T, F32, (B, D)).unstack(x)
    n_ta = g.tensor_array(T, I64, ()).unstack(n)
    t_bound = g.const(T, I64)

    def step(t, a):
        a = g.op1("Add", [a, x_ta.read(t)])
        m = n_ta.read(t)
        r = g.while_loop(lambda k, s: g.op1("Less", [k, m]),
                         lambda k, s: [g.op1("Add", [k, g.const(1, I64)]),
                                       g.op1("Tanh", [g.op1("Add", [g.op1("MatMul", [s, W]), c])])],
                         [g.const(0, I64), a], K, name="ponder")
        return [g.op1("Add", [t, g.const(1, I64)]), r[1]]
    res = g.while_loop(lambda t, a: g.op1("Less", [t, t_bound]), step, [g.const(0, I64), a0], K,
                       name="steps")
    y = g.op1("ReduceSum", [g.op1("Mul", [R, res[1]])])
    names = ["x", "W", "c", "a0"]
    grads = {"d" + k: gt for k, gt in zip(names, g.gradients(y, [x, W, c, a0]))}
    return RNNProgram(g, {"y": y, "aT": res[1]}, grads, T, B, D, D, 1)
