"""fp64 op kernels of the oracle (test infrastructure only; see oracle/__init__.py).

Every kernel is the plain mathematical definition in float64 numpy. The LSTM cell is not
written out in the paper, which only cites Hochreiter & Schmidhuber;
DESIGN.md reading R9 fixes the PyTorch convention: gate order i, f, g, o; pre-activation
``Z = [x, h] @ W.T + b`` with ``W = [W_ih | W_hh]`` of shape [4H, I+H]; sigma for i, f, o and
tanh for g; ``c' = f*c + i*g``; ``h' = o*tanh(c')``; no peepholes; optional ``forget_bias``
added to the f pre-activation.

Variable-length masking (reading R10, TF ``dynamic_rnn`` semantics): with
``live_b = t < len_b``, ``h_next = where(live, h', h)``, ``c_next = where(live, c', c)``,
``out = where(live, h', 0)``.

``lstm_cell_grad`` is the chain rule of ``lstm_cell`` written out; it is pinned against the
generic autodiff of the composite graph, against ``torch.nn.LSTM`` and against central finite
differences (tests/test_oracle_lstm.py).
"""
from __future__ import annotations

import numpy as np


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def lstm_cell(x, h, c, W, b, t=None, lens=None, forget_bias=0.0):
    """Returns (h_next, c_next, out, gates) with gates = post-activation [i, f, g, o]."""
    H = h.shape[1]
    z = np.concatenate([x, h], axis=1) @ W.T + b
    i = sigmoid(z[:, 0 * H:1 * H])
    f = sigmoid(z[:, 1 * H:2 * H] + forget_bias)
    g = np.tanh(z[:, 2 * H:3 * H])
    o = sigmoid(z[:, 3 * H:4 * H])
    c_new = f * c + i * g
    h_new = o * np.tanh(c_new)
    gates = np.concatenate([i, f, g, o], axis=1)
    if lens is None:
        return h_new, c_new, h_new.copy(), gates
    live = (t < np.asarray(lens))[:, None]
    return (np.where(live, h_new, h), np.where(live, c_new, c),
            np.where(live, h_new, 0.0), gates)


def lstm_cell_grad(x, h, c, W, gates, dh_next, dc_next, dout, t=None, lens=None):
    """Gradient of ``lstm_cell`` w.r.t. (x, h, c, W, b) given upstream grads of
    (h_next, c_next, out). Gates are the saved post-activation values."""
    H = h.shape[1]
    I = x.shape[1]
    i, f, g, o = (gates[:, k * H:(k + 1) * H] for k in range(4))
    c_new = f * c + i * g
    tc = np.tanh(c_new)
    dh = dh_next + dout                          # both outputs equal h' on live rows
    do = dh * tc
    dcn = dh * o * (1.0 - tc * tc) + dc_next
    di = dcn * g
    dg = dcn * i
    df = dcn * c
    dc = dcn * f
    dz = np.concatenate([di * i * (1.0 - i), df * f * (1.0 - f),
                         dg * (1.0 - g * g), do * o * (1.0 - o)], axis=1)
    if lens is not None:
        live = (t < np.asarray(lens))[:, None]
        dz = np.where(live, dz, 0.0)
        dc = np.where(live, dc, dc_next)         # c_next = c on finished rows
    dxh = dz @ W
    dx = dxh[:, :I]
    dhp = dxh[:, I:]
    if lens is not None:
        dhp = np.where(live, dhp, dh_next)       # h_next = h on finished rows
    dW = dz.T @ np.concatenate([x, h], axis=1)
    db = dz.sum(axis=0)
    return dx, dhp, dc, dW, db


def matmul(a, b, ta=False, tb=False):
    return (a.T if ta else a) @ (b.T if tb else b)


def eval_op(op: str, vals, attrs):
    """Pure kernels for non-control, non-resource ops; returns a list of outputs."""
    if op == "Identity" or op == "StopGradient":
        return [vals[0]]
    if op == "Const":
        return [np.array(attrs["value"], copy=True)]
    if op == "Add":
        return [vals[0] + vals[1]]
    if op == "AddN":
        out = vals[0]
        for v in vals[1:]:
            out = out + v
        return [out]
    if op == "Sub":
        return [vals[0] - vals[1]]
    if op == "Mul":
        return [vals[0] * vals[1]]
    if op == "Neg":
        return [-vals[0]]
    if op == "MatMul":
        return [matmul(vals[0], vals[1], attrs.get("ta", False), attrs.get("tb", False))]
    if op == "Transpose":
        return [np.ascontiguousarray(vals[0].T)]
    if op == "ReduceSum":
        if attrs.get("axis") == 0:
            return [vals[0].sum(axis=0)]
        return [np.asarray(vals[0].sum())]
    if op == "BiasAdd":
        return [vals[0] + vals[1][None, :]]
    if op == "ReduceMax":
        return [np.asarray(vals[0].max())]
    if op == "ReduceMin":
        return [np.asarray(vals[0].min())]
    if op == "Fill":
        return [np.full(attrs["shape"], vals[0], dtype=np.asarray(vals[0]).dtype)]
    if op == "ZerosLike":
        return [np.zeros_like(vals[0])]
    if op == "Less":
        return [np.asarray(vals[0] < vals[1])]
    if op == "LessEqual":
        return [np.asarray(vals[0] <= vals[1])]
    if op == "Greater":
        return [np.asarray(vals[0] > vals[1])]
    if op == "Equal":
        return [np.asarray(vals[0] == vals[1])]
    if op == "LogicalAnd":
        return [np.asarray(np.logical_and(vals[0], vals[1]))]
    if op == "LogicalNot":
        return [np.asarray(np.logical_not(vals[0]))]
    if op == "Select":
        c = np.asarray(vals[0])
        a, b = vals[1], vals[2]
        if c.ndim == 1 and np.ndim(a) == 2:      # row mask [B] over [B, n]
            c = c[:, None]
        return [np.where(c, a, b)]
    if op == "Sigmoid":
        return [sigmoid(vals[0])]
    if op == "Tanh":
        return [np.tanh(vals[0])]
    if op == "Relu":
        return [np.maximum(vals[0], 0.0)]
    if op == "ReluGrad":
        return [vals[0] * (vals[1] > 0.0)]
    if op == "Concat":
        return [np.concatenate(vals, axis=attrs["axis"])]
    if op == "Slice":
        idx = tuple(slice(b0, b0 + s) for b0, s in zip(attrs["begin"], attrs["size"]))
        return [np.array(vals[0][idx], copy=True)]
    if op == "SliceGrad":
        out = np.zeros(attrs["shape"], dtype=vals[0].dtype)
        idx = tuple(slice(b0, b0 + s) for b0, s in zip(attrs["begin"], attrs["size"]))
        out[idx] = vals[0]
        return [out]
    if op == "Reshape":
        return [np.reshape(vals[0], attrs["shape"]).copy()]
    if op == "Cast":
        return [np.asarray(vals[0]).astype({"f64": np.float64, "i64": np.int64,
                                            "bool": bool}[attrs["dtype"]])]
    if op == "LSTMCell":
        x, h, c, W, b = vals[:5]
        if attrs.get("masked"):
            r = list(lstm_cell(x, h, c, W, b, vals[5], vals[6], attrs.get("forget_bias", 0.0)))
        else:
            r = list(lstm_cell(x, h, c, W, b, forget_bias=attrs.get("forget_bias", 0.0)))
        return r
    if op == "LSTMCellGrad":
        x, h, c, W, gates = vals[:5]
        if attrs.get("masked"):
            t, lens, dhn, dcn, dout = vals[5:10]
            return list(lstm_cell_grad(x, h, c, W, gates, dhn, dcn, dout, t, lens))
        dhn, dcn, dout = vals[5:8]
        return list(lstm_cell_grad(x, h, c, W, gates, dhn, dcn, dout))
    raise NotImplementedError(op)
