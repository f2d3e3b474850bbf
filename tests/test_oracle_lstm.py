"""Pins for the oracle's LSTM workload (CPU only).

* torch.nn.LSTM (float64) + torch.autograd on each unpadded sequence -- a library routine
  independent of the oracle (readings R9, R10).
* Central finite differences, step 1e-6, inputs U[0.5, 1.5], max relative error <= 1e-5
  (SPEC.md:263).
* Fused LSTMCell / LSTMCellGrad == the composite of primitive ops differentiated by the
  generic autodiff.
* Brute-force enumeration of the MoE cond's route bits against a host-language (out-of-graph)
  torch loop with Python ``if`` (PAPER.md:160-167 describes out-of-graph control flow).
* Length semantics: each row's final state equals a separate unpadded run of that row.
* Invariants on every run: Exit fires once per frame, pushes == pops per stack, the window
  bound, parallel_iterations / scheduling invariance (bit-identical values).
"""
import itertools

import numpy as np
import pytest
import torch

from oracle import interp, kernels
from oracle.autodiff import gradients
from oracle.graph import FLOAT, INT, Builder
from oracle.models import dynamic_rnn_lstm, run_program
from synth import rnn_inputs
from torch_lstm_ref import torch_dynamic_rnn


def _maxrel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


CASES = [
    (5, 2, 4, 8, 1, "full"),        # cfg1 (BASELINE.json configs[0]): L1 H8 B2 T5, I=4
    (5, 2, 4, 8, 1, "uniform"),
    (5, 3, 4, 8, 2, "with_zero"),   # zero-length row: final state = initial state
    (6, 4, 3, 5, 3, "capped"),      # t >= max_len takes the empty_update branch
]


@pytest.mark.parametrize("T,B,I,H,L,mode", CASES)
def test_matches_torch_lstm(T, B, I, H, L, mode):
    p = dynamic_rnn_lstm(T, B, I, H, L)
    for seed in (0, 1):
        f = rnn_inputs(T, B, I, H, L, seed=seed, len_mode=mode)
        r = run_program(p, f)
        ref = torch_dynamic_rnn(f, T, B, I, H, L)
        for k, v in ref.items():
            assert _maxrel(r[k], v) <= 1e-12, (k, _maxrel(r[k], v))


def test_finite_differences():
    T, B, I, H, L = 4, 2, 3, 4, 2
    p = dynamic_rnn_lstm(T, B, I, H, L)
    f = rnn_inputs(T, B, I, H, L, seed=5, len_mode="uniform", uniform_pos=True)
    r = run_program(p, f)
    rng = np.random.default_rng(0)
    h = 1e-6

    def loss(ff):
        return float(interp.run(p.b.g, ff, [p.fetch["y"]])[0])
    worst = 0.0
    for name in ["x", "W0", "b0", "h0_0", "c0_0", "W1", "b1", "h0_1", "c0_1"]:
        g = r["d" + name]
        for _ in range(3):
            idx = tuple(int(rng.integers(0, s)) for s in f[name].shape)
            fp = dict(f)
            fm = dict(f)
            fp[name] = f[name].copy()
            fm[name] = f[name].copy()
            fp[name][idx] += h
            fm[name][idx] -= h
            fd = (loss(fp) - loss(fm)) / (2 * h)
            worst = max(worst, abs(fd - g[idx]) / max(abs(g).max(), 1e-12))
    assert worst <= 1e-5, worst


def _composite_cell(b, x, hh, c, W, bias, t, lens, H):
    """LSTMCell written out with primitive ops (reading R9/R10)."""
    z = b.op1("BiasAdd", [b.matmul(b.op1("Concat", [x, hh], {"axis": 1}), W, tb=True), bias])
    B = b.g.shape(x)[0]

    def sl(k):
        return b.op1("Slice", [z], {"begin": (0, k * H), "size": (B, H)})
    i, fg, o = (b.op1("Sigmoid", [sl(k)]) for k in (0, 1, 3))
    g = b.op1("Tanh", [sl(2)])
    cn = b.add(b.mul(fg, c), b.mul(i, g))
    hn = b.mul(o, b.op1("Tanh", [cn]))
    live = b.op1("Less", [b.op1("Fill", [t], {"shape": (B,)}), lens])
    return (b.op1("Select", [live, hn, hh]), b.op1("Select", [live, cn, c]),
            b.op1("Select", [live, hn, b.zeros((B, H))]))


def test_fused_cell_equals_composite():
    B, I, H = 3, 4, 5
    rng = np.random.default_rng(7)
    feeds = {"x": rng.standard_normal((B, I)), "h": rng.standard_normal((B, H)),
             "c": rng.standard_normal((B, H)), "W": rng.standard_normal((4 * H, I + H)) * 0.4,
             "bias": rng.standard_normal(4 * H), "t": np.int64(2),
             "len": np.array([1, 3, 5], dtype=np.int64),
             "Rh": rng.standard_normal((B, H)), "Rc": rng.standard_normal((B, H)),
             "Ro": rng.standard_normal((B, H))}
    outs = []
    for fused in (True, False):
        b = Builder()
        ph = {k: b.placeholder(k, INT if k in ("t", "len") else FLOAT, np.shape(v))
              for k, v in feeds.items()}
        if fused:
            hn, cn, o, _ = b.op("LSTMCell", [ph["x"], ph["h"], ph["c"], ph["W"], ph["bias"],
                                             ph["t"], ph["len"]], {"masked": True})
        else:
            hn, cn, o = _composite_cell(b, ph["x"], ph["h"], ph["c"], ph["W"], ph["bias"],
                                        ph["t"], ph["len"], H)
        y = b.add(b.add(b.reduce_sum(b.mul(ph["Rh"], hn)), b.reduce_sum(b.mul(ph["Rc"], cn))),
                  b.reduce_sum(b.mul(ph["Ro"], o)))
        gs = gradients(b, y, [ph["x"], ph["h"], ph["c"], ph["W"], ph["bias"]])
        outs.append(interp.run(b.g, feeds, [hn, cn, o, y] + gs))
    for a, c in zip(*outs):
        assert _maxrel(a, c) <= 1e-13


def _torch_moe_out_of_graph(f, T, B, I, H, L, route, act="relu"):
    """Host-language loop with Python `if` on the route bits (out-of-graph control flow)."""
    x = torch.tensor(f["x"], requires_grad=True)
    params = {}
    for k in f:
        if k.startswith(("W", "b", "h0_", "c0_", "WA", "WB")):
            params[k] = torch.tensor(f[k], requires_grad=True)
    lens = [int(v) for v in f["len"]]
    hs = [params[f"h0_{l}"] for l in range(L)]
    cs = [params[f"c0_{l}"] for l in range(L)]
    outs = []
    for t in range(T):
        inp = x[t]
        for l in range(L):
            W, bb = params[f"W{l}"], params[f"b{l}"]
            z = torch.cat([inp, hs[l]], 1) @ W.T + bb
            i, fg, g, o = z[:, :H].sigmoid(), z[:, H:2 * H].sigmoid(), z[:, 2 * H:3 * H].tanh(), \
                z[:, 3 * H:].sigmoid()
            cn = fg * cs[l] + i * g
            hn = o * cn.tanh()
            live = torch.tensor([t < n for n in lens])[:, None]
            out = torch.where(live, hn, torch.zeros_like(hn))
            hs[l] = torch.where(live, hn, hs[l])
            cs[l] = torch.where(live, cn, cs[l])
            fn = torch.relu if act == "relu" else torch.tanh
            if route[t, l]:
                out = out + fn(out @ params[f"WA{l}"])
            else:
                out = out + fn(out @ params[f"WB{l}"])
            inp = out
        outs.append(inp)
    y = (torch.tensor(f["R_out"]) * torch.stack(outs)).sum()
    for l in range(L):
        y = y + (torch.tensor(f[f"R_h{l}"]) * hs[l]).sum() + (torch.tensor(f[f"R_c{l}"]) * cs[l]).sum()
    y.backward()
    res = {"y": y.item(), "dx": x.grad.numpy()}
    for k, v in params.items():
        res["d" + k] = v.grad.numpy() if v.grad is not None else np.zeros(v.shape)
    return res


@pytest.mark.parametrize("act", ["relu", "tanh"])
def test_moe_cond_brute_force(act):
    """All 2^T route patterns of a T=4, L=1 loop with a gated branch (cfg5 structure), for
    both expert activations (reading R21)."""
    T, B, I, H, L = 4, 2, 3, 4, 1
    p = dynamic_rnn_lstm(T, B, I, H, L, moe=True, moe_act=act)
    base = rnn_inputs(T, B, I, H, L, seed=11, len_mode="uniform", moe=True)
    for bits in itertools.product([False, True], repeat=T):
        f = dict(base)
        f["route"] = np.array(bits).reshape(T, L)
        r, tr = run_program(p, f, return_trace=True)
        ref = _torch_moe_out_of_graph(f, T, B, I, H, L, f["route"], act)
        for k, v in ref.items():
            assert _maxrel(r[k], v) <= 1e-12, (bits, k)
        assert set(tr.pushes) == set(tr.pops)
        assert all(tr.pushes[s] == tr.pops[s] for s in tr.pushes)


def test_length_semantics_self_consistency():
    """A row's final state equals a separate unpadded run of that row alone (reading R10)."""
    T, B, I, H = 6, 3, 2, 4
    f = rnn_inputs(T, B, I, H, 1, seed=2, len_mode="uniform")
    r = run_program(dynamic_rnn_lstm(T, B, I, H, 1, with_grads=False), f)
    for bi in range(B):
        n = int(f["len"][bi])
        h, c = f["h0_0"][bi:bi + 1], f["c0_0"][bi:bi + 1]
        for t in range(n):
            h, c, _, _ = kernels.lstm_cell(f["x"][t, bi:bi + 1], h, c, f["W0"], f["b0"])
        assert np.allclose(r["hT0"][bi], h[0], rtol=0, atol=1e-15)
        assert np.allclose(r["cT0"][bi], c[0], rtol=0, atol=1e-15)
        assert np.all(r["out"][n:, bi] == 0.0)


@pytest.mark.parametrize("K,seed", [(1, None), (8, 3), (32, 4), (2, 5)])
def test_invariants_and_parallel_iterations(K, seed):
    T, B, I, H, L = 5, 3, 4, 6, 2
    p = dynamic_rnn_lstm(T, B, I, H, L, parallel_iterations=32)
    f = rnn_inputs(T, B, I, H, L, seed=9, len_mode="capped")
    ref = run_program(p, f, K=1)
    r, tr = run_program(p, f, K=K, sched_seed=seed, return_trace=True)
    for k in ref:
        assert np.array_equal(np.asarray(r[k]), np.asarray(ref[k])), k
    # each Exit fires once per frame instance
    assert tr.exit_fires and all(v == 1 for v in tr.exit_fires.values())
    # forward push count equals backward pop count, per stack
    assert tr.pushes and all(tr.pushes[s] == tr.pops[s] for s in tr.pushes)
    # trip counts: forward and gradient loop both run T iterations
    assert sorted(tr.trip_counts.values()) == [T, T]
    # window bound and no dead token ever reaches a loop Merge
    assert all(m <= K for m in tr.max_inflight.values())
    assert tr.live_merge_dead_inputs == 0
    # branch bits: outer cond t < max_len, inner cond t < min_len (reading R10)
    mx, mn = int(f["len"].max()), int(f["len"].min())
    outer = {tag[-1][1]: v for (cid, tag), v in tr.branch.items() if cid == 0 and len(tag) == 1}
    assert outer == {t: t < mx for t in range(T)}
    inner = {tag[-1][1]: v for (cid, tag), v in tr.branch.items() if cid == 1 and len(tag) == 1}
    assert inner == {t: t < mn for t in range(mx)}



def test_synth_bf16_rounding_is_torchs_bf16():
    """Reading R16: bf16 parity inputs are rounded to bf16 by the input generator (round to
    nearest even, as a float32 -> bf16 cast; checked against torch, a library routine); the
    oracle then runs fp64 on exactly those values."""
    import torch

    from synth import rnn_inputs, round_bf16
    rng = np.random.default_rng(0)
    a = rng.standard_normal(20000) * 10.0 ** rng.integers(-12, 12, 20000)
    assert np.array_equal(round_bf16(a), torch.tensor(a, dtype=torch.float32).to(torch.bfloat16).double().numpy())
    f = rnn_inputs(3, 2, 4, 8, 1, seed=0, len_mode="full", bf16=True)
    for k, v in f.items():
        if v.dtype == np.float64:
            assert np.array_equal(round_bf16(v), v), k
