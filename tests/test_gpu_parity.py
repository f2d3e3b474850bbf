"""GPU parity: the CUDA path (through the C-ABI) vs the fp64 oracle on the same seeded inputs.

Bar (BASELINE.json north_star): control decisions bit-exact (trip counts, branches taken,
stack push/pop counts, Exit firings); forward outputs and gradients within max relative
error 1e-5 on the fp32 path, measured normwise per tensor (reading R15:
max|g - o| / max|o|).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import __graft_entry__  # noqa: E402

__graft_entry__.build()

from paper_1805_01772_b200 import cf  # noqa: E402
from paper_1805_01772_b200.models import dynamic_rnn_lstm, feeds_to_device  # noqa: E402

from oracle.models import dynamic_rnn_lstm as oracle_rnn  # noqa: E402
from oracle.models import run_program  # noqa: E402
from synth import rnn_inputs  # noqa: E402


def normwise(v, r):
    r = np.asarray(r, dtype=np.float64)
    return float(np.abs(np.asarray(v, dtype=np.float64) - r).max() / max(np.abs(r).max(), 1e-30))


def run_device(T, B, I, H, L, f, K=0, precision=None, **kw):
    p = dynamic_rnn_lstm(T, B, I, H, L, **kw)
    s = cf.Session(p.g, p.fetch_tensors(), precision=precision or cf.F32, parallel_iterations=K)
    n_conds = 64
    outs, dead, tr = s.run(feeds_to_device(f, session=s), trace=True, branch_cap=n_conds * (T + 1))
    torch.cuda.synchronize()
    vals = {n: o.double().cpu().numpy() for n, o in zip(p.fetch_names(), outs)}
    return vals, dead, tr


def check_parity(T, B, I, H, L, mode, seed, K=None, tol=1e-5, precision=None, **kw):
    """Every tensor against the plain fp64 oracle (no precision mirroring, reading R16): the
    bf16 runs feed both sides the same bf16-rounded inputs and hold every output and gradient
    to the north star's 2e-2, normwise (reading R15)."""
    bf = precision == cf.BF16
    f = rnn_inputs(T, B, I, H, L, seed=seed, len_mode=mode, moe=kw.get("moe", False), bf16=bf)
    dev, dead, tr = run_device(T, B, I, H, L, f, K=K or 0, precision=precision, **kw)
    q = oracle_rnn(T, B, I, H, L, **kw)
    ref, otr = run_program(q, f, K=K, return_trace=True)
    assert not any(dead)
    errs = {k: normwise(dev[k], ref[k]) for k in ref}
    worst = max(errs.values())
    assert worst <= tol, sorted(errs.items(), key=lambda kv: -kv[1])[:4]
    # ---- control trace, bit-exact
    assert tr["trip_count"] == [otr.trip_counts[((), "rnn")], otr.trip_counts[((), "rnn_grad")]]
    assert tr["pushes"] == sum(otr.pushes.values())
    assert tr["pops"] == sum(otr.pops.values()) == tr["pushes"]
    assert tr["exit_fires"] == sum(otr.exit_fires.values())
    bb = T + 1
    bits = tr["branch_bits"]
    for (cid, tag), v in otr.branch.items():
        it = tag[-1][1] if tag else 0
        assert bits[cid * bb + it] == (2 if v else 1), (cid, tag, v)
    n_dev = sum(1 for b in bits if b)
    assert n_dev == len({(c, (t[-1][1] if t else 0)) for (c, t) in otr.branch})
    return worst, tr


@pytest.mark.parametrize("mode", ["full", "uniform", "with_zero"])
def test_cfg1_tiny(mode):
    """BASELINE.json configs[0]: 1 layer, hidden 8, batch 2, seq_len 5 (I = 4)."""
    check_parity(5, 2, 4, 8, 1, mode, seed=0)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_multilayer_ragged(seed):
    """3 layers, odd sizes (ragged tiles everywhere), t >= max_len takes empty_update."""
    check_parity(7, 37, 13, 45, 3, "capped", seed=seed)


def test_multi_tile_lengths():
    """Several GEMM tiles in every dimension, variable lengths, 2 layers."""
    check_parity(9, 70, 40, 72, 2, "uniform", seed=4)


@pytest.mark.parametrize("K", [1, 2, 8, 32])
def test_parallel_iterations_bit_identical(K):
    T, B, I, H, L = 8, 33, 20, 40, 2
    f = rnn_inputs(T, B, I, H, L, seed=7, len_mode="uniform")
    base, _, _ = run_device(T, B, I, H, L, f, K=1)
    dev, _, tr = run_device(T, B, I, H, L, f, K=K)
    for k in base:
        assert np.array_equal(base[k], dev[k]), k
    assert max(tr["max_inflight"]) <= K


@pytest.mark.parametrize("act", ["relu", "tanh"])
def test_moe_gated_branch(act):
    """cond nested in the loop body with exact route bits (BASELINE.json configs[4] shape)."""
    check_parity(6, 16, 24, 32, 2, "uniform", seed=3, moe=True, moe_act=act)


def test_cfg2_dynamic_rnn():
    """BASELINE.json configs[1]: 1 layer, hidden 512, batch 64, seq_len 100, variable
    lengths via cond/dead tokens; the capped variant runs the dead empty_update branch."""
    worst, tr = check_parity(100, 64, 512, 512, 1, "uniform", seed=0)
    assert tr["trip_count"] == [100, 100]


def test_cfg2_capped_lengths():
    check_parity(100, 64, 512, 512, 1, "capped", seed=1)


def test_missing_feed_is_an_error():
    p = dynamic_rnn_lstm(3, 2, 2, 4, 1)
    s = cf.Session(p.g, p.fetch_tensors())
    f = feeds_to_device(rnn_inputs(3, 2, 2, 4, 1, seed=0))
    del f["x"]
    with pytest.raises(cf.CfError) as e:
        s.run(f)
    assert e.value.code == "CF_E_MISSING_FEED"


# ---------------------------------------------------------------- bf16 tcgen05 path
BF16_TOL = 2e-2   # north star: max relative error 2e-2 on the bf16 tensor-core path


def test_bf16_small_ragged_batch():
    """2 layers, batch 40 (one partial 128-row tile), variable lengths."""
    check_parity(5, 40, 256, 256, 2, "uniform", seed=0, tol=BF16_TOL, precision=cf.BF16)


def test_bf16_multilayer_capped():
    """3 layers, batch 130 (two row tiles, ragged), H != I, empty_update branch taken."""
    check_parity(8, 130, 256, 512, 3, "capped", seed=1, tol=BF16_TOL, precision=cf.BF16)


def test_bf16_wide_batch_256_row_tiles():
    """B >= 256: the forward and d[x,h] GEMMs use 256-row tiles (two TMEM accumulators per
    CTA); B = 300 leaves a ragged second half-tile."""
    cf.debug_set_m2_rows(256)
    try:
        check_parity(4, 300, 256, 256, 2, "uniform", seed=3, tol=BF16_TOL, precision=cf.BF16)
    finally:
        cf.debug_set_m2_rows(0)   # the product default (512)


def test_bf16_cfg3_shape():
    """BASELINE.json configs[2] exactly as bench.py runs it (L=8, H=I=1024, B=512, K=32, the
    product's 256-row tiles) except T truncated to 8; lengths U{4..8} so the masked cells and
    the length conds run too. Plain fp64 oracle, 2e-2 normwise, control trace bit-exact."""
    worst, tr = check_parity(8, 512, 1024, 1024, 8, "upper_half", seed=0, K=32, tol=BF16_TOL,
                             precision=cf.BF16)
    assert tr["trip_count"] == [8, 8]


@pytest.mark.parametrize("B", [512, 640])
def test_bf16_dead_tile_skip(B):
    """A length-sorted batch: the second half of the rows finishes by T/4, so whole 256-row
    forward / d[x,h] tiles and 128-row backward-EW tiles have no live row in later steps and
    skip their GEMM / math; B = 640 leaves a ragged last tile. Plain fp64
    oracle, 2e-2 normwise, control trace bit-exact."""
    check_parity(12, B, 256, 256, 2, "split_tiles", seed=4, tol=BF16_TOL, precision=cf.BF16)


def test_bf16_cfg2_shape():
    """BASELINE.json configs[1] shape on the tcgen05 path."""
    check_parity(100, 64, 512, 512, 1, "uniform", seed=2, tol=BF16_TOL, precision=cf.BF16)


@pytest.mark.parametrize("K", [1, 32])
def test_bf16_parallel_iterations_bit_identical(K):
    T, B, I, H, L = 6, 96, 256, 256, 2
    f = rnn_inputs(T, B, I, H, L, seed=5, len_mode="uniform", bf16=True)
    base, _, _ = run_device(T, B, I, H, L, f, K=8, precision=cf.BF16)
    dev, _, tr = run_device(T, B, I, H, L, f, K=K, precision=cf.BF16)
    for k in base:
        assert np.array_equal(base[k], dev[k]), k
    assert max(tr["max_inflight"]) <= K


def test_bf16_moe_tensor_core_experts():
    """The expert GEMMs and their gradients on the tcgen05 generic GEMM (HK_MATMUL_TC): B = 128,
    H = 512 (two 256-column tiles, K = 512), the forward o·W, dO = dE·Wᵀ (K-major B) and
    dW = oᵀ·dE (MN-major A and B) all take it. Plain fp64 oracle, bf16 bar."""
    check_parity(5, 128, 256, 512, 2, "uniform", seed=9, tol=BF16_TOL, precision=cf.BF16,
                 moe=True, moe_act="tanh")


@pytest.mark.parametrize("K", [1, 8, 32])
def test_bf16_moe_parallel_iterations_sweep(K):
    """BASELINE.json configs[4] in small: parallel_iterations in {1, 8, 32}, a nested MoE-style
    gated cond in the body (route bits select the expert), bf16 tensor-core LSTM path;
    control bit-exact, values within the bf16 bar against the plain fp64 oracle, and
    bit-identical across K. tanh experts (reading R21): a ReLU expert's mask would be a float
    decision taken on bf16-stored values."""
    T, B, I, H, L = 6, 64, 256, 256, 2
    worst, tr = check_parity(T, B, I, H, L, "uniform", seed=8, K=K, tol=BF16_TOL, precision=cf.BF16,
                             moe=True, moe_act="tanh")
    assert max(tr["max_inflight"]) <= K
    f = rnn_inputs(T, B, I, H, L, seed=8, len_mode="uniform", moe=True, bf16=True)
    a, _, _ = run_device(T, B, I, H, L, f, K=K, precision=cf.BF16, moe=True, moe_act="tanh")
    b, _, _ = run_device(T, B, I, H, L, f, K=32, precision=cf.BF16, moe=True, moe_act="tanh")
    for k in a:
        assert np.array_equal(a[k], b[k]), k
