"""Seeded synthetic input generator shared by the oracle and the CUDA path.

Holds NONE of the method's arithmetic: it only draws random tensors. Recipe (SURVEY.md §8(d),
DESIGN.md "Input recipe"): ``numpy.random.default_rng(seed)``; W, b ~ U(-1/sqrt(H), 1/sqrt(H))
(PyTorch LSTM init); x ~ N(0, 1); h0, c0 ~ N(0, 0.1^2); R ~ N(0, 1); lengths per the config;
MoE experts ~ U(-1/sqrt(H), 1/sqrt(H)); route bits ~ Bernoulli(0.5). With ``bf16=True`` every
float input is rounded to the nearest bfloat16 value first (reading R16) so that the fp64
oracle and the bf16 device path start from identical numbers.
"""
from __future__ import annotations

from typing import Dict

import numpy as np


def round_bf16(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float64 (exact)."""
    f = np.asarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def lengths(rng: np.random.Generator, B: int, T: int, mode: str) -> np.ndarray:
    if mode == "full":
        return np.full(B, T, dtype=np.int64)
    if mode == "uniform":          # len_b ~ U{1..T}, one row forced to T
        l = rng.integers(1, T + 1, size=B)
        l[rng.integers(0, B)] = T
        return l.astype(np.int64)
    if mode == "capped":           # len_b ~ U{1..0.75T}: exercises the empty_update branch
        l = rng.integers(1, max(1, (3 * T) // 4) + 1, size=B)
        return l.astype(np.int64)
    if mode == "upper_half":       # len_b ~ U{T/2..T}
        return rng.integers(T // 2, T + 1, size=B).astype(np.int64)
    if mode == "split_tiles":      # length-sorted batch: first half U{T/2..T} (one row T),
        h = B // 2                 # second half U{1..T/4}: whole row tiles finish early
        l = np.concatenate([rng.integers(T // 2, T + 1, size=h),
                            rng.integers(1, max(1, T // 4) + 1, size=B - h)])
        l[0] = T
        return l.astype(np.int64)
    if mode == "with_zero":        # includes a zero-length row and a full row
        l = rng.integers(0, T + 1, size=B)
        l[0] = 0
        l[-1] = T
        return l.astype(np.int64)
    raise ValueError(mode)


def rnn_inputs(T: int, B: int, I: int, H: int, L: int = 1, seed: int = 0,
               len_mode: str = "full", moe: bool = False, bf16: bool = False,
               uniform_pos: bool = False) -> Dict[str, np.ndarray]:
    """Feeds for the dynamic_rnn LSTM program (names match both builders)."""
    rng = np.random.default_rng(seed)
    k = 1.0 / np.sqrt(H)
    f: Dict[str, np.ndarray] = {}
    if uniform_pos:   # SPEC.md:263 finite-difference recipe: inputs U[0.5, 1.5]
        f["x"] = rng.uniform(0.5, 1.5, size=(T, B, I))
    else:
        f["x"] = rng.standard_normal((T, B, I))
    f["len"] = lengths(rng, B, T, len_mode)
    for l in range(L):
        il = I if l == 0 else H
        f[f"W{l}"] = rng.uniform(-k, k, size=(4 * H, il + H))
        f[f"b{l}"] = rng.uniform(-k, k, size=(4 * H,))
        f[f"h0_{l}"] = 0.1 * rng.standard_normal((B, H))
        f[f"c0_{l}"] = 0.1 * rng.standard_normal((B, H))
        f[f"R_h{l}"] = rng.standard_normal((B, H))
        f[f"R_c{l}"] = rng.standard_normal((B, H))
        if moe:
            f[f"WA{l}"] = rng.uniform(-k, k, size=(H, H))
            f[f"WB{l}"] = rng.uniform(-k, k, size=(H, H))
    f["R_out"] = rng.standard_normal((T, B, H))
    if moe:
        f["route"] = rng.random((T, L)) < 0.5
    if bf16:
        for name, v in f.items():
            if v.dtype == np.float64:
                f[name] = round_bf16(v)
    return f


def shard_inputs(feeds: Dict[str, np.ndarray], rank: int, world: int) -> Dict[str, np.ndarray]:
    """Batch shard `rank` of `world` (batch data parallelism): rows [rank * B / world,
    (rank + 1) * B / world) of every per-sample input (x, R_out: axis 1; len, h0, c0, R_h,
    R_c: axis 0); the weights are shared. Pure slicing."""
    out = {}
    for k, v in feeds.items():
        v = np.asarray(v)
        if k in ("x", "R_out"):
            b = v.shape[1] // world
            out[k] = v[:, rank * b:(rank + 1) * b]
        elif k == "len" or k.startswith(("h0_", "c0_", "R_h", "R_c")):
            b = v.shape[0] // world
            out[k] = v[rank * b:(rank + 1) * b]
        else:
            out[k] = v
    return out
