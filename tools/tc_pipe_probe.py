"""Mainloop throughput of the 256-row tcgen05 engine in isolation (cf_debug_tc_pipe): persistent
CTAs, 256 x 256 tiles, accumulator-read-only epilogue; the weight operand cycles over nb copies
(nb = 1: 16 MB, L2-resident; nb = 8: 128 MB, like cfg3's 8 layers). One JSON line per case."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_1805_01772_b200 import cf  # noqa: E402

for (M, N, K) in [(512, 4096, 2048), (512, 2048, 4096)]:
    for nb in (1, 8):
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        B = torch.randn(nb, N, K, device="cuda").to(torch.bfloat16)
        for pf in (0, 4, -1):   # -1: 128-row tiles (tc_tile)
            reps = max(1, 40 // nb)
            ms = cf.debug_tc_pipe(M, N, K, nb, reps, pf, A, B)
            fl = 2.0 * M * N * K * nb * reps
            tiles = (M // (128 if pf < 0 else 256)) * (N // 256) * nb * reps
            print(json.dumps({"M": M, "N": N, "K": K, "weight_copies": nb, "weight_MB": nb * N * K * 2 / 2**20,
                              "prefetch": max(pf, 0), "rows": 128 if pf < 0 else 256, "tiles": tiles, "ms": ms, "tflops": fl / ms / 1e9,
                              "us_per_tile_per_sm": ms * 1e3 * 148 / tiles}), flush=True)
