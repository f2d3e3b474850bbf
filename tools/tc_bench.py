"""Throughput of the tcgen05 tile engine alone (cf_debug_tc_gemm: one 128 x bn tile per CTA,
4-stage TMA ring, fp32 TMEM accumulator, plain fp32 store epilogue) next to torch.matmul."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_1805_01772_b200 import cf  # noqa: E402


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = []
for (M, N, K, bn) in [(512, 4096, 2048, 256), (4096, 4096, 4096, 256), (8192, 8192, 4096, 256),
                      (512, 4096, 2048, 128), (2048, 2048, 16384, 256)]:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    C = torch.empty(M, N, device="cuda")
    ms = timeit(lambda: cf.debug_tc_gemm(M, N, K, bn, 0, 0, A, B, C))
    ms_t = timeit(lambda: torch.matmul(A, B.t()))
    fl = 2.0 * M * N * K
    tiles = (M // 128) * (N // bn)
    res.append({"M": M, "N": N, "K": K, "bn": bn, "tiles": tiles, "tc_ms": ms, "tc_tflops": fl / ms / 1e9,
                "us_per_tile_wave": ms * 1e3 / max(1, -(-tiles // 148)),
                "torch_ms": ms_t, "torch_tflops": fl / ms_t / 1e9})
    print(json.dumps(res[-1]), flush=True)
