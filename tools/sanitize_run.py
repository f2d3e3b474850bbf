"""Small runs of the device path for compute-sanitizer (memcheck / racecheck / synccheck):
fp32 and bf16 (tcgen05) multi-layer LSTM programs with ragged lengths, plus the MoE cond.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1805_01772_b200 import cf  # noqa: E402
from paper_1805_01772_b200.models import dynamic_rnn_lstm, feeds_to_device  # noqa: E402
from synth import rnn_inputs  # noqa: E402

cases = [("f32", 4, 40, 24, 32, 2, {}), ("bf16", 4, 300, 256, 256, 2, {}),
         ("bf16", 3, 96, 256, 256, 2, {"moe": True, "moe_act": "tanh"})]
for prec, T, B, I, H, L, kw in cases:
    p = dynamic_rnn_lstm(T, B, I, H, L, **kw)
    s = cf.Session(p.g, p.fetch_tensors(), precision=cf.BF16 if prec == "bf16" else cf.F32,
                   watchdog_ms=600000)
    f = rnn_inputs(T, B, I, H, L, seed=1, len_mode="uniform", moe=kw.get("moe", False), bf16=prec == "bf16")
    outs, dead, tr = s.run(feeds_to_device(f, session=s), trace=True)
    torch.cuda.synchronize()
    ok = all(bool(torch.isfinite(o.float()).all()) for o in outs if o.numel())
    print(f"{prec} T={T} B={B} H={H} L={L} {kw}: trip {tr['trip_count']} finite={ok}", flush=True)
