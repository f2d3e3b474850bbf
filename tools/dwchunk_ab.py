"""A/B of the dW chunk length (CF_DW_CHUNK at compile time; default 8 steps) on cfg3: ms per run.

One session per chunk length (the dz and swap-in rings are sized for it). Also checks the
fetched gradients against the first chunk (fp32 accumulation order is the only difference, so
they agree to rounding) and, with PHASES=1, prints the tile phase clocks of one run."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
from bench import CONFIGS  # noqa: E402
from paper_1805_01772_b200 import cf  # noqa: E402
from paper_1805_01772_b200.models import dynamic_rnn_lstm, feeds_to_device  # noqa: E402
from synth import rnn_inputs  # noqa: E402

c = dict(CONFIGS[os.environ.get("CFG", "cfg3")])
p = dynamic_rnn_lstm(c["T"], c["B"], c["I"], c["H"], c["L"])
f = rnn_inputs(c["T"], c["B"], c["I"], c["H"], c["L"], seed=0, len_mode=c["len_mode"], bf16=True)
chunks = [int(x) for x in os.environ.get("CHUNKS", "8 12 16").split()]
sessions = {}
for ch in chunks:
    os.environ["CF_DW_CHUNK"] = str(ch)
    s = cf.Session(p.g, p.fetch_tensors(), precision=cf.BF16)
    sessions[ch] = (s, feeds_to_device(f, session=s), s.alloc_outputs())
os.environ.pop("CF_DW_CHUNK")
flags = [int(x) for x in os.environ.get("FLAGS", "0").split(",")]   # cf_debug_set_flags A/B
knob0 = [int(x) for x in os.environ.get("KNOB0", "0").split(",")]   # cf_debug_set_knob(0, v)
knob1 = [int(x) for x in os.environ.get("KNOB1", "0").split(",")]   # cf_debug_set_knob(1, v)
m2rows = [int(x) for x in os.environ.get("M2ROWS", "0").split(",")]   # cf_debug_set_m2_rows
ref = None
for rep in range(2):
    for ch in chunks:
        for fl, k0, m2, k1 in [(a, b, c, e) for a in flags for b in knob0 for c in m2rows
                                for e in knob1]:
            cf.debug_set_flags(fl)
            cf.debug_set_knob(0, k0)
            cf.debug_set_knob(1, k1)
            cf.debug_set_m2_rows(m2)
            s, dev, outs = sessions[ch]
            s.run(dev, outs)
            ts = []
            for _ in range(3):
                _, _, tr = s.run(dev, outs, trace=True)
                ts.append(tr["wall_ms"])
            torch.cuda.synchronize()
            if ref is None:
                ref = [o.clone() for o in outs]
            err = max(float(((a.double() - b.double()).abs().max() /
                             (b.double().abs().max() + 1e-30))) for a, b in zip(outs, ref))
            print(f"dw_chunk={ch} flags={fl} knob0={k0} knob1={k1} m2rows={m2}: {sorted(ts)[1]:.2f} ms  max rel diff vs the first "
                  f"{err:.2e}", flush=True)
cf.debug_set_flags(0)
cf.debug_set_knob(0, 0)
cf.debug_set_knob(1, 0)
cf.debug_set_knob(2, 0)
cf.debug_set_m2_rows(0)
if os.environ.get("PHASES"):
    cf.debug_set_knob(0, knob0[-1])
    s, dev, outs = sessions[chunks[0]]
    cf.debug_tile_phases(reset=True)
    cf.debug_set_flags(1 << 22)
    _, _, tr = s.run(dev, outs, trace=True)
    torch.cuda.synchronize()
    cf.debug_set_flags(0)
    ph = cf.debug_tile_phases(reset=True)
    ghz = ph[19] / max(ph[18], 1)   # SM cycles per ns over the forward tiles
    print(f"phases: SM clock under load {ghz:.3f} GHz (forward tiles' cycles / globaltimer ns)")
    for k, name in enumerate(["fwd", "dxh", "dw", "bwd_ew"]):
        n = max(ph[4 * k], 1)
        print(f"phases {name}: tiles {ph[4 * k]}  setup {ph[4 * k + 1] / n / ghz / 1e3:.2f} us  "
              f"mainloop {ph[4 * k + 2] / n / ghz / 1e3:.2f} us  epilogue {ph[4 * k + 3] / n / ghz / 1e3:.2f} us"
              f"  (run {tr['wall_ms']:.2f} ms with the clocks on)", flush=True)
    n = max(ph[0], 1)
    print(f"phases fwd epilogue: TMEM+math+staging {ph[16] / n / ghz / 1e3:.2f} us, barrier "
          f"{ph[17] / n / ghz / 1e3:.2f} us, copy-out = the rest", flush=True)
