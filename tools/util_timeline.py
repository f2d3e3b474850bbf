"""SM utilisation over time from a profile_run.py .npy (busy SMs per bin, by instance kind).

    python tools/util_timeline.py gpurun_out/x_prof.npy [bin_ms] [ranges like 0-3,20-30]"""
import sys

import numpy as np

KINDS = ["NOP", "EW", "FILL", "COPY", "RSUM", "RSUM0", "MATMUL", "LSTM_FWD", "LSTM_BWD_EW",
         "LSTM_BWD_MM", "ACC", "PREPWP", "PREPWT", "FWD", "EWbf", "DXH", "DW", "SWAP", "WAIT",
         "XPROJ", "MMTC"]
r = np.load(sys.argv[1])
binms = float(sys.argv[2]) if len(sys.argv) > 2 else 0.25
ranges = [tuple(float(v) for v in x.split("-")) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else None
st, en, busy, kind = r[:, 2], r[:, 3], r[:, 4], r[:, 5].astype(int)
ok = np.isfinite(st) & np.isfinite(en) & (en > st)
nb = int(np.nanmax(en[ok]) / 1e6 / binms) + 1
util = np.zeros((nb, len(KINDS)))
for i in np.where(ok)[0]:
    a, b = st[i] / 1e6 / binms, en[i] / 1e6 / binms
    rate = busy[i] / 1e6 / binms / (b - a)
    for j in range(int(a), int(b) + 1):
        lo, hi = max(a, j), min(b, j + 1)
        if hi > lo:
            util[j, min(kind[i], len(KINDS) - 1)] += rate * (hi - lo)
for j in range(nb):
    t = j * binms
    if ranges and not any(lo <= t <= hi for lo, hi in ranges):
        continue
    parts = " ".join(f"{KINDS[k]}:{util[j, k]:5.1f}" for k in range(len(KINDS)) if util[j, k] > 0.5)
    print(f"{t:7.2f} ms  busy {util[j].sum():6.1f}  {parts}")
print(f"mean busy SMs {util.sum() / nb:.1f} over {nb * binms:.2f} ms")
