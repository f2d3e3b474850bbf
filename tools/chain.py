"""Forward recurrence chain analysis of an instance-profiler run: publish latency after the
producers finished, queue wait, span (LSTM_FWD_TC instances in creation order = [t][layer])."""
import sys

import numpy as np

r = np.load(sys.argv[1])
L = int(sys.argv[2]) if len(sys.argv) > 2 else 8
kind = r[:, 5].astype(int)
f = r[kind == 13]
f = f[np.argsort(f[:, 0])]
T = f.shape[0] // L
F = f.reshape(T, L, -1)
cre, pub, st, en = F[..., 0], F[..., 1], F[..., 2], F[..., 3]
gap = np.array([pub[t, l] - max(en[t, l - 1], en[t - 1, l]) for t in range(1, T) for l in range(1, L)])
lead = np.array([max(en[t, l - 1], en[t - 1, l]) - cre[t, l] for t in range(1, T) for l in range(1, L)])
print(f"fwd: publish-after-deps mean {gap.mean()/1e3:.1f} p50 {np.median(gap)/1e3:.1f} p90 "
      f"{np.percentile(gap, 90)/1e3:.1f} us; driver lead (deps end - create) mean {lead.mean()/1e3:.1f} "
      f"us, <0 in {np.mean(lead < 0)*100:.0f}%; queue {np.mean(st - pub)/1e3:.1f} us; span "
      f"{np.mean(en - st)/1e3:.1f} us; per step {np.mean(np.diff(en[T//4:3*T//4, L-1]))/1e3:.1f} us")
