"""Phase timeline of an instance-profiler run (tools/profile_run.py .npy): per time bucket,
worker-SM occupancy by heavy kind, plus forward/backward phase boundaries and the driver's
lead (instance creation ahead of the dependency release)."""
import sys

import numpy as np

KINDS = ["NOP", "EW", "FILL", "COPY", "REDUCE_SUM", "REDUCE_SUM0", "MATMUL", "LSTM_FWD",
         "LSTM_BWD_EW", "LSTM_BWD_MM", "ACC", "PREP_WP", "PREP_WT", "LSTM_FWD_TC",
         "LSTM_BWD_EW_BF", "LSTM_DXH_TC", "LSTM_DW_TC", "SWAP", "WAIT", "LSTM_XPROJ_TC"]


def main(path, nb=40, workers=147):
    r = np.load(path)   # cols: create, publish, first start, last end (ns, rel), busy ns, kind, ntiles
    kind = r[:, 5].astype(int)
    end = np.nanmax(r[:, 3])
    print(f"run {end * 1e-6:.2f} ms, {r.shape[0]} instances")
    for k in np.unique(kind):
        m = kind == k
        print(f"{KINDS[k]:16s} n={m.sum():6d} first={np.nanmin(r[m, 2]) * 1e-6:8.2f} "
              f"last_end={np.nanmax(r[m, 3]) * 1e-6:8.2f} ms  busy={r[m, 4].sum() * 1e-6:8.1f} SM-ms  "
              f"create->publish {np.nanmean(r[m, 1] - r[m, 0]) * 1e-3:7.1f} us  "
              f"publish->start {np.nanmean(r[m, 2] - r[m, 1]) * 1e-3:6.1f} us  "
              f"span {np.nanmean(r[m, 3] - r[m, 2]) * 1e-3:6.1f} us")
    # occupancy: spread each instance's busy time uniformly over its span
    edges = np.linspace(0, end, nb + 1)
    occ = {}
    for k in np.unique(kind):
        m = (kind == k) & np.isfinite(r[:, 2]) & np.isfinite(r[:, 3])
        o = np.zeros(nb)
        for s, e, b in zip(r[m, 2], r[m, 3], r[m, 4]):
            if e <= s:
                continue
            lo = np.clip((edges[:-1]), s, e)
            hi = np.clip(edges[1:], s, e)
            o += b * (hi - lo) / (e - s)
        occ[KINDS[k]] = o / ((edges[1] - edges[0]) * workers)
    names = [k for k in occ if occ[k].sum() > 0.01]
    print("t_ms   " + " ".join(f"{n[:9]:>9s}" for n in names) + "     total")
    for b in range(nb):
        tot = sum(occ[n][b] for n in names)
        print(f"{edges[b] * 1e-6:6.1f} " + " ".join(f"{occ[n][b]:9.2f}" for n in names) + f" {tot:9.2f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
