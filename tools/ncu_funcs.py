"""Per-function instruction counts and warp-stall samples of the device driver from an ncu
source page (--print-source=sass csv) and the matching runtime.cu.o (function symbol sizes)."""
import bisect
import csv
import os
import subprocess
import sys
import tempfile


def syms_of(obj):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True,
                   stdout=subprocess.DEVNULL)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    out = subprocess.run(["readelf", "-sW", os.path.join(d, cub)], capture_output=True, text=True).stdout
    syms = []
    for l in out.splitlines():
        f = l.split()
        if len(f) < 8 or f[3] != "FUNC":
            continue
        name = f[7].split("Driver")[-1] if "Driver" in f[7] else f[7][-40:]
        syms.append((int(f[1], 16), int(f[2], 0), name))
    return sorted([s for s in syms if s[1] > 0 and s[0] > 0])


def main(rep, obj, top=22):
    csvp = rep + ".sass.csv"
    with open(csvp, "w") as fo:
        subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], stdout=fo,
                       stderr=subprocess.DEVNULL)
    subs = syms_of(obj)
    keys = [s[0] for s in subs]
    hdr, recs = None, []
    for r in csv.reader(open(csvp)):
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and r and r[0].startswith("0x"):
            recs.append((int(r[0], 16), dict(zip(hdr, r))))
    base = recs[0][0]

    def I(x):
        try:
            return int(x)
        except ValueError:
            return 0
    agg = {}
    for a, d in recs:
        off = a - base
        k = bisect.bisect_right(keys, off) - 1
        name = subs[k][2] if k >= 0 and off < subs[k][0] + subs[k][1] else "kernel-body"
        x = agg.setdefault(name, [0, 0, {}])
        x[0] += I(d["Instructions Executed"])
        x[1] += I(d["Warp Stall Sampling (All Samples)"])
        for kk, v in d.items():
            if kk.startswith("stall_") and "Not Issued" not in kk and I(v):
                x[2][kk[6:]] = x[2].get(kk[6:], 0) + I(v)
    drv = {k: v for k, v in agg.items() if k != "kernel-body"}
    ts = sum(v[1] for v in drv.values())
    print(f"driver functions: {sum(v[0] for v in drv.values())} warp-instr, {ts} samples")
    for n, (i, s, st) in sorted(drv.items(), key=lambda x: -x[1][1])[:top]:
        tops = sorted(st.items(), key=lambda x: -x[1])[:4]
        print(f"{n[:30]:30s} instr {i:9d} samples {s:6d} {100 * s / max(ts, 1):5.1f}%  {tops}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
