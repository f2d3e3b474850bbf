"""Per-CUDA-line warp-stall samples from an ncu source page (--print-source=cuda,sass csv),
restricted to a line range of one file (e.g. the device driver's code)."""
import csv
import sys


def main(path, lo, hi, top=40, fname="runtime.cu"):
    cur_file = None
    out = []
    with open(path) as f:
        rd = csv.reader(f)
        hdr = None
        for r in rd:
            if len(r) >= 2 and r[0] == "File Path":
                cur_file = r[1]
                continue
            if r and r[0] == "Line No":
                hdr = r
                continue
            if hdr is None or not r or not r[0] or not cur_file or not cur_file.endswith(fname):
                continue
            ln = int(r[0])
            if lo <= ln <= hi:
                d = dict(zip(hdr[4:], r[4:]))
                s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
                stalls = {k: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k
                          and v.isdigit() and int(v) > 0}
                out.append((s, ln, r[1][:90], sorted(stalls.items(), key=lambda x: -x[1])[:3]))
    tot = sum(o[0] for o in out)
    print(f"total samples in {fname}:{lo}-{hi}: {tot}")
    for s, ln, src, st in sorted(out, reverse=True)[:top]:
        print(f"{s:7d} {100.0 * s / max(tot, 1):5.1f}%  {ln:5d}  {src:90s} {st}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]) if len(sys.argv) > 4 else 40)
