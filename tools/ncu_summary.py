"""Summarise one `ncu --set full` capture of cf_driver_kernel into the JSON bench.py reads as
roofline.traffic (profiles/traffic_cfg3_bf16.json). Usage:

    python tools/ncu_summary.py <capture.ncu-rep> <out.json> "<source description>"

Reads `ncu -i ... --page raw --csv` (the metric names of /opt/skills/guides/B200_PROFILING.md)
and keeps the previous file's `round1` key, if any.
"""
import csv
import io
import json
import os
import subprocess
import sys


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    names, units, vals = rows[0], rows[1], rows[2]   # header, units, the first (only) launch
    return {n: (v, u) for n, u, v in zip(names, units, vals)}


def num(m, name, scale_by_unit=None):
    if name not in m:
        stem = name.split(".")[0]
        raise SystemExit(f"{name} not in the capture; similar: {[k for k in m if k.startswith(stem)]}")
    v, u = m[name]
    x = float(v.replace(",", ""))
    return x * (scale_by_unit or {}).get(u, 1.0)


def main():
    rep, out, source = sys.argv[1], sys.argv[2], sys.argv[3]
    m = raw_metrics(rep)
    byte_scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    time_scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
    clk_scale = {"hz": 1e-9, "Khz": 1e-6, "Mhz": 1e-3, "Ghz": 1.0}
    rd = num(m, "dram__bytes_read.sum", byte_scale)
    wr = num(m, "dram__bytes_write.sum", byte_scale)
    res = {
        "source": source,
        "gpu_time_ms": num(m, "gpu__time_duration.sum", time_scale),
        "dram_read_bytes": rd,
        "dram_write_bytes": wr,
        "bytes_per_launch": rd + wr,
        "tensor_pipe_active_pct_elapsed": num(
            m, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        "l2_hit_pct": num(m, "lts__t_sector_hit_rate.pct"),
        "sm_clock_ghz": num(m, "sm__cycles_elapsed.avg.per_second", clk_scale),
        "registers_per_thread": num(m, "launch__registers_per_thread"),
    }
    if os.path.exists(out):
        prev = json.load(open(out))
        if "round1" in prev:
            res["round1"] = prev["round1"]
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
