"""How much a concurrent copy slows the cfg3 step (the e2e gap): ms per cf_run
alone, while 662.7 MB (one step's inputs) stream host->device from pinned memory, and while the
same bytes are copied device->device, each on a separate copy stream started just before the
run; h2d_64MB_src repeats one 64 MB pinned window (the same DMA rate over far fewer host
pages); h2d_late_N issues the H2D copy N ms after the launch from a helper thread (cf_run blocks
the host for the whole run), so it overlaps a later part of the step. Times are CUDA events on the session's stream around each run."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
from bench import CONFIGS  # noqa: E402
from paper_1805_01772_b200 import cf  # noqa: E402
from paper_1805_01772_b200.models import dynamic_rnn_lstm, feeds_to_device  # noqa: E402
from synth import rnn_inputs  # noqa: E402

c = dict(CONFIGS["cfg3"])
p = dynamic_rnn_lstm(c["T"], c["B"], c["I"], c["H"], c["L"])
f = rnn_inputs(c["T"], c["B"], c["I"], c["H"], c["L"], seed=0, len_mode=c["len_mode"], bf16=True)
stream = torch.cuda.Stream()
s = cf.Session(p.g, p.fetch_tensors(), precision=cf.BF16, stream=stream.cuda_stream)
dev = feeds_to_device(f, session=s)
outs = s.alloc_outputs()
nbytes = 662704128
host = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
src = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
cs = torch.cuda.Stream()


host_ms = []


def run(mode, n=6):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if mode in ("h2d", "d2d"):
            with torch.cuda.stream(cs):
                dst.copy_(host if mode == "h2d" else src, non_blocking=True)
        elif mode == "h2d_64MB_src":   # the same bytes from one 64 MB pinned window (few host pages)
            with torch.cuda.stream(cs):
                w = 64 << 20
                for o in range(0, nbytes - w + 1, w):
                    dst[o:o + w].copy_(host[:w], non_blocking=True)
        th = None
        if mode.startswith("h2d_late"):   # cf_run blocks the host: a helper thread issues the copy
            delay = int(mode.split("_")[-1]) * 1e-3

            def late():
                time.sleep(delay)
                with torch.cuda.stream(cs):
                    dst.copy_(host, non_blocking=True)
            th = threading.Thread(target=late)
        a.record(stream)
        t0 = time.perf_counter()
        if th:
            th.start()
        s.run(dev, outs)
        host_ms.append(1e3 * (time.perf_counter() - t0))
        b.record(stream)
        if th:
            th.join()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


s.run(dev, outs)
for mode in ["alone", "h2d", "h2d_late_10", "h2d_late_20", "h2d_late_30", "h2d_late_40"] * 2:
    host_ms.clear()
    print(f"{mode}: {run(mode):.2f} ms per run (host time in cf_run {sorted(host_ms)[len(host_ms) // 2]:.2f} ms)",
          flush=True)
