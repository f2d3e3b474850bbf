#!/bin/bash
# Probe the GPU box: SMs, L2, clocks, host cores, pinned copy bandwidth.
mkdir -p gpurun_out
{
nvidia-smi
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | head -20
python - <<'PY'
import torch, time
p = torch.cuda.get_device_properties(0)
print("name", p.name, "sms", p.multi_processor_count, "L2", getattr(p, "L2_cache_size", None), "smem/blk optin", getattr(p,"shared_memory_per_block_optin",None))
n = 256 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory(); d = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, f in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))]:
    f(); torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); [f() for _ in range(5)]; e.record(); torch.cuda.synchronize()
    print(name, "GB/s", 5 * n / (s.elapsed_time(e) * 1e-3) / 1e9)
PY
} > gpurun_out/box_facts.txt 2>&1
