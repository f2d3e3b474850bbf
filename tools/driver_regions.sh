#!/bin/bash
# driver cost alone (workers skip tiles) and its region profile
python tools/driver_cost.py 2>&1 | grep flags
python tools/profile_run.py --no-tiles --out gpurun_out/prof_nt.json > /dev/null 2>&1
python tools/chain.py gpurun_out/prof_nt.npy
python -c "
import json; d=json.load(open('gpurun_out/prof_nt.json'))['driver']
for k,v in sorted(d.items(), key=lambda x:-x[1]['us'])[:16]: print(k, v['n'], round(v['us']), round(v['us']/max(v['n'],1),2))
"
