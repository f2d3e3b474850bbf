timeout 600 python tools/copy_interference.py 2>&1 | tail -8
