timeout 300 python scripts/time_small.py variants/*.so 2>&1 | tail -16
