timeout 300 python scripts/prof_bicubic.py variants/*.so 2>&1 | tail -12
