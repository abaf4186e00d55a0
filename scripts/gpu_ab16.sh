timeout 900 python -m pytest tests -m gpu -x -q --timeout=200 2>&1 | tail -2
timeout 300 python scripts/prof_bicubic.py variants/*.so 2>&1 | tail -8
