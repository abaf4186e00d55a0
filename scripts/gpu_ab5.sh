timeout 900 python -m pytest tests -m gpu -x -q --timeout=200 2>&1 | tail -3
timeout 300 python scripts/time_small.py variants/*.so 2>&1 | tail -8
timeout 600 python scripts/time_libs.py --frames 32 variants/*.so 2>&1 | tail -4
timeout 600 python scripts/time_libs.py --frames 1 --scene c2 variants/*.so 2>&1 | tail -4
