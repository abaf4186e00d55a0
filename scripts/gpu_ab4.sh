set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout=200 2>&1 | tail -3
timeout 600 python scripts/time_libs.py --frames 32 variants/*.so 2>&1 | tail -4
timeout 600 python scripts/time_libs.py --frames 1 --scene c4 variants/*.so 2>&1 | tail -4
timeout 300 python scripts/time_small.py variants/*.so 2>&1 | tail -16
