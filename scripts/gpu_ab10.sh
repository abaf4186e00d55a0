timeout 900 python -m pytest tests -m gpu -x -q --timeout=200 2>&1 | tail -2
bash scripts/gpu_ab9.sh
