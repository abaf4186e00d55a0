timeout 900 python -m pytest tests -m gpu -x -q --timeout=200 2>&1 | tail -2
bash scripts/gpu_ab9.sh
timeout 900 compute-sanitizer --tool racecheck --print-limit 5 python -m pytest tests/test_gpu_parity.py -q -x -k "perspective_mixed or big_window_waves or rng_ties" 2>&1 | tail -3
timeout 900 compute-sanitizer --tool racecheck --print-limit 5 python -m pytest tests/test_gpu_bicubic.py -q -x -k "ragged or random_uv" 2>&1 | tail -3
