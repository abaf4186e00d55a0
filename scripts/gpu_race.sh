timeout 900 compute-sanitizer --tool racecheck --print-limit 3 python -m pytest tests/test_gpu_parity.py -q -x -k "perspective_mixed or big_window_waves or rng_ties or config1" 2>&1 | grep -v "^\s*$" | tail -12
timeout 900 compute-sanitizer --tool racecheck --print-limit 3 python -m pytest tests/test_gpu_bicubic.py -q -x 2>&1 | grep -v "^\s*$" | tail -12
