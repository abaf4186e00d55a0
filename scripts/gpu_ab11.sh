timeout 900 python -m pytest tests -m gpu -x -q --timeout=200 2>&1 | tail -2
timeout 600 python scripts/time_libs.py --frames 32 variants/*.so 2>&1 | tail -3
timeout 600 python scripts/time_libs.py --frames 1 --scene c4 variants/*.so 2>&1 | tail -3
timeout 600 python scripts/time_libs.py --frames 1 --scene c4 --fb 0 variants/*.so 2>&1 | tail -3
timeout 600 python scripts/time_libs.py --frames 8 --scene c4 variants/*.so 2>&1 | tail -3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ctf_ --csv python scripts/prof_c4.py > gpurun_out/c4conc.csv 2>&1
