timeout 900 python -m pytest tests -m gpu -x -q --timeout=200 2>&1 | tail -2
timeout 300 python scripts/prof_bicubic.py variants/*.so 2>&1 | tail -8
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bicubic -c 1 -o gpurun_out/prof_bic2 python scripts/prof_bicubic.py > /dev/null 2>&1
