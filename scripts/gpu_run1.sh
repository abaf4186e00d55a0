set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q --timeout=120 2>&1 | tail -4
timeout 600 python scripts/time_libs.py --frames 32 variants/a_base.so variants/b_new.so 2>&1 | tail -3
timeout 600 python scripts/time_libs.py --frames 8 --scene c4 variants/a_base.so variants/b_new.so 2>&1 | tail -3
timeout 300 python scripts/time_small.py 2>&1 | tail -8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ctf_ -s 4 -c 1 -o gpurun_out/prof_c2a python scripts/prof_c2.py > gpurun_out/ncu_c2a.log 2>&1
tail -2 gpurun_out/ncu_c2a.log
