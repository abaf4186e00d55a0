mkdir -p gpurun_out
timeout 300 python scripts/time_config3.py 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ctf_collab_lean -s 1 -c 1 -o gpurun_out/prof_c3b python scripts/time_config3.py > gpurun_out/ncu_c3b.log 2>&1
tail -1 gpurun_out/ncu_c3b.log
