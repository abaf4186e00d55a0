mkdir -p gpurun_out
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:ctf_ -s 4 -c 1 -o gpurun_out/prof_c2b python scripts/prof_c2.py > gpurun_out/ncu_c2b.log 2>&1
tail -2 gpurun_out/ncu_c2b.log
