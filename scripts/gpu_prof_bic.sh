mkdir -p gpurun_out
timeout 300 python scripts/prof_bicubic.py 2>&1 | tail -4
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ctf_ -s 1 -c 1 -o gpurun_out/prof_bic python scripts/prof_bicubic.py > gpurun_out/ncu_bic.log 2>&1
tail -1 gpurun_out/ncu_bic.log
