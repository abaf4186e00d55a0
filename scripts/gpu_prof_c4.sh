set -x
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg,sm__cycles_elapsed.avg,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:ctf_ --csv python scripts/prof_c4.py > gpurun_out/c4_launches.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ctf_collab_rest -s 8 -c 1 -o gpurun_out/prof_c4rest python scripts/prof_c4.py > /dev/null 2>&1
ls -la gpurun_out
