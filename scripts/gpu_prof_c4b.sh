mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__occupancy_limit_shared_mem --clock-control none -k regex:ctf_ --csv python scripts/prof_c4.py > gpurun_out/c4b_launches.csv 2>&1
