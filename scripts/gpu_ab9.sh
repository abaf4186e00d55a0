timeout 600 python scripts/time_libs.py --frames 32 variants/*.so 2>&1 | tail -3
timeout 600 python scripts/time_libs.py --frames 1 --scene c4 variants/*.so 2>&1 | tail -3
timeout 600 python scripts/time_libs.py --frames 8 --scene c4 variants/*.so 2>&1 | tail -3
for l in variants/*.so; do
  timeout 300 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:ctf_collab -c 3 --csv \
     python scripts/time_libs.py --frames 16 --rounds 1 --reps 1 $l 2>/dev/null | python scripts/ncu_inst_per_wave.py $l 16
done
