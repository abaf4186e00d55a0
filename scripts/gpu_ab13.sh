timeout 900 python -m pytest tests -m gpu -x -q --timeout=200 2>&1 | tail -2
timeout 300 python scripts/prof_bicubic.py variants/a_base.so variants/b_bic.so 2>&1 | tail -8
for l in variants/*.so; do
timeout 300 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:bicubic -c 1 --csv python scripts/prof_bicubic.py $l 2>/dev/null | python scripts/ncu_inst_per_wave.py $l 1 | head -2
done
