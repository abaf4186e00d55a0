# A/B on one B200: interleaved timing of variants/*.so (c5, c4) + per-kernel instruction counts
# (ncu, one 16-frame call per library: warp-instructions per wave of the lean and rest kernels)
set -x
mkdir -p gpurun_out
LIBS=${LIBS:-variants/*.so}
if [ "${TESTS:-0}" = "1" ]; then
  timeout 600 python -m pytest tests -m gpu -x -q --timeout=120 2>&1 | tail -4
fi
timeout 600 python scripts/time_libs.py --frames 32 $LIBS 2>&1 | tail -8
timeout 600 python scripts/time_libs.py --frames 8 --scene c4 $LIBS 2>&1 | tail -8
for l in $LIBS; do
  timeout 300 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:ctf_collab -c 3 --csv \
     python scripts/time_libs.py --frames 16 --rounds 1 --reps 1 $l 2>/dev/null | python scripts/ncu_inst_per_wave.py $l 16
done
