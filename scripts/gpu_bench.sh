# tests + bench + ncu evidence on one B200 (run under gpurun from the repo root)
set -x
mkdir -p gpurun_out
TAG=${TAG:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
if [ "${TESTS:-1}" = "1" ]; then
  timeout 600 python -m pytest tests -m gpu -x -q --timeout=120 2>&1 | tail -15
fi
timeout 900 python bench.py --steps ${STEPS:-20} --warmup 3 --cpu-seconds ${CPUS:-12} > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -5 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
# launch list of the same command (cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ctf_ -c 60 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-configs > gpurun_out/ncu_launch_bench_$TAG.json 2>&1
python scripts/launch_shares.py gpurun_out/launches_$TAG.csv
# one full capture of the three BC1 COLLAB kernels of one 64-frame step (the bench step)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:ctf_collab_ -s 3 -c 3 \
    -o gpurun_out/prof_$TAG python bench.py --warmup 1 --profile-launches 1 > gpurun_out/ncu_full_$TAG.log 2>&1
tail -3 gpurun_out/ncu_full_$TAG.log
if [ "${MLPPROF:-0}" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ctf_collab_lean_kernel -s 1 -c 1 \
    -o gpurun_out/prof_mlp_$TAG python bench.py --profile-config3 2 > gpurun_out/ncu_mlp_$TAG.log 2>&1
tail -2 gpurun_out/ncu_mlp_$TAG.log
fi
