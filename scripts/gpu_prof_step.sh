# per-kernel launch list of the bench step (config 5) + source-level capture of one kernel (run under gpurun)
#   KREGEX: kernel regex for the full capture (default: the wide/fallback rest kernel)
set -x
mkdir -p gpurun_out
TAG=${TAG:-step}
KREGEX=${KREGEX:-ctf_collab_rest_kernel}
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:ctf_ -c 40 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-configs > /dev/null 2>&1
python scripts/launch_shares.py gpurun_out/launches_$TAG.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s ${SKIP:-2} -c 1 \
    -o gpurun_out/prof_$TAG python bench.py --frames 64 --warmup 1 --profile-launches 1 > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
