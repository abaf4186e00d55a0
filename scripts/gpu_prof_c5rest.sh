# ncu: source-level capture of the config-5 lean fallback kernel (16 frames of the camera path),
# and the launch list of one config-4 C+ call (run under gpurun)
set -x
mkdir -p gpurun_out
TAG=${TAG:-c5fb}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ctf_collab_rest_kernel -s 2 -c 1 \
    -o gpurun_out/prof_c5fb_$TAG python bench.py --frames 16 --warmup 1 --profile-launches 1 > gpurun_out/ncu_c5fb_$TAG.log 2>&1
tail -2 gpurun_out/ncu_c5fb_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:ctf_ --csv \
    --log-file gpurun_out/launches_c4_$TAG.csv python scripts/prof_c4.py > /dev/null 2>&1
python scripts/launch_shares.py gpurun_out/launches_c4_$TAG.csv
