# bench line (no cpu/e2e legs) + ncu launch list of the same command, for per-kernel shares
set -x
mkdir -p gpurun_out
TAG=${TAG:-bq}
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -3 gpurun_out/bench_$TAG.err; python -c "import json;d=json.load(open('gpurun_out/bench_$TAG.json'));print(d['value'],d['roofline']['frac'],d['gpu_launches'],{k:round(v.get('gpix_s',0),2) for k,v in d['configs'].items()})"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ctf_ -c 60 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-configs > gpurun_out/ncu_launch_$TAG.json 2>&1
python scripts/launch_shares.py gpurun_out/launches_$TAG.csv
