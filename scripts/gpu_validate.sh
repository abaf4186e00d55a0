# re-validate HEAD on one B200 (tests, smoke, bench) and sweep the e2e chunk size
set -x
mkdir -p gpurun_out
TAG=${TAG:-v}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q --timeout=180 2>&1 | tail -8
timeout 900 python bench.py --steps 20 --warmup 3 --cpu-seconds 12 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
for c in 2 4; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-configs --e2e-chunk $c 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('chunk', $c, d['value'], d['e2e']['value'], d['e2e']['link_frac'])"
done
