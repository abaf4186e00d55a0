# quick iteration on one B200: gpu tests, short bench (no cpu / e2e legs), ncu of the lean kernel
set -x
mkdir -p gpurun_out
TAG=${TAG:-q}
if [ "${TESTS:-1}" = "1" ]; then
  timeout 600 python -m pytest tests -m gpu -x -q --timeout=120 2>&1 | tail -15
fi
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -3 gpurun_out/bench_$TAG.err; python -c "import json;d=json.load(open('gpurun_out/bench_$TAG.json'));print(d['value'],d['roofline']['frac'],{k:round(v.get('gpix_s',0),2) for k,v in d['configs'].items()})"
if [ "${NCU:-1}" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ctf_collab_ -s 6 -c 2 \
    -o gpurun_out/prof_$TAG python bench.py --frames 16 --warmup 3 --profile-launches 1 > gpurun_out/ncu_full_$TAG.log 2>&1
tail -3 gpurun_out/ncu_full_$TAG.log
fi
