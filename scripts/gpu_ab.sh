# A/B: gpu tests on the in-tree lib, then interleaved timing of variants/*.so (c5 and c4 scenes)
set -x
mkdir -p gpurun_out
TAG=${TAG:-ab}
if [ "${TESTS:-1}" = "1" ]; then
  timeout 600 python -m pytest tests -m gpu -x -q --timeout=120 2>&1 | tail -8
fi
timeout 600 python scripts/time_libs.py --frames 32 ${LIBS:-variants/*.so} 2>&1 | tail -8
timeout 600 python scripts/time_libs.py --frames 8 --scene c4 ${LIBS:-variants/*.so} 2>&1 | tail -8
if [ "${NCU:-1}" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ctf_collab_ -s 6 -c 2 \
    -o gpurun_out/prof_$TAG python bench.py --frames 16 --warmup 3 --profile-launches 1 > gpurun_out/ncu_full_$TAG.log 2>&1
tail -2 gpurun_out/ncu_full_$TAG.log
fi
