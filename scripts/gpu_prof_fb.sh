# ncu --set full of the three BC1 COLLAB kernels of one 64-frame bench step
set -x
mkdir -p gpurun_out
TAG=${TAG:-pf}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ctf_collab_ -s 3 -c 3 \
    -o gpurun_out/prof_$TAG python bench.py --warmup 1 --profile-launches 1 > gpurun_out/ncu_full_$TAG.log 2>&1
tail -2 gpurun_out/ncu_full_$TAG.log
