# ncu source-level capture of the config-3 latent-MLP lean kernel (run under gpurun)
set -x
mkdir -p gpurun_out
TAG=${TAG:-mlp}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-ctf_collab_lean_kernel} -s 1 -c 1 \
    -o gpurun_out/prof_mlp_$TAG python bench.py --profile-config3 2 > gpurun_out/ncu_mlp_$TAG.log 2>&1
tail -2 gpurun_out/ncu_mlp_$TAG.log
