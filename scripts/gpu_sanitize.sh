# compute-sanitizer passes (memcheck / racecheck / synccheck / initcheck) over small GPU parity
# cases of every kernel family (run under gpurun)
set -x
mkdir -p gpurun_out
TAG=${TAG:-r02}
SEL="config1_uniform_4x and 1-30 or tiny_frames or clustered or latent_mlp_texture or full_waves_at_texture_borders or (workspace_lists and 3-0) or release_paired_runs or multi_frame_work_lists or mask_and_box_variants or (release_kernel_matches_oracle and (4- or 5- or 6-)) or rng_ties or (big_window_waves and (9.0 or 7.5))"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 3 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py -q -x -k "$SEL" > gpurun_out/sanitize_${tool}_$TAG.log 2>&1
  echo "$tool parity exit=$?"
  tail -3 gpurun_out/sanitize_${tool}_$TAG.log
  # r02 kernels: fused single launch, wide-window bitmaps, bicubic bitmap collect, strips
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 3 --print-limit 20 \
    python -m pytest tests/test_gpu_fused.py tests/test_gpu_bicubic.py tests/test_gpu_sharding.py -q -x \
      -k "grazing or camera0 or ragged or perspective or (strips and 2) or latent" > gpurun_out/sanitize_${tool}_r02kernels_$TAG.log 2>&1
  echo "$tool r02-kernels exit=$?"
  tail -3 gpurun_out/sanitize_${tool}_r02kernels_$TAG.log
done
