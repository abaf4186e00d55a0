# compute-sanitizer passes over small GPU parity cases (run under gpurun)
set -x
mkdir -p gpurun_out
TAG=${TAG:-r01}
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 3 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py -q -x -k "config1_uniform_4x and 1-30 or tiny_frames or clustered or latent_mlp_texture or full_waves_at_texture_borders or (workspace_lists and 3-0) or release_paired_runs or multi_frame_work_lists or mask_and_box_variants or (release_kernel_matches_oracle and (4- or 5- or 6-))" \
    > gpurun_out/sanitize_${tool}_$TAG.log 2>&1
  echo "$tool exit=$?"
  tail -4 gpurun_out/sanitize_${tool}_$TAG.log
done
