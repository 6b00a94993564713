#!/bin/bash
# compute-sanitizer over a small GPU test subset that exercises every kernel
# family (projection, binning, tile sort, the NP=2 evaluation/usage
# compositing kernel, the seam / record kernels, SSE): memcheck, racecheck
# (shared-memory hazards), synccheck (barrier misuse).  Outputs under
# gpurun_out/sanitizer_*.txt.   tools/sanitize.sh
mkdir -p gpurun_out
SEL="render_with_usage_matches_oracle or render_single_view or seam_forward_matches_oracle or psnr_device or render_bucket_overflow"
for tool in memcheck racecheck synccheck; do
  echo "\$ compute-sanitizer --tool $tool python -m pytest tests/test_gpu_render.py -m gpu -q -k \"$SEL\"" > gpurun_out/sanitizer_$tool.txt
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 \
    python -m pytest tests/test_gpu_render.py -m gpu -q -p no:cacheprovider -k "$SEL" >> gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitizer_$tool.txt
done
