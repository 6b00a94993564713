#!/bin/bash
# compute-sanitizer over small GPU test subsets that exercise every kernel
# family of the path: projection, binning, tile sorts, the NP=2 evaluation /
# usage compositing kernel, the seam / record kernels, SSE (test_gpu_render),
# the GSDP decode + apply kernels, the streamed and pipelined probes
# (test_gpu_codec_delta, test_gpu_pruning_grouping): memcheck, racecheck
# (shared-memory hazards), synccheck (barrier misuse).
# Outputs under gpurun_out/sanitizer_*.txt.   tools/sanitize.sh
mkdir -p gpurun_out
SEL="render_with_usage_matches_oracle or render_single_view or seam_forward_matches_oracle or psnr_device or render_bucket_overflow"
SEL2="probe_sequence or probe_payloads or decode_apply or gsdp"
for tool in memcheck racecheck synccheck; do
  out=gpurun_out/sanitizer_$tool.txt
  echo "\$ compute-sanitizer --tool $tool python -m pytest tests/test_gpu_render.py -m gpu -q -k \"$SEL\"" > $out
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 \
    python -m pytest tests/test_gpu_render.py -m gpu -q -p no:cacheprovider -k "$SEL" >> $out 2>&1
  echo "$tool (render) rc=$?"; tail -2 $out
  echo "\$ compute-sanitizer --tool $tool python -m pytest tests/test_gpu_codec_delta.py tests/test_gpu_pruning_grouping.py -m gpu -q -k \"$SEL2\"" >> $out
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 \
    python -m pytest tests/test_gpu_codec_delta.py tests/test_gpu_pruning_grouping.py -m gpu -q -p no:cacheprovider \
    -k "$SEL2" >> $out 2>&1
  echo "$tool (decode/probe) rc=$?"; tail -2 $out
done
