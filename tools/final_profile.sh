#!/bin/bash
# Round-end evidence in one GPU call (run from the repo root via gpurun):
# bench line, reference arm, ncu launch list of the bench command, a full ncu
# capture of k_composite and of the other step kernels, summaries.
#   tools/final_profile.sh TAG
TAG=${1:-final}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench=$?"
timeout 900 python bench.py --impl reference > gpurun_out/ref_$TAG.json 2> gpurun_out/ref_$TAG.err; echo "ref=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu1_$TAG.log 2>&1; echo "ncu1=$?"
python tools/launches.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_summary_$TAG.txt
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_composite -c 1 \
  -o gpurun_out/prof_composite_$TAG -f python tools/step_once.py --reps 1 > gpurun_out/ncu2_$TAG.log 2>&1; echo "ncu2=$?"
timeout 900 ncu --set full --clock-control none --profile-from-start off -k "regex:k_project|k_bin|k_sort_tiles|k_gsdp_da" -c 7 \
  -o gpurun_out/prof_others_$TAG -f python tools/step_once.py --reps 1 > gpurun_out/ncu3_$TAG.log 2>&1; echo "ncu3=$?"
python tools/ncu_summary.py gpurun_out/prof_composite_$TAG.ncu-rep 40 --traffic-json gpurun_out/composite_traffic_$TAG.json \
  > gpurun_out/composite_ncu_$TAG.txt 2>&1
tail -c 600 gpurun_out/bench_$TAG.json
python tools/ncu_details.py gpurun_out/prof_others_$TAG.ncu-rep > gpurun_out/others_ncu_$TAG.txt 2>&1
