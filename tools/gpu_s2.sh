set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
bash tools/gpu_iter.sh s2a "" full
timeout 900 python bench.py > gpurun_out/bench_s2a.json 2> gpurun_out/bench_s2a.err; echo bench=$?
tail -c 3000 gpurun_out/bench_s2a.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_s2a.json 2>&1; echo ref=$?
cat gpurun_out/ref_s2a.json | tail -c 1500
