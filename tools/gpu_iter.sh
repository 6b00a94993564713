#!/bin/bash
# One GPU iteration: parity tests (-m gpu, optional filter), the launch list of
# one C2 step, and optionally a full ncu capture of k_composite.
#   tools/gpu_iter.sh TAG [pytest -k expr] [full]
TAG=$1; K=${2:-}; FULL=${3:-}
mkdir -p gpurun_out
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest=$?"
else
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest=$?"
fi
tail -3 gpurun_out/pytest_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_$TAG.csv python tools/step_once.py --reps 1 > gpurun_out/ncu1_$TAG.log 2>&1
echo "ncu1=$?"
python tools/launches.py gpurun_out/launches_$TAG.csv | head -12
if [ -n "$FULL" ]; then
  timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_composite -c 1 \
    -o gpurun_out/prof_composite_$TAG -f python tools/step_once.py --reps 1 > gpurun_out/ncu2_$TAG.log 2>&1
  echo "ncu2=$?"
fi
