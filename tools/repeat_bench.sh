for i in 1 2 3 4 5 6 7 8 9 10; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/rep_$i.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/rep_$i.json').read().strip().splitlines()[-1]); print('run $i', d['value'], d['ms_per_step'], d['roofline']['timing_pass']['ms_per_step'], d['e2e']['value'])"
done
