#!/bin/bash
# Time each built variant with a short bench run: tools/ab.sh name1 name2 ...
# (AB_CONFIG=C5 tools/ab.sh ... for another BASELINE config)
mkdir -p gpurun_out
CFG=${AB_CONFIG:-C2}
for v in "$@"; do
  if [ "$v" = "main" ]; then L=""; else L=paper_2512_20943_b200/lib/variants/$v.so; fi
  AIRGS_B200_LIB=$L timeout 600 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err
  python -c "
import json,sys; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1])
c=d.get('clocks',{})
st=d['roofline']['stages']
print('$v $CFG', d['value'], 'views/s  step ms', d['ms_per_step'], ' '.join('%s %.4f' % (k, v['ms_per_step']) for k, v in st.items()), ' q0', d['qualities_db'][0], ' sm_mhz', c.get('sm_mhz'), c.get('reasons'))" || tail -3 gpurun_out/ab_$v.err
done
