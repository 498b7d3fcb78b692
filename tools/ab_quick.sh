#!/bin/bash
# quick per-config bench lines (no CPU baseline / FGMRES): tools/ab_quick.sh c5 c4 c2
for c in "$@"; do
timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-fgmres > gpurun_out/q_$c.json 2> gpurun_out/q_$c.err
python - <<PY
import json
d=json.loads(open('gpurun_out/q_$c.json').read().strip().splitlines()[-1])
print('$c', round(d['value'],1), d['unit'], round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],4), 'apply_frac', round(d.get('apply_frac_of_peak',0),4), 'e2e', round(d['e2e']['value'],1), d.get('per_kernel_ms'))
PY
done
