#!/bin/bash
# A/B of the fused-lift first layer on C5 (GNPC_NO_LIFT_FUSE=1 keeps the separate lift kernel)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_strip.py -m gpu -x -q > gpurun_out/lift_tests.log 2>&1
tail -4 gpurun_out/lift_tests.log
for e in 0 1; do
GNPC_NO_LIFT_FUSE=$e timeout 600 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline --no-fgmres > gpurun_out/lift_c5_$e.json 2> gpurun_out/lift_c5_$e.err
python - <<PY
import json
d=json.loads(open('gpurun_out/lift_c5_$e.json').read().strip().splitlines()[-1])
print('nofuse=$e C5', round(d['value'],1), round(d['ms_per_step'],4), round(d['roofline']['frac'],4), 'apply_frac', round(d.get('apply_frac_of_peak',0),4), 'e2e', round(d['e2e']['value'],1), d.get('per_kernel_ms'))
PY
done
