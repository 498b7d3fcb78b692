#!/bin/bash
# A/B of the length-sorted apply on C4 (GNPC_NO_ROWSORT=1 keeps the natural node order)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sell.py tests/test_gpu_apply.py tests/test_gpu_fullsize.py tests/test_gpu_fgmres.py tests/test_integration.py -m gpu -x -q > gpurun_out/rowsort_tests.log 2>&1
tail -6 gpurun_out/rowsort_tests.log
for e in 0 1; do
GNPC_NO_ROWSORT=$e timeout 600 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/rowsort_c4_$e.json 2> gpurun_out/rowsort_c4_$e.err
python - <<PY
import json
d=json.loads(open('gpurun_out/rowsort_c4_$e.json').read().strip().splitlines()[-1])
print('nosort=$e C4', round(d['value'],1), round(d['ms_per_step'],4), round(d['roofline']['frac'],4), 'apply_frac', round(d.get('apply_frac_of_peak',0),4), 'e2e', round(d['e2e']['value'],1), d.get('per_kernel_ms'), 'fgmres ms/it', d.get('fgmres',{}).get('ms_per_iteration'))
PY
done
