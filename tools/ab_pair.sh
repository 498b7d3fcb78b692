# A/B: pair-union slices (default) vs plain sliced-ELL on C5
for v in 0 1; do
  GNPC_NO_PAIR=$v timeout 600 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline --no-fgmres --no-extras > gpurun_out/abp_c5_$v.log 2>&1
  python -c "
import json,sys
d=json.loads(open('gpurun_out/abp_c5_$v.log').read().strip().splitlines()[-1])
print('c5 no_pair=$v', 'value %.1f'%d['value'], 'frac %.3f'%d['roofline']['frac'], d['per_kernel_ms'])" || tail -20 gpurun_out/abp_c5_$v.log
done
