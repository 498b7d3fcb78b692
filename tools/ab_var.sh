# bench C5 (or $CFG) with each variant library in var/ (plus the default build)
CFG=${CFG:-c5}
for v in default ${VARS}; do
  if [ $v = default ]; then L=""; else L="GNPC_LIB=var/$v.so"; fi
  env $L timeout 300 python bench.py --config $CFG --steps 20 --warmup 5 --no-cpu-baseline --no-fgmres --no-extras > gpurun_out/var_${CFG}_$v.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/var_${CFG}_$v.log').read().strip().splitlines()[-1])
print('$CFG $v', 'value %.1f'%d['value'], 'frac %.3f'%d['roofline']['frac'], {k: round(v,4) if v else v for k,v in d['per_kernel_ms'].items()})" || tail -3 gpurun_out/var_${CFG}_$v.log
done
