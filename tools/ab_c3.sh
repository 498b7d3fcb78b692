# C3 training step A/B over variant libraries (default build first)
for v in default ${VARS}; do
  if [ $v = default ]; then L=""; else L="GNPC_LIB=var/$v.so"; fi
  env $L timeout 600 python bench.py --config c3 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/c3_$v.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/c3_$v.log').read().strip().splitlines()[-1])
print('c3 $v', 'value %.2f'%d['value'], 'ms %.3f'%d['ms_per_step'], 'frac %.3f'%d['roofline']['frac'], 'clocks', d.get('clocks',{}).get('reasons'))" || tail -3 gpurun_out/c3_$v.log
done
