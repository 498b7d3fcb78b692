# Time variant builds: tools/var_run.sh <config> <name>...  (bench value per variant)
cfg=$1; shift
for v in "$@"; do
  for rep in 1 2; do
  GNPC_LIB=$PWD/var/$v.so timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline --no-fgmres > gpurun_out/var_${cfg}_$v.log 2>&1 || tail -3 gpurun_out/var_${cfg}_$v.log
  python -c "
import json;d=json.loads(open('gpurun_out/var_${cfg}_$v.log').read().strip().splitlines()[-1]);print('$cfg $v',round(d['value'],1),d['unit'],'frac',round(d['roofline']['frac'],3),d.get('per_kernel_ms'))"
  done
done
