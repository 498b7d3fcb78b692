# strip-window parity first (bounded), then the C5 A/B: strip windows / pair-union / plain sliced-ELL
timeout 300 python -m pytest -x -q tests/test_gpu_strip.py 2>&1 | tail -15
for v in pw pair sell; do
  case $v in pw) E="";; pair) E="GNPC_NO_PW=1";; sell) E="GNPC_NO_PW=1 GNPC_NO_PAIR=1";; esac
  env $E timeout 300 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline --no-fgmres --no-extras > gpurun_out/abw_c5_$v.log 2>&1
  python -c "
import json,sys
d=json.loads(open('gpurun_out/abw_c5_$v.log').read().strip().splitlines()[-1])
print('c5 $v', 'value %.1f'%d['value'], 'frac %.3f'%d['roofline']['frac'], d['per_kernel_ms'])" || tail -5 gpurun_out/abw_c5_$v.log
done
