timeout 600 python -m pytest -x -q tests/test_gpu_apply.py tests/test_gpu_sell.py tests/test_gpu_fullsize.py -k "apply or sell or c4" 2>&1 | tail -2
for v in g4 l1; do
  case $v in g4) E="";; l1) E="GNPC_NO_G4=1";; esac
  env $E timeout 300 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline --no-fgmres --no-extras > gpurun_out/g4_c4_$v.log 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/g4_c4_$v.log').read().strip().splitlines()[-1])
print('c4 $v', 'value %.1f'%d['value'], 'frac %.3f'%d['roofline']['frac'], {k: round(v,4) if v else v for k,v in d['per_kernel_ms'].items()})" || tail -5 gpurun_out/g4_c4_$v.log
done
