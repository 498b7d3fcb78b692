set -e
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in c2 c4 c5; do timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-fgmres > gpurun_out/q_$c.log 2>&1 || tail -5 gpurun_out/q_$c.log; python -c "
import json;d=json.loads(open('gpurun_out/q_$c.log').read().strip().splitlines()[-1]);print('$c',round(d['value'],1),d['unit'],'frac',round(d['roofline']['frac'],3),d['per_kernel_ms'], 'e2e', round(d['e2e']['value'],1))"; done
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 > gpurun_out/q_c3.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/q_c3.log').read().strip().splitlines()[-1]);print('c3',round(d['value'],2),d['ms_per_step'])"
