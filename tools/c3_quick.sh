# C3 training: parity tests + bench line + launch list (ncu only after the plain run exits 0)
timeout 600 python -m pytest tests/test_gpu_train.py tests/test_gpu_sampler.py -q -x 2>&1 | tail -3
A="python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline"
timeout 300 $A > gpurun_out/c3q.log 2>&1 && python -c "
import json;d=json.loads(open('gpurun_out/c3q.log').read().strip().splitlines()[-1]);print('c3', round(d['value'],2), d['ms_per_step'])"
B="python bench.py --config c3 --steps 2 --warmup 3"
timeout 300 $B > gpurun_out/plain_c3.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 150 -c 200 --csv --log-file gpurun_out/launches_c3.csv $B > gpurun_out/ncu_c3l.log 2>&1
