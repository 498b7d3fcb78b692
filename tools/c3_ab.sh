# C3 training: parity tests, then the bench line with and without the
# piecewise encoder (GNPC_NO_PW_ENCODER=1 selects the MLP kernels)
timeout 600 python -m pytest tests/test_gpu_train.py tests/test_gpu_sampler.py -q -x 2>&1 | tail -3
for v in 0 1; do
  GNPC_NO_PW_ENCODER=$v timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c3_pw$v.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/c3_pw$v.log').read().strip().splitlines()[-1]);print('no_pw=$v', round(d['value'],2), d['ms_per_step'])" || tail -5 gpurun_out/c3_pw$v.log
done
