# windowed sliced-ELL (d = 16): GPU parity tests, then C2 bench with and without windows
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for w in 0 1; do
  GNPC_NO_WIN=$w timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-fgmres > gpurun_out/c2w$w.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/c2w$w.log').read().strip().splitlines()[-1]);print('no_win=$w', round(d['value'],1), round(d['ms_per_step']*1e3,1), 'us frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), d['per_kernel_ms'])" || tail -5 gpurun_out/c2w$w.log
done
