# A/B: tile order (GNPC_TORDER) x L2 policy (GNPC_L2HINT) on the apply configs
for c in ${CFGS:-c5 c4 c2}; do
  for to in 1 0; do for l2 in 1 0; do
    GNPC_TORDER=$to GNPC_L2HINT=$l2 timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-fgmres --no-extras > gpurun_out/ab_${c}_t${to}_h${l2}.log 2>&1
    python - "$c" "$to" "$l2" gpurun_out/ab_${c}_t${to}_h${l2}.log <<'PY'
import json,sys
c,to,l2,f=sys.argv[1:]
try:
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(c,"torder",to,"l2hint",l2,"value %.1f"%d["value"],"frac %.3f"%d["roofline"]["frac"],d["per_kernel_ms"])
except Exception as e:
    print(c,to,l2,"FAILED",open(f).read()[-500:])
PY
  done; done
done
