# C3 step time per variant build (var/<name>.so), two runs each
for v in "$@"; do for r in 1 2; do
GNPC_LIB=$PWD/var/$v.so timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],2))"
done; done
