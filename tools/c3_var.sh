for v in base nomb base nomb; do GNPC_LIB=$PWD/var/$v.so timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],2))"; done
B="python bench.py --config c3 --steps 2 --warmup 3"
GNPC_LIB=$PWD/var/nomb.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 150 -c 200 --csv --log-file gpurun_out/launches_c3_nomb.csv $B > /dev/null 2>&1
