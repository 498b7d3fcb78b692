B="python bench.py --config c3 --steps 16 --warmup 3 --no-cpu-baseline"
timeout 300 $B > gpurun_out/plain_late.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 900 -c 108 --csv --log-file gpurun_out/launches_c3_late.csv $B > gpurun_out/ncu_late.log 2>&1
