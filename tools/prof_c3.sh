A="python bench.py --config c3 --steps 2 --warmup 3"
$A > gpurun_out/plain_c3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 150 -c 200 --csv --log-file gpurun_out/launches_c3.csv $A > gpurun_out/ncu_c3l.log 2>&1
tail -1 gpurun_out/plain_c3.log | cut -c1-300
