# trained GNP at full size (C4, C5) + C1 profile set
timeout 1500 python tools/r2_trained_scale.py c4 600 16 300 > gpurun_out/r02_trained_c4.log 2>&1; tail -1 gpurun_out/r02_trained_c4.log | head -c 1500; echo
timeout 2400 python tools/r2_trained_scale.py c5 300 8 500 > gpurun_out/r02_trained_c5.log 2>&1; tail -1 gpurun_out/r02_trained_c5.log | head -c 1500; echo
B="python bench.py --config c1 --steps 20 --warmup 5 --no-cpu-baseline"
$B > gpurun_out/r02_c1.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_c1.csv $B > /dev/null 2>&1
$B > /dev/null 2>&1 && timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_apply_sell -s 5 -c 1 -o gpurun_out/r02_prof_c1 $B > gpurun_out/r02_ncu_c1.log 2>&1
tail -1 gpurun_out/r02_c1.log | head -c 600
