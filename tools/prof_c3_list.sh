A="python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline"
$A > gpurun_out/r02_plain_c3.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_c3.csv $A > /dev/null 2>&1
$A > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_train_sell -s 8 -c 1 -o gpurun_out/r02_prof_c3_tw $A > gpurun_out/r02_ncu_c3tw.log 2>&1
ls gpurun_out | grep r02_
