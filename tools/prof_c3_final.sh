# C3 launch list (the two timed steps) + training-layer captures (fwd and bwd)
C="python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 300 $C > gpurun_out/plain_c3.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 162 -c 104 --csv --log-file gpurun_out/launches_c3.csv $C > gpurun_out/ncu_c3l.log 2>&1
D="python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $D > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_train_sell -s 10 -c 1 -o gpurun_out/prof_ts_bwd $D > gpurun_out/ncu_tsb.log 2>&1
timeout 300 $D > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_train_sell -s 1 -c 1 -o gpurun_out/prof_ts_fwd $D > gpurun_out/ncu_tsf.log 2>&1
C5="python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-fgmres"
timeout 300 $C5 > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_layer_sell -s 12 -c 1 -o gpurun_out/prof_sell_c5 $C5 > gpurun_out/ncu_c5.log 2>&1
ls gpurun_out/*.ncu-rep
