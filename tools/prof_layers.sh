# full captures (with source) of the training layer (backward, KIND 2) and the
# C5 apply layer; each ncu only after the same command exited 0 without it
A="python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $A > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_train_sell -s 10 -c 1 -o gpurun_out/prof_ts_c3 $A > gpurun_out/ncu_ts.log 2>&1
B="python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-fgmres"
timeout 300 $B > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_layer_sell -s 12 -c 1 -o gpurun_out/prof_sell_c5 $B > gpurun_out/ncu_c5.log 2>&1
ls gpurun_out/*.ncu-rep
