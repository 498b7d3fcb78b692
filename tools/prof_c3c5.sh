# r01 launch lists for C3 (training step) and C5 (apply), plus full captures of
# the training layer and the weight-gradient reduction. Each ncu only after the
# same command exited 0 without it.
set -u
A="python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline"
$A > gpurun_out/plain_c3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv $A > gpurun_out/ncu_c3l.log 2>&1
tail -1 gpurun_out/plain_c3.log | cut -c1-400; echo
B="python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-fgmres"
$B > gpurun_out/plain_c5.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c5.csv $B > gpurun_out/ncu_c5l.log 2>&1
tail -1 gpurun_out/plain_c5.log | cut -c1-400; echo
$A > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_train_sell -s 10 -c 1 -o gpurun_out/prof_trainsell_c3 $A > gpurun_out/ncu_ts.log 2>&1
$A > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_wgrad_bf16 -s 6 -c 1 -o gpurun_out/prof_wgrad_c3 $A > gpurun_out/ncu_wg.log 2>&1
ls gpurun_out | head -40
