# r01 profile set: default bench line, its launch list, full captures of the
# dominant kernels (each ncu only after the same command exited 0 without it)
python bench.py > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log | head -c 300; echo
A="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
$A > gpurun_out/plain_l.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c2.csv $A > gpurun_out/ncu_l.log 2>&1
B="python tools/fused_times.py c2"
$B > gpurun_out/plain_f2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_apply_sell -s 1 -c 1 -o gpurun_out/prof_fused_c2 $B > gpurun_out/ncu_f2.log 2>&1
for c in c5 c4; do
B="python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-fgmres"
$B > gpurun_out/plain_$c.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_layer_sell -s 12 -c 1 -o gpurun_out/prof_sell_$c $B > gpurun_out/ncu_$c.log 2>&1
done
ls gpurun_out | head -30
