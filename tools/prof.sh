set -x
python bench.py > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log | head -c 600; echo
A="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
$A > gpurun_out/plain_l.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv $A > gpurun_out/ncu_l.log 2>&1
for c in c2 c5; do
B="python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-fgmres"
$B > gpurun_out/plain_$c.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_layer_sell -s 12 -c 1 -o gpurun_out/prof_sell_$c $B > gpurun_out/ncu_$c.log 2>&1
done
ls gpurun_out
