# Round profile set (each ncu only after the same command exited 0 without it):
# default bench line + its launch list, C3 step launch list, full captures of
# the new training kernels (tensor-core decoder backward, encoder interval
# sums, piecewise lift) and the training layer.
set -u
python bench.py > gpurun_out/bench_default.log 2>&1; tail -1 gpurun_out/bench_default.log | head -c 200; echo
A="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
$A > gpurun_out/plain_l.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c2.csv $A > gpurun_out/ncu_l.log 2>&1
C="python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline"
# launches 162.. are the 2 timed steps (3 warm-up steps x 54 launches before them)
$C > gpurun_out/plain_c3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 162 -c 104 --csv --log-file gpurun_out/launches_c3.csv $C > gpurun_out/ncu_c3l.log 2>&1
D="python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline"
for k in k_decoder_tc k_enc_buckets k_lift_pw_batched; do
  $D > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_$k $D > gpurun_out/ncu_$k.log 2>&1
done
ls gpurun_out/*.ncu-rep
