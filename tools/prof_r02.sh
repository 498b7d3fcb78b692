# r02 profile set: default bench line, reference arm, C5 launch list, full capture of the C5 layer
timeout 1200 python bench.py > gpurun_out/r02_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r02_bench.log | head -c 400; echo
timeout 900 python bench.py --impl reference > gpurun_out/r02_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/r02_ref.log | head -c 400; echo
B="python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-fgmres --no-extras"
$B > gpurun_out/r02_plain_c5.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_c5.csv $B > gpurun_out/r02_ncu_l.log 2>&1
$B > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_layer_sell -s 12 -c 1 -o gpurun_out/r02_prof_c5_layer $B > gpurun_out/r02_ncu_f.log 2>&1
ls gpurun_out/ | grep r02
