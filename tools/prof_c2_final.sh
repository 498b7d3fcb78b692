# C2 fused-apply capture + launch list after the lift / norm changes (ncu after a clean run)
B="python tools/fused_times.py c2"
timeout 300 $B > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_apply_sell -s 1 -c 1 -o gpurun_out/prof_fused_c2 $B > gpurun_out/ncu_f2.log 2>&1
A="python bench.py --steps 20 --warmup 3 --no-cpu-baseline"
timeout 300 $A > gpurun_out/plain_l.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c2.csv $A > gpurun_out/ncu_l.log 2>&1
ls gpurun_out/prof_fused_c2.ncu-rep
