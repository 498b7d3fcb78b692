B="python tools/fused_times.py c5"
$B > gpurun_out/plain_f.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_apply_sell -s 1 -c 1 -o gpurun_out/prof_fused_c5 $B > gpurun_out/ncu_f.log 2>&1
tail -1 gpurun_out/ncu_f.log
