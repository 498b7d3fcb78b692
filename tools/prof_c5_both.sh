B="python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-fgmres --no-extras"
$B > gpurun_out/plain_c5b.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_layer_sell -s 14 -c 2 -o gpurun_out/prof_c5_both $B > gpurun_out/ncu_c5b.log 2>&1
ls -la gpurun_out/*.ncu-rep
