A="python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline"
$A > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_train_sell -s 8 -c 1 -o gpurun_out/r02_prof_c3_fwd $A > gpurun_out/r02_ncu_c3f.log 2>&1
ls -la gpurun_out/r02_prof_c3_fwd.ncu-rep
