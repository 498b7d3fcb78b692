B="python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-fgmres --no-extras"
timeout 300 $B > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_apply_sell<\(int\)16, float" -s 3 -c 1 -o gpurun_out/r02f_prof_c2_fused $B > gpurun_out/r02f_ncu_c2.log 2>&1
ls -la gpurun_out/r02f_prof_c2_fused.ncu-rep
