# the r02 captures the first pass missed (demangled names print template args as "(int)32, (bool)1")
mkdir -p gpurun_out
NB="--steps 3 --warmup 3 --no-cpu-baseline --no-fgmres --no-extras"
B="python bench.py --config c5 $NB"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_layer_sell<\(int\)32, \(bool\)1, float" -s 2 -c 1 -o gpurun_out/r02f_prof_c5_last $B > gpurun_out/r02f_ncu_b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_layer_sell<\(int\)32, \(bool\)0, float" -s 14 -c 1 -o gpurun_out/r02f_prof_c5_layer $B > gpurun_out/r02f_ncu_c.log 2>&1
B="python bench.py --config c4 $NB"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_layer_sell<\(int\)16, \(bool\)0, float" -s 14 -c 1 -o gpurun_out/r02f_prof_c4_layer $B > gpurun_out/r02f_ncu_d.log 2>&1
ls -la gpurun_out | grep "r02f_prof"
