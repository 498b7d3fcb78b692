# r02 final profile set (after: fused lift, length-sorted C4): launch lists and
# full captures; every ncu run follows a clean run of the same command
mkdir -p gpurun_out
NB="--steps 3 --warmup 3 --no-cpu-baseline --no-fgmres --no-extras"
for c in c5 c4; do
  B="python bench.py --config $c $NB"
  timeout 600 $B > gpurun_out/r02f_plain_$c.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02f_launches_$c.csv $B > gpurun_out/r02f_ncu_l_$c.log 2>&1
done
B="python bench.py --config c5 $NB"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_layer_sell_lift" -s 2 -c 1 -o gpurun_out/r02f_prof_c5_lift $B > gpurun_out/r02f_ncu_a.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_layer_sell<32, true" -s 2 -c 1 -o gpurun_out/r02f_prof_c5_last $B > gpurun_out/r02f_ncu_b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_layer_sell<32, false" -s 14 -c 1 -o gpurun_out/r02f_prof_c5_layer $B > gpurun_out/r02f_ncu_c.log 2>&1
B="python bench.py --config c4 $NB"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_layer_sell<16, false" -s 14 -c 1 -o gpurun_out/r02f_prof_c4_layer $B > gpurun_out/r02f_ncu_d.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_long_chunks" -s 14 -c 1 -o gpurun_out/r02f_prof_c4_chunks $B > gpurun_out/r02f_ncu_e.log 2>&1
ls -la gpurun_out | grep r02f
