# full ncu captures of one C5 non-last layer: pair-union (default) and plain sliced-ELL
B="python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-fgmres --no-extras"
$B > gpurun_out/plain_c5p.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_layer_sell -s 12 -c 1 -o gpurun_out/prof_c5_pair $B > gpurun_out/ncu_c5p.log 2>&1
GNPC_NO_PAIR=1 $B > gpurun_out/plain_c5s.log 2>&1 && GNPC_NO_PAIR=1 ncu --set full --clock-control none --import-source on -k regex:k_layer_sell -s 12 -c 1 -o gpurun_out/prof_c5_sell $B > gpurun_out/ncu_c5s.log 2>&1
ls -la gpurun_out/*.ncu-rep
