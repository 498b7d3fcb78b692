B="python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-fgmres"
$B > gpurun_out/plain_c4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_layer_sell|k_long_chunks" -s 20 -c 2 -o gpurun_out/prof_c4 $B > gpurun_out/ncu_c4.log 2>&1
tail -2 gpurun_out/ncu_c4.log
timeout 300 python -m pytest tests/test_gpu_apply.py tests/test_gpu_fgmres.py tests/test_gpu_sell.py -q -x 2>&1 | tail -4
