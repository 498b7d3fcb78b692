B="python bench.py --config c3 --steps 2 --warmup 3"
$B > gpurun_out/plain_w.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_train_sell -s 10 -c 2 -o gpurun_out/prof_trainsell $B > gpurun_out/ncu_w.log 2>&1
tail -1 gpurun_out/ncu_w.log
