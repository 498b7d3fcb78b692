B="python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline"
timeout 300 $B > gpurun_out/plain_enc.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KERN:-k_enc_buckets} -s 1 -c 1 -o gpurun_out/prof_${KERN:-enc} $B > gpurun_out/ncu_enc.log 2>&1
tail -2 gpurun_out/ncu_enc.log
