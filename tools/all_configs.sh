# one bench line per config (C2 is the default line; FGMRES legs included)
for c in c1 c2 c4 c5; do timeout 900 python bench.py --config $c --steps 30 --warmup 5 > gpurun_out/all_$c.log 2>&1; tail -1 gpurun_out/all_$c.log | cut -c1-150; done
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 > gpurun_out/all_c3.log 2>&1; tail -1 gpurun_out/all_c3.log | cut -c1-150
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/all_ref.log 2>&1; tail -1 gpurun_out/all_ref.log | cut -c1-300
