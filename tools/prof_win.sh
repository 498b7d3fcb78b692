B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fgmres"
GNPC_NO_FUSED_APPLY=1 timeout 300 $B > /dev/null 2>&1 && GNPC_NO_FUSED_APPLY=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_layer_sell -s 12 -c 1 -o gpurun_out/prof_win_c2 $B > gpurun_out/ncu_win.log 2>&1
GNPC_NO_WIN=1 GNPC_NO_FUSED_APPLY=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_layer_sell -s 12 -c 1 -o gpurun_out/prof_nowin_c2 $B > gpurun_out/ncu_nowin.log 2>&1
ls gpurun_out/*win*
