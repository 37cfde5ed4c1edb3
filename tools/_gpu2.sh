timeout 600 python tools/c5_sweep.py --sizes 1024,4096,16384 --rhos 0.01,0.5 --bits 1,8 > gpurun_out/c5.log 2>&1
timeout 300 python tools/e2e_breakdown.py C2 4 > gpurun_out/e2e.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_tiled -c 1 -o gpurun_out/c5_8k python tools/c5_sweep.py --sizes 8192 --rhos 0.1 --bits 4 --reps 1 > gpurun_out/ncu_c5.log 2>&1
tail -5 gpurun_out/ncu_c5.log
