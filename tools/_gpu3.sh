timeout 300 python tools/cold_step.py C2 4 > gpurun_out/cold.log 2>&1
timeout 600 python tools/c5_sweep.py --sizes 4096,16384 --rhos 0.5 --bits 4 > gpurun_out/c5b.log 2>&1
QG_TILED_SMEM_KB=200 timeout 600 python tools/c5_sweep.py --sizes 4096,16384 --rhos 0.5 --bits 4 > gpurun_out/c5c.log 2>&1
