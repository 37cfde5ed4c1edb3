timeout 300 python tools/phase_tiled.py C2 4 > gpurun_out/phase_c2.log 2>&1
QG_FUSED_EPOCH=0 timeout 300 python tools/phase_tiled.py C2 4 > gpurun_out/phase_c2_nofuse.log 2>&1
