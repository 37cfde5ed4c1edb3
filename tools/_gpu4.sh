timeout 300 python tools/phase_tiled.py C2 4 > gpurun_out/phase_c2.log 2>&1
timeout 300 python tools/phase_tiled.py C4 8 8 > gpurun_out/phase_c4.log 2>&1
