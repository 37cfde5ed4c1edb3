QG_SCREEN=0 timeout 300 python tools/phase_tiled.py C4 8 8 > gpurun_out/phase_c4_noscreen.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_tiled -c 2 -o gpurun_out/c4_screen python tools/phase_tiled.py C4 8 8 > gpurun_out/ncu_c4.log 2>&1
QG_SCREEN=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_tiled -c 2 -o gpurun_out/c4_noscreen python tools/phase_tiled.py C4 8 8 > gpurun_out/ncu_c4b.log 2>&1
