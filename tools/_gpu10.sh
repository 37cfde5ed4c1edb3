timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/cold_step.py C2 4 > gpurun_out/cold.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_tiled -c 2 -o gpurun_out/c4_tiled python tools/phase_tiled.py C4 8 8 > gpurun_out/ncu_c4.log 2>&1
timeout 300 python tools/phase_tiled.py C4 8 8 > gpurun_out/phase_c4.log 2>&1
