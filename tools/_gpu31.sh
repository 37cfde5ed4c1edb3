timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 100 python tools/cold_step.py C2 4 > gpurun_out/cold.log 2>&1
timeout 100 python tools/phase_tiled.py C2 4 > gpurun_out/phase_c2.log 2>&1
timeout 200 python tools/run_config.py C4 8 > gpurun_out/c4.log 2>&1
timeout 100 python tools/run_config.py C3 > gpurun_out/c3.log 2>&1
