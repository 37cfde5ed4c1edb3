timeout 300 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
timeout 120 python tools/cold_step.py C2 4 > gpurun_out/cold.log 2>&1
timeout 120 python tools/phase_tiled.py C4 8 8 > gpurun_out/phase_c4.log 2>&1
timeout 200 python tools/run_config.py C4 8 > gpurun_out/c4.log 2>&1
timeout 120 python tools/run_config.py C3 > gpurun_out/c3.log 2>&1
timeout 200 python tools/c5_sweep.py --sizes 4096,16384 --rhos 0.1 --bits 4 > gpurun_out/c5.log 2>&1
