timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/cold_step.py C2 4 > gpurun_out/cold.log 2>&1
QG_A_BITS=0 timeout 300 python tools/cold_step.py C2 4 > gpurun_out/cold_bytes.log 2>&1
timeout 300 python tools/run_config.py C3 > gpurun_out/c3.log 2>&1
timeout 600 python tools/run_config.py C4 8 > gpurun_out/c4.log 2>&1
QG_A_BITS=0 timeout 600 python tools/run_config.py C4 8 > gpurun_out/c4_bytes.log 2>&1
timeout 600 python tools/c5_sweep.py --sizes 4096,16384 --rhos 0.1 --bits 4 > gpurun_out/c5.log 2>&1
QG_A_BITS=0 timeout 600 python tools/c5_sweep.py --sizes 4096,16384 --rhos 0.1 --bits 4 > gpurun_out/c5_bytes.log 2>&1
