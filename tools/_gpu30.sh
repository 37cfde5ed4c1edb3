timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
QG_SCREEN=1 timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_screen.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_screen.log
for sc in 0 1; do echo "== QG_SCREEN=$sc"; QG_SCREEN=$sc timeout 120 python tools/phase_tiled.py C4 8 8 2>&1 | cut -c1-170 | head -2; done
