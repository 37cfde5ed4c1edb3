QG_SCREEN=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "screen or requant" > gpurun_out/pytest_screen.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_screen.log
for sc in 0 1; do echo "== QG_SCREEN=$sc"; QG_SCREEN=$sc timeout 120 python tools/phase_tiled.py C4 8 8 2>&1 | cut -c1-170; done
for sc in 0 1; do echo "== QG_SCREEN=$sc"; QG_SCREEN=$sc timeout 200 python tools/run_config.py C4 8 2>&1 | head -1; QG_SCREEN=$sc timeout 100 python tools/cold_step.py C2 4 | head -3 | tail -2; done
