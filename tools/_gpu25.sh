timeout 900 python -m pytest tests/test_gpu_acceptance.py -x -q > gpurun_out/pytest_acc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_acc.log
