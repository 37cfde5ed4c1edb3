for m in cal int int_screen; do
  timeout 120 python tools/_repro.py $m > gpurun_out/r_$m.log 2>&1; tail -1 gpurun_out/r_$m.log
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/cold_step.py C2 4 > gpurun_out/cold.log 2>&1
QG_FUSED_EPOCH=0 timeout 300 python tools/cold_step.py C2 4 > gpurun_out/cold_nofuse.log 2>&1
timeout 300 python tools/phase_tiled.py C2 4 > gpurun_out/phase_c2.log 2>&1
