timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --config C4 --bits 8 --no-sweep --no-c5 --steps 30 --warmup 5 --cpu-sample-s 20 > gpurun_out/bench_c4.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c4.log
timeout 300 python bench.py --config C3 --no-sweep --no-c5 --steps 50 --warmup 5 > gpurun_out/bench_c3.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_c3.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu --no-c5 > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_tiled -s 12 -c 6 -o gpurun_out/c2_tiled_final python tools/cold_step.py > gpurun_out/ncu_c2.log 2>&1
