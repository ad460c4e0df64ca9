set -x
timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -25 > gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
bash tools/gpu_perf.sh s5
bash tools/gpu_variants.sh var5 citation3 "RB_COMPOSITE=0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 3 -c 1 -o gpurun_out/r1s5p_full python bench.py --workload citation3_parts --steps 1 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/r1s5p_full.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1s5p_launches.csv python bench.py --workload citation3_parts --steps 1 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
