set -x
timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -25 > gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
bash tools/gpu_perf.sh s23
