set -x
timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -25 > gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
bash tools/gpu_perf.sh s11
bash tools/gpu_variants.sh var11 citation3 "RB_JIT_MIRROR=0"
bash tools/gpu_variants.sh var11 citation3_parts "RB_JIT_MIRROR=0"
