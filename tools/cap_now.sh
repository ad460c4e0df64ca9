set -x
timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -25 > gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
bash tools/gpu_perf.sh s15
bash tools/gpu_variants.sh var15 citation3 "RB_JIT_ROWS=4 RB_JIT_MINBLOCKS=4" "RB_JIT_ROWS=3 RB_JIT_MINBLOCKS=4 RB_JIT_UNROLL=2"
