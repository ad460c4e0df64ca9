set -x
timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -25 > gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
bash tools/gpu_perf.sh s7
bash tools/gpu_variants.sh var7 citation3 "RB_JIT_UNROLL=4" "RB_JIT_ROWS=3" "RB_JIT_ROWS=4 RB_JIT_MINBLOCKS=2" "RB_JIT_ROWS=4"
bash tools/gpu_variants.sh var7 person5 "RB_JIT_UNROLL=4" "RB_JIT_ROWS=3" "RB_JIT_BITS=8"
