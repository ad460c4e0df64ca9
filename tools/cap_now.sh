set -x
bash tools/gpu_variants.sh var13 citation3 "RB_JIT_ROWS=3" "RB_JIT_ROWS=4 RB_JIT_MINBLOCKS=2" "RB_JIT_UNROLL=2" "RB_JIT_MINBLOCKS=4" "RB_JIT_UNROLL=8"
bash tools/gpu_variants.sh var13 person5 "RB_JIT_ROWS=3" "RB_JIT_UNROLL=4"
