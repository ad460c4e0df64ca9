set -x
bash tools/gpu_variants.sh var9 citation3 "RB_JIT_ROWS=3" "RB_JIT_ROWS=2"
bash tools/gpu_variants.sh var9 person5 "RB_JIT_BITS=8 RB_JIT_ROWS=1 RB_JIT_MINBLOCKS=4" "RB_JIT_BITS=8 RB_JIT_ROWS=1 RB_JIT_MINBLOCKS=3" "RB_JIT_ROWS=1 RB_JIT_MINBLOCKS=4" "RB_JIT_ROWS=2"
bash tools/gpu_variants.sh var9 edit_heavy "RB_JIT_ROWS=3"
