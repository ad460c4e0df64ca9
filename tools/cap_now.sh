set -x
bash tools/gpu_perf.sh s8
bash tools/gpu_variants.sh var8 edit_heavy "RB_JIT_UNROLL=2"
bash tools/gpu_variants.sh var8 linkage "RB_JIT_UNROLL=2"
