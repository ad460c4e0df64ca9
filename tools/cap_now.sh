set -x
timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -25 > gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
bash tools/gpu_perf.sh s28
bash tools/gpu_variants.sh var28 edit_heavy "RB_FOLD_BAG=0"
bash tools/gpu_variants.sh var28 linkage "RB_FOLD_BAG=1"
