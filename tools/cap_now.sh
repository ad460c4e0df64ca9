set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_random_shapes.py -q -m gpu -x 2>&1 | tail -2
bash tools/gpu_variants.sh var19 citation3 "RB_X=1" "RB_X=2"
bash tools/gpu_variants.sh var19 person5 "RB_X=1"
