set -x
python bench.py --steps 3 --no-cpu > gpurun_out/cap/c3_bench.json 2> gpurun_out/cap/c3_bench.err
bash profiles/capture.sh r1s3c citation3 1000000 2024
bash profiles/capture.sh r1s3e edit_heavy 1000000 11
