set -x
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -1 gpurun_out/final_bench.json | cut -c1-200
bash profiles/capture.sh r1s29c citation3 1000000 2024
bash profiles/capture.sh r1s29e edit_heavy 1000000 11
