set -x
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -1 gpurun_out/final_bench.json | cut -c1-300
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; tail -1 gpurun_out/final_ref.json | cut -c1-300
bash profiles/capture.sh r1s15c citation3 1000000 2024
bash tools/scale_runs.sh
