set -x
timeout 1500 python -m pytest tests/ -q -m gpu 2>&1 | tail -25 > gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()"
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -1 gpurun_out/final_bench.json | cut -c1-300
timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; tail -1 gpurun_out/final_ref.json | cut -c1-200
bash tools/gpu_perf.sh s20
bash profiles/capture.sh r1s20c citation3 1000000 2024
bash profiles/capture.sh r1s20e edit_heavy 1000000 11
