set -x
timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -25 > gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests.log
bash tools/gpu_perf.sh s27
timeout 600 python bench.py --workload citation_small --steps 5 > gpurun_out/citation_small.json 2> gpurun_out/citation_small.err; tail -1 gpurun_out/citation_small.json | cut -c1-300
