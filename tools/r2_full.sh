#!/bin/bash
# full GPU test suite + default bench + the reference's published suites.  usage: r2_full.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out/$TAG
nproc > gpurun_out/$TAG/nproc.txt; lscpu | grep "Model name" >> gpurun_out/$TAG/nproc.txt
timeout 1800 python -m pytest tests/ -x -q -m gpu > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/$TAG/pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/$TAG/p5pipe_10M.json 2> gpurun_out/$TAG/p5pipe_10M.err; echo "10M rc=$?"
grep "^step" gpurun_out/$TAG/p5pipe_10M.err | tail -5
timeout 900 python tools/reference_suites.py --reference --out gpurun_out/$TAG/suites.jsonl > gpurun_out/$TAG/suites.log 2>&1; echo "suites rc=$?"
cat gpurun_out/$TAG/suites.jsonl | cut -c1-600
