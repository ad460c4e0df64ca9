#!/bin/bash
# New-bench shakedown on the GPU box: small default-workload run, a 2-rank
# run on the one GPU (gloo exchange), then the default 10M run.  usage: bench_check.sh TAG
TAG=${1:-bc}
mkdir -p gpurun_out/$TAG
timeout 900 python bench.py --tuples 1000000 --steps 3 --cpu-pairs 30000000 > gpurun_out/$TAG/p5pipe_1M.json 2> gpurun_out/$TAG/p5pipe_1M.err; echo "1M rc=$?"
tail -c 3000 gpurun_out/$TAG/p5pipe_1M.json
timeout 900 python bench.py --gpus 2 --tuples 300000 --steps 3 --no-secondary > gpurun_out/$TAG/p5pipe_2rank.json 2> gpurun_out/$TAG/p5pipe_2rank.err; echo "2rank rc=$?"
tail -c 1500 gpurun_out/$TAG/p5pipe_2rank.json
timeout 1500 python bench.py > gpurun_out/$TAG/p5pipe_10M.json 2> gpurun_out/$TAG/p5pipe_10M.err; echo "10M rc=$?"
tail -c 4000 gpurun_out/$TAG/p5pipe_10M.json
