#!/bin/bash
TAG=${1:-r2t2}
mkdir -p gpurun_out/$TAG
timeout 900 python -m pytest tests/test_deferred.py tests/test_pipeline.py -q -m gpu > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/$TAG/pytest_gpu.log
RB_HOST_TIMING=1 timeout 900 python bench.py --no-cpu --no-secondary --steps 2 --warmup 3 > gpurun_out/$TAG/p5pipe_timing.json 2> gpurun_out/$TAG/p5pipe_timing.err
echo "timing rc=$?"; grep -v "^rb partition" gpurun_out/$TAG/p5pipe_timing.err | tail -8
RB_HOST_TIMING=1 timeout 600 python bench.py --workload citation3_parts --steps 5 --no-cpu > gpurun_out/$TAG/c3p.json 2> gpurun_out/$TAG/c3p.err
tail -4 gpurun_out/$TAG/c3p.err
