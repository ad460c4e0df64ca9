#!/bin/bash
TAG=${1:-r2t3}
mkdir -p gpurun_out/$TAG
timeout 900 python -m pytest tests/test_pipeline.py tests/test_partitioning.py tests/test_multirank.py tests/test_distributed.py -q -m gpu > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/$TAG/pytest_gpu.log
RB_HOST_TIMING=1 timeout 900 python bench.py --no-cpu --no-secondary --steps 3 --warmup 3 > gpurun_out/$TAG/p5pipe_timing.json 2> gpurun_out/$TAG/p5pipe_timing.err
echo "timing rc=$?"; grep -v "^rb run:" gpurun_out/$TAG/p5pipe_timing.err | tail -9
python -c "import json; d=json.loads(open('gpurun_out/$TAG/p5pipe_timing.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'], d['e2e'].get('phases_s'))"
