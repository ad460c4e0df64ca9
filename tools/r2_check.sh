#!/bin/bash
# pipeline GPU tests + drop-in tests + default bench (1M quick, 10M full).  usage: r2_check.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out/$TAG
timeout 1200 python -m pytest tests/test_device_pipeline.py tests/test_pipeline.py tests/test_reference_dropin.py -x -q -m gpu > gpurun_out/$TAG/pytest_pipe.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/$TAG/pytest_pipe.log
timeout 900 python bench.py --tuples 1000000 --steps 3 --cpu-pairs 30000000 > gpurun_out/$TAG/p5pipe_1M.json 2> gpurun_out/$TAG/p5pipe_1M.err; echo "1M rc=$?"
grep "^step" gpurun_out/$TAG/p5pipe_1M.err | tail -3
timeout 1500 python bench.py > gpurun_out/$TAG/p5pipe_10M.json 2> gpurun_out/$TAG/p5pipe_10M.err; echo "10M rc=$?"
grep "^step" gpurun_out/$TAG/p5pipe_10M.err | tail -5
tail -c 1500 gpurun_out/$TAG/p5pipe_10M.err
