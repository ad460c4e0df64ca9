#!/bin/bash
TAG=${1:-r2f}
mkdir -p gpurun_out/$TAG
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_deferred.py tests/test_pipeline.py tests/test_device_pipeline.py tests/test_reference_dropin.py tests/test_scheduler.py -x -q -m gpu > gpurun_out/$TAG/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/$TAG/pytest.log
timeout 1500 python bench.py > gpurun_out/$TAG/p5pipe_10M.json 2> gpurun_out/$TAG/p5pipe_10M.err; echo "10M rc=$?"
grep "^step" gpurun_out/$TAG/p5pipe_10M.err | tail -3
python -c "import json; d=json.loads(open('gpurun_out/$TAG/p5pipe_10M.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['e2e']['phases_s'], d['roofline']['bound'], d['roofline']['frac'], d['secondary']['value'], d['parity']['bit_exact'], d['parity']['full_step']['recall']['exact'])"
