#!/bin/bash
TAG=${1:-r2i}
mkdir -p gpurun_out/$TAG
timeout 1500 python -m pytest tests/test_device_pipeline.py tests/test_pipeline.py tests/test_reference_dropin.py -x -q -m gpu > gpurun_out/$TAG/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/$TAG/pytest.log
timeout 1500 python bench.py --no-secondary > gpurun_out/$TAG/p5pipe_10M.json 2> gpurun_out/$TAG/p5pipe_10M.err; echo "10M rc=$?"
grep "^step\|WARNING" gpurun_out/$TAG/p5pipe_10M.err | tail -3
python -c "import json; d=json.loads(open('gpurun_out/$TAG/p5pipe_10M.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['kernel_specialized'], d['parity']['bit_exact'], d['parity']['full_step']['recall']['exact'], d['parity']['full_step']['witness_exact'])"
RB_IMPLIED_OFF=1 timeout 900 python bench.py --no-secondary --no-cpu --steps 3 > gpurun_out/$TAG/p5pipe_10M_off.json 2> gpurun_out/$TAG/p5pipe_10M_off.err; echo "off rc=$?"
grep "^step" gpurun_out/$TAG/p5pipe_10M_off.err | tail -2
