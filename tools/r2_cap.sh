#!/bin/bash
# targeted GPU tests + default bench + ncu capture of the headline pair kernel.  usage: r2_cap.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out/$TAG
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_deferred.py tests/test_device_pipeline.py tests/test_pipeline.py tests/test_edit_fuzz.py -x -q -m gpu > gpurun_out/$TAG/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/$TAG/pytest.log
timeout 1500 python bench.py --no-secondary > gpurun_out/$TAG/p5pipe_10M.json 2> gpurun_out/$TAG/p5pipe_10M.err; echo "10M rc=$?"
grep "^step" gpurun_out/$TAG/p5pipe_10M.err | tail -3
python -c "import json; d=json.loads(open('gpurun_out/$TAG/p5pipe_10M.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e'])"
bash profiles/capture.sh $TAG person5_pipeline 10000000
