#!/bin/bash
TAG=${1:-r2g}
mkdir -p gpurun_out/$TAG
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_deferred.py tests/test_pipeline.py tests/test_device_pipeline.py -x -q -m gpu > gpurun_out/$TAG/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/$TAG/pytest.log
timeout 1500 python bench.py --no-secondary > gpurun_out/$TAG/p5pipe_10M.json 2> gpurun_out/$TAG/p5pipe_10M.err; echo "10M rc=$?"
grep "^step" gpurun_out/$TAG/p5pipe_10M.err | tail -2
python -c "import json; d=json.loads(open('gpurun_out/$TAG/p5pipe_10M.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['e2e']['phases_s'], d['kernel_specialized'], d['roofline']['frac'])"
bash tools/gpu_variants.sh $TAG person5_pipeline "RB_JIT_UNROLL=4" "RB_JIT_UNROLL=1" "RB_JIT_MINBLOCKS=4" "RB_PACK_MAX=0" "RB_GATE=0"
