#!/bin/bash
TAG=${1:-r2pv2}
mkdir -p gpurun_out/$TAG
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_pipeline.py tests/test_random_shapes.py tests/test_device_pipeline.py -q -x -m gpu > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/$TAG/pytest_gpu.log
timeout 900 python bench.py --no-cpu --no-secondary --steps 5 > gpurun_out/$TAG/p5pipe.json 2> gpurun_out/$TAG/p5pipe.err
echo "pipeline rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/p5pipe.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'])" 2>&1 | tail -1)"
grep "^step" gpurun_out/$TAG/p5pipe.err | tail -1
for wl in citation3 person5 person5_parts citation3_parts linkage; do
  timeout 600 python bench.py --workload $wl --steps 5 --no-cpu --tuples 1000000 > gpurun_out/$TAG/$wl.json 2> gpurun_out/$TAG/$wl.err
  echo "$wl rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/$wl.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'])" 2>&1 | tail -1)"
done
for wl in citation3 person5; do
  RB_PREANY=1 timeout 600 python bench.py --workload $wl --steps 5 --no-cpu --tuples 1000000 > gpurun_out/$TAG/${wl}_on.json 2> gpurun_out/$TAG/${wl}_on.err
  echo "$wl pre-vote forced on rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/${wl}_on.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], d['ms_per_step'])" 2>&1 | tail -1)"
done
RB_PREANY=0 timeout 600 python bench.py --workload person5 --steps 5 --no-cpu --tuples 1000000 > gpurun_out/$TAG/person5_off.json 2> gpurun_out/$TAG/person5_off.err
echo "person5 pre-vote off rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/person5_off.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], d['ms_per_step'])" 2>&1 | tail -1)"
