#!/bin/bash
TAG=${1:-r2tree}
mkdir -p gpurun_out/$TAG
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "golden or random" > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/$TAG/pytest_gpu.log
timeout 900 python bench.py --no-cpu --no-secondary --steps 5 > gpurun_out/$TAG/p5pipe.json 2> gpurun_out/$TAG/p5pipe.err
echo "pipeline rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/p5pipe.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'])" 2>&1 | tail -1)"
grep "^step" gpurun_out/$TAG/p5pipe.err | tail -1
for wl in person5_parts linkage; do
  timeout 600 python bench.py --workload $wl --steps 5 --no-cpu > gpurun_out/$TAG/${wl}.json 2> gpurun_out/$TAG/${wl}.err
  echo "$wl rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/${wl}.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], d['ms_per_step'])" 2>&1 | tail -1)"
done
timeout 600 python bench.py --workload person5 --tuples 1000000 --steps 5 --no-cpu > gpurun_out/$TAG/person5.json 2> gpurun_out/$TAG/person5.err
echo "person5 1M rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/person5.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], d['ms_per_step'])" 2>&1 | tail -1)"
