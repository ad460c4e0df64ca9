#!/bin/bash
TAG=${1:-r2e}
mkdir -p gpurun_out/$TAG
timeout 1800 python -m pytest tests/ -x -q -m gpu > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/$TAG/pytest_gpu.log
timeout 1500 python bench.py --no-secondary > gpurun_out/$TAG/p5pipe_10M.json 2> gpurun_out/$TAG/p5pipe_10M.err; echo "10M rc=$?"
grep "^step" gpurun_out/$TAG/p5pipe_10M.err | tail -3
python -c "import json; d=json.loads(open('gpurun_out/$TAG/p5pipe_10M.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['e2e']['phases_s'], d['roofline']['bound'], d['roofline']['frac'])"
for wl in linkage person5_parts citation3_parts; do
  timeout 600 python bench.py --workload $wl --steps 3 --no-cpu > gpurun_out/$TAG/$wl.json 2> gpurun_out/$TAG/$wl.err
  echo "$wl rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/$wl.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'])" 2>&1 | tail -1)"
done
timeout 900 python tools/reference_suites.py --reference --suites async,overlap --out gpurun_out/$TAG/suites.jsonl > gpurun_out/$TAG/suites.log 2>&1; echo "suites rc=$?"
cut -c1-700 gpurun_out/$TAG/suites.jsonl
