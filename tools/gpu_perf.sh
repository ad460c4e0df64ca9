#!/bin/bash
# GPU check + quick per-workload bench lines (run under gpurun).  usage: gpu_perf.sh TAG [tests]
TAG=${1:-perf}
mkdir -p gpurun_out/$TAG
if [ "${2:-}" = "tests" ]; then
  timeout 1500 python -m pytest tests/ -x -q -m gpu > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/$TAG/pytest_gpu.log
fi
for wl in citation3 edit_heavy person5 person5_parts linkage citation3_parts citation_small; do
  timeout 600 python bench.py --workload $wl --steps 3 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/$TAG/$wl.json 2> gpurun_out/$TAG/$wl.err
  echo "$wl rc=$? $(python -c "import json,sys; d=json.loads(open('gpurun_out/$TAG/$wl.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'])" 2>&1 | tail -1)"
done
