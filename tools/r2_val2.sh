#!/bin/bash
# smoke + every GPU test + the pipeline's host-phase breakdown + the small-partition line
TAG=${1:-r2x}
mkdir -p gpurun_out/$TAG
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$TAG/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python -m pytest tests/ -q -m gpu > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/$TAG/pytest_gpu.log
RB_HOST_TIMING=1 timeout 900 python bench.py --no-cpu --no-secondary --steps 2 --warmup 3 > gpurun_out/$TAG/p5pipe_timing.json 2> gpurun_out/$TAG/p5pipe_timing.err
echo "timing rc=$?"; grep -v "^rb partition" gpurun_out/$TAG/p5pipe_timing.err | tail -12
for wl in citation3_parts; do
  timeout 600 python bench.py --workload $wl --steps 10 --no-cpu > gpurun_out/$TAG/$wl.json 2> gpurun_out/$TAG/$wl.err
  echo "$wl rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/$wl.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'], d['roofline']['capture_current'])" 2>&1 | tail -1)"
done
