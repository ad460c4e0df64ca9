#!/bin/bash
TAG=${1:-r2d}
mkdir -p gpurun_out/$TAG
timeout 900 python -m pytest tests/test_deferred.py tests/test_gpu_parity.py -q -x -m gpu > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/$TAG/pytest_gpu.log
timeout 300 python tools/e2e_parts_diag.py citation3_parts 2> gpurun_out/$TAG/e2e_parts.err; echo "diag rc=$?"; cat gpurun_out/$TAG/e2e_parts.err | tail -7
for wl in citation3_parts citation_small; do
  timeout 600 python bench.py --workload $wl --steps 10 --no-cpu > gpurun_out/$TAG/$wl.json 2> gpurun_out/$TAG/$wl.err
  echo "$wl rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/$wl.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'], d['e2e'].get('phases_s'))" 2>&1 | tail -1)"
done
for rows in 3; do
  RB_JIT_ROWS=$rows timeout 900 python bench.py --no-cpu --no-secondary --steps 3 > gpurun_out/$TAG/p5pipe_rows$rows.json 2> gpurun_out/$TAG/p5pipe_rows$rows.err
  echo "rows=$rows pipeline rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/p5pipe_rows$rows.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'])" 2>&1 | tail -1)"
  grep "^step" gpurun_out/$TAG/p5pipe_rows$rows.err | tail -2
done
timeout 900 python bench.py --no-cpu --no-secondary --steps 3 > gpurun_out/$TAG/p5pipe.json 2> gpurun_out/$TAG/p5pipe.err
echo "pipeline rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/p5pipe.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'], d['e2e'].get('phases_s'))" 2>&1 | tail -1)"
grep "^step" gpurun_out/$TAG/p5pipe.err | tail -2
