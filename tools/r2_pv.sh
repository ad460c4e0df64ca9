#!/bin/bash
# the stage-1 pre-vote kernel: GPU tests, the headline with parity, every workload's line, the pre-vote off
TAG=${1:-r2pv}
mkdir -p gpurun_out/$TAG
timeout 1800 python -m pytest tests/ -q -x -m gpu > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/$TAG/pytest_gpu.log
timeout 1200 python bench.py --no-secondary --steps 5 > gpurun_out/$TAG/p5pipe.json 2> gpurun_out/$TAG/p5pipe.err
echo "pipeline rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/p5pipe.json').read().strip().splitlines()[-1]); p=d.get('parity') or {}; print('%.3e'%d['value'], d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'], p.get('bit_exact'), (p.get('full_step') or {}).get('recall',{}).get('exact'))" 2>&1 | tail -1)"
grep "^step" gpurun_out/$TAG/p5pipe.err | tail -2
for wl in citation3 edit_heavy linkage person5_parts citation3_parts citation_small; do
  timeout 600 python bench.py --workload $wl --steps 5 --no-cpu > gpurun_out/$TAG/$wl.json 2> gpurun_out/$TAG/$wl.err
  echo "$wl rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/$wl.json').read().strip().splitlines()[-1]); p=d.get('parity') or {}; print('%.3e'%d['value'], d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'], p.get('bit_exact'))" 2>&1 | tail -1)"
done
RB_PREANY=0 timeout 900 python bench.py --no-cpu --no-secondary --steps 3 > gpurun_out/$TAG/p5pipe_off.json 2> gpurun_out/$TAG/p5pipe_off.err
echo "pre-vote off rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/p5pipe_off.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], d['ms_per_step'])" 2>&1 | tail -1)"
