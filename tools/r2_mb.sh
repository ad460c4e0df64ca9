#!/bin/bash
TAG=${1:-r2mb}
mkdir -p gpurun_out/$TAG
for mb in 4 3; do
  RB_JIT_MINBLOCKS=$mb timeout 900 python bench.py --no-cpu --no-secondary --steps 5 > gpurun_out/$TAG/p5pipe_mb$mb.json 2> gpurun_out/$TAG/p5pipe_mb$mb.err
  echo "mb=$mb pipeline rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/p5pipe_mb$mb.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'])" 2>&1 | tail -1)"
  grep "^step" gpurun_out/$TAG/p5pipe_mb$mb.err | tail -1
  for wl in person5_parts linkage; do
    RB_JIT_MINBLOCKS=$mb timeout 600 python bench.py --workload $wl --steps 5 --no-cpu > gpurun_out/$TAG/${wl}_mb$mb.json 2> gpurun_out/$TAG/${wl}_mb$mb.err
    echo "mb=$mb $wl rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/${wl}_mb$mb.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], d['ms_per_step'])" 2>&1 | tail -1)"
  done
done
