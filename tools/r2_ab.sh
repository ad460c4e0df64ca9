#!/bin/bash
# A/B of an environment knob on the small-partition and headline workloads
TAG=${1:-r2ab}; VAR=${2:-RB_SMALLRES}
mkdir -p gpurun_out/$TAG
for v in 1 0; do
  for wl in citation3_parts person5_parts; do
    env $VAR=$v timeout 600 python bench.py --workload $wl --steps 10 --no-cpu > gpurun_out/$TAG/${wl}_$v.json 2> gpurun_out/$TAG/${wl}_$v.err
    echo "$VAR=$v $wl rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/${wl}_$v.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'], (d.get('parity') or {}).get('bit_exact'))" 2>&1 | tail -1)"
  done
  env $VAR=$v timeout 900 python bench.py --no-cpu --no-secondary --steps 5 > gpurun_out/$TAG/p5pipe_$v.json 2> gpurun_out/$TAG/p5pipe_$v.err
  echo "$VAR=$v pipeline rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/p5pipe_$v.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'])" 2>&1 | tail -1)"
  grep "^step" gpurun_out/$TAG/p5pipe_$v.err | tail -2
done
