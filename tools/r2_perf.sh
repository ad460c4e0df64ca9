#!/bin/bash
# GPU tests + the per-workload lines (no CPU leg) + a host-timing breakdown of 512-tuple partitions
TAG=${1:-r2p}; TESTS=${2:-1}
mkdir -p gpurun_out/$TAG
if [ "$TESTS" = 1 ]; then
  timeout 1800 python -m pytest tests/ -q -x -m gpu > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/$TAG/pytest_gpu.log
fi
for wl in citation3_parts citation_small person5_parts citation3; do
  timeout 600 python bench.py --workload $wl --steps 10 --no-cpu > gpurun_out/$TAG/$wl.json 2> gpurun_out/$TAG/$wl.err
  echo "$wl rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/$wl.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'], (d.get('parity') or {}).get('bit_exact'))" 2>&1 | tail -1)"
done
RB_HOST_TIMING=1 timeout 600 python bench.py --workload citation3_parts --steps 5 --no-cpu > gpurun_out/$TAG/c3p_timing.json 2> gpurun_out/$TAG/c3p_timing.err
timeout 900 python bench.py --no-cpu --no-secondary --steps 5 > gpurun_out/$TAG/p5pipe.json 2> gpurun_out/$TAG/p5pipe.err
echo "pipeline rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/p5pipe.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'])" 2>&1 | tail -1)"
grep "^step" gpurun_out/$TAG/p5pipe.err | tail -3
