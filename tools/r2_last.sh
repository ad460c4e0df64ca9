#!/bin/bash
TAG=${1:-r2last}
mkdir -p gpurun_out/$TAG
timeout 900 python bench.py --workload linkage --tuples 10000000 --steps 3 > gpurun_out/$TAG/wl_linkage_10M.json 2> gpurun_out/$TAG/wl_linkage_10M.err
echo "linkage 10M rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/wl_linkage_10M.json').read().strip().splitlines()[-1]); p=d.get('parity') or {}; print('%.3e'%d['value'], d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'], p.get('bit_exact'))" 2>&1 | tail -1)"
timeout 900 python bench.py --workload person5_parts --tuples 10000000 --steps 3 > gpurun_out/$TAG/wl_person5_parts_10M.json 2> gpurun_out/$TAG/wl_person5_parts_10M.err
echo "person5_parts 10M rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/wl_person5_parts_10M.json').read().strip().splitlines()[-1]); p=d.get('parity') or {}; print('%.3e'%d['value'], d['ms_per_step'], 'e2e %.3e'%d['e2e']['value'], p.get('bit_exact'))" 2>&1 | tail -1)"
