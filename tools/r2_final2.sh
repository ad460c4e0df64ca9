#!/bin/bash
# final validation: smoke, every GPU test, the default bench line, the reference arm, the reference suites
TAG=${1:-r2zz}
mkdir -p gpurun_out/$TAG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/$TAG/gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$TAG/smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests/ -q -m gpu > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/$TAG/pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err; echo "bench rc=$?"
grep "^step" gpurun_out/$TAG/bench.err | tail -2
timeout 900 python bench.py --impl reference > gpurun_out/$TAG/bench_ref.json 2> gpurun_out/$TAG/bench_ref.err; echo "ref rc=$?"
timeout 1200 python tools/reference_suites.py --reference --out gpurun_out/$TAG/suites.jsonl > gpurun_out/$TAG/suites.log 2>&1; echo "suites rc=$?"
for wl in citation3 edit_heavy person5 linkage citation3_parts citation_small person5_parts; do
  timeout 900 python bench.py --workload $wl --steps 3 > gpurun_out/$TAG/wl_$wl.json 2> gpurun_out/$TAG/wl_$wl.err
  echo "$wl rc=$? $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/wl_$wl.json').read().strip().splitlines()[-1]); p=d.get('parity') or {}; print('%.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'], 'exact', p.get('bit_exact'), (p.get('full_step') or {}).get('recall',{}).get('exact'), d['roofline']['bound'], d['roofline']['frac'])" 2>&1 | tail -1)"
done
