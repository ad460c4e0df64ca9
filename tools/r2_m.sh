#!/bin/bash
TAG=${1:-r2m}
mkdir -p gpurun_out/$TAG
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$TAG/smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests/ -x -q -m gpu > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/$TAG/pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err; echo "bench rc=$?"
grep "^step\|WARNING" gpurun_out/$TAG/bench.err | tail -3
python -c "import json; d=json.loads(open('gpurun_out/$TAG/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['bound'], d['roofline']['frac'], d['roofline']['capture_current'], d['secondary']['value'], d['cpu_baseline']['value'], d['parity']['bit_exact'], d['parity']['full_step']['recall']['exact'])"
timeout 900 python bench.py --impl reference > gpurun_out/$TAG/bench_ref.json 2> gpurun_out/$TAG/bench_ref.err; echo "ref rc=$?"; tail -c 600 gpurun_out/$TAG/bench_ref.json
timeout 900 python tools/reference_suites.py --reference --suites scaling,overlap --out gpurun_out/$TAG/suites.jsonl > gpurun_out/$TAG/suites.log 2>&1; echo "suites rc=$?"; cut -c1-400 gpurun_out/$TAG/suites.jsonl
