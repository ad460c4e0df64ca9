timeout 900 python -m pytest tests/test_deferred.py tests/test_pipeline.py -q -m gpu -x 2>&1 | tail -5
timeout 600 python bench.py --workload person5_parts > gpurun_out/p5parts_packed.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/p5parts_packed.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['parity'])"
