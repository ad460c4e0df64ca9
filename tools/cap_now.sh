timeout 900 python -m pytest tests/test_deferred.py tests/test_pipeline.py tests/test_scheduler.py tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
RB_HOST_TIMING=1 timeout 600 python tools/batch_phases.py person5_parts 2>&1 | tail -2
timeout 600 python bench.py --workload person5_parts > gpurun_out/p5parts_packed2.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/p5parts_packed2.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['parity'])"
