timeout 900 python -m pytest tests/test_deferred.py tests/test_pipeline.py tests/test_scheduler.py tests/test_gpu_parity.py tests/test_distributed.py -q -m gpu -x 2>&1 | tail -3
for wl in linkage citation3_parts person5_parts; do timeout 900 python bench.py --workload $wl --no-cpu > gpurun_out/rp_$wl.json 2> gpurun_out/rp_$wl.err; echo "$wl $(grep '^step' gpurun_out/rp_$wl.err | tail -1)"; python -c "
import json; d=json.loads(open('gpurun_out/rp_$wl.json').read().strip().splitlines()[-1]); print('%.4g'%d['value'])"; done
timeout 1800 python bench.py --workload person5_parts --tuples 10000000 --no-cpu --steps 3 > gpurun_out/rp_10M.json 2> gpurun_out/rp_10M.err; grep step gpurun_out/rp_10M.err | tail -2
