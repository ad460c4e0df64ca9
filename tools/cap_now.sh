timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -6
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --workload person5_parts > gpurun_out/p5parts_asym.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/p5parts_asym.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['parity'])"
