set -x
timeout 900 python bench.py > gpurun_out/bench_full_parity.json 2> gpurun_out/bench_full_parity.err
tail -1 gpurun_out/bench_full_parity.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], json.dumps(d['parity']))"
