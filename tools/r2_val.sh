#!/bin/bash
# validation of the current tree: smoke, every GPU test, the small-partition and default bench lines
TAG=${1:-r2v}
mkdir -p gpurun_out/$TAG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/$TAG/gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$TAG/smoke.log 2>&1; echo "smoke rc=$?"
for wl in citation3_parts citation_small citation3; do
  timeout 600 python bench.py --workload $wl --steps 5 > gpurun_out/$TAG/wl_$wl.json 2> gpurun_out/$TAG/wl_$wl.err
  echo "$wl rc=$? $(tail -c 600 gpurun_out/$TAG/wl_$wl.json)"
done
timeout 2400 python -m pytest tests/ -q -x -m gpu > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/$TAG/pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err; echo "bench rc=$?"
tail -c 400 gpurun_out/$TAG/bench.json
