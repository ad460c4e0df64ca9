#!/bin/bash
# bench one workload under several JIT shapes (env overrides).  usage: gpu_variants.sh TAG WORKLOAD "ENV1" "ENV2" ...
TAG=$1; WL=$2; shift 2
mkdir -p gpurun_out/$TAG
for v in "$@"; do
  env $v timeout 900 python bench.py --workload $WL --steps 3 --warmup 3 --no-cpu --no-secondary --e2e-steps 1 > gpurun_out/$TAG/$WL.${v// /_}.json 2>gpurun_out/$TAG/$WL.${v// /_}.err
  echo "$WL [$v] $(python -c "import json; d=json.loads(open('gpurun_out/$TAG/$WL.${v// /_}.json').read().strip().splitlines()[-1]); print('%.3e'%d['value'], 'pair %.1f ms'%d['roofline']['kernel_ms'], 'e2e %.3e'%d['e2e']['value'])" 2>&1 | tail -1)"
done
