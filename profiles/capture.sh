#!/bin/bash
# Profile capture run on the GPU box (under gpurun).  Writes into gpurun_out/.
#   1. launch list (device time of every launch) of a short bench command
#   2. one `ncu --set full` capture of the timed pair-kernel launch at the bench size,
#      its details page as CSV and its summary in profiles/traffic.json (copied out)
# usage: capture.sh TAG [WORKLOAD] [N] [COUNT]   (the first COUNT pair-kernel launches inside bench.py's "timed" NVTX range)
set -u
TAG=${1:-r2}
WL=${2:-person5_pipeline}
N=${3:-10000000}
COUNT=${4:-1}   # pair-kernel launches captured (2 for config 4 (i): the implied-root run and the rest)
CMD="python bench.py --workload $WL --tuples $N --steps 1 --warmup 3 --no-cpu --no-secondary --e2e-steps 1"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_launches.log 2>&1
echo "launch list rc=$?"
timeout 2400 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" \
    -k regex:pair_kernel -c $COUNT \
    -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_full.log 2>&1
echo "full capture rc=$?"
tail -2 gpurun_out/${TAG}_full.log
ncu -i gpurun_out/${TAG}_full.ncu-rep --page details --csv > gpurun_out/${TAG}_pair_kernel_details.csv 2>/dev/null
PAIRS=$(grep -o '"pairs_per_step": [0-9]*' gpurun_out/${TAG}_launches.log | head -1 | grep -o '[0-9]*$')
cp profiles/traffic.json gpurun_out/${TAG}_traffic_before.json
python tools/ncu_summary.py gpurun_out/${TAG}_full.ncu-rep $WL $N profiles/${TAG}_pair_kernel_details.csv $PAIRS
cp profiles/traffic.json gpurun_out/${TAG}_traffic.json
