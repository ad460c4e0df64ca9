#!/bin/bash
# Profile capture run on the GPU box (under gpurun).  Writes into gpurun_out/.
#   1. launch list (device time of every launch) of a short bench command
#   2. one `ncu --set full` capture of the timed pair-kernel launch at the bench size
# usage: capture.sh TAG [WORKLOAD] [N] [SEED]
set -u
TAG=${1:-r1}
WL=${2:-citation3}
N=${3:-1000000}
SEED=${4:-2024}
CMD="python bench.py --workload $WL --tuples $N --seed $SEED --steps 1 --warmup 3 --no-cpu --e2e-steps 1"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_launches.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 3 -c 1 \
    -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_full.log 2>&1
tail -2 gpurun_out/${TAG}_full.log
