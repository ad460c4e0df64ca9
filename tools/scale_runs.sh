#!/bin/bash
# Large single-GPU runs for DESIGN.md: config 4 (ii) 10M single partition, config 5 at 5M x 5M.
mkdir -p gpurun_out/scale
timeout 1800 python bench.py --workload person5 --tuples 10000000 --steps 1 --warmup 3 --no-cpu --e2e-steps 1 \
    > gpurun_out/scale/person5_10M.json 2> gpurun_out/scale/person5_10M.err
echo "person5 10M rc=$?"; tail -1 gpurun_out/scale/person5_10M.json | cut -c1-400
timeout 1800 python bench.py --workload linkage --tuples 10000000 --steps 3 --warmup 3 \
    > gpurun_out/scale/linkage_10M.json 2> gpurun_out/scale/linkage_10M.err
echo "linkage 10M rc=$?"; tail -1 gpurun_out/scale/linkage_10M.json | cut -c1-400
