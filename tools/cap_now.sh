timeout 1800 python bench.py --workload linkage --tuples 10000000 > gpurun_out/link_10M.json 2> gpurun_out/link_10M.err; echo rc=$?; grep step gpurun_out/link_10M.err | tail -4
