timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -4
timeout 1800 python bench.py --workload person5 --tuples 10000000 --no-cpu --steps 3 > gpurun_out/p5_10M.json 2> gpurun_out/p5_10M.err; echo rc=$?; grep step gpurun_out/p5_10M.err | tail -4; tail -1 gpurun_out/p5_10M.json | cut -c1-200
timeout 1800 python bench.py --workload person5_parts --tuples 10000000 > gpurun_out/p5parts_10M_d.json 2> gpurun_out/p5parts_10M_d.err; echo rc=$?; grep step gpurun_out/p5parts_10M_d.err | tail -3
