set -x
timeout 900 python bench.py --workload person5_parts > gpurun_out/bench_p5parts.json 2> gpurun_out/bench_p5parts.err
tail -1 gpurun_out/bench_p5parts.json | cut -c1-1500
tail -5 gpurun_out/bench_p5parts.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/p5parts_launches.csv timeout 600 python bench.py --workload person5_parts --steps 1 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:rb_pair_kernel_spec -s 3 -c 1 -o gpurun_out/p5parts_full timeout 900 python bench.py --workload person5_parts --steps 1 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
ls gpurun_out
