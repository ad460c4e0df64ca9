set -x
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo n2 rc=$?; tail -1 gpurun_out/bench_n2.json | cut -c1-200
bash profiles/capture.sh r1s24p person5 1000000 4
bash profiles/capture.sh r1s24l linkage 1000000 5
bash tools/scale_runs.sh
