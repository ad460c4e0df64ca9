set -x
timeout 900 python tools/ingest_e2e.py 1000000 > gpurun_out/ingest_e2e.json 2> gpurun_out/ingest_e2e.err; tail -1 gpurun_out/ingest_e2e.json
bash profiles/capture.sh r1s11l linkage 1000000 5
bash profiles/capture.sh r1s11p person5 1000000 4
