#!/bin/bash
bash profiles/capture.sh r2w person5_pipeline 10000000 2
bash profiles/capture.sh r2w_c3parts citation3_parts 1000000
bash profiles/capture.sh r2w_csmall citation_small 4591
timeout 900 python -m pytest tests/test_full_golden.py -q -m gpu > gpurun_out/r2w_full_golden.log 2>&1; echo "full golden rc=$?"; tail -2 gpurun_out/r2w_full_golden.log
