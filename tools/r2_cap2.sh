#!/bin/bash
# ncu captures of the current kernel source: the headline and the small-partition workloads
bash profiles/capture.sh r2l person5_pipeline 10000000
bash profiles/capture.sh r2l_c3parts citation3_parts 1000000
bash profiles/capture.sh r2l_csmall citation_small 4591
ls -la gpurun_out/ | grep r2l
