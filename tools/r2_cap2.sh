#!/bin/bash
# ncu captures of the current kernel source: the headline and the small-partition workloads
bash profiles/capture.sh r2h person5_pipeline 10000000
bash profiles/capture.sh r2h_c3parts citation3_parts 1000000
bash profiles/capture.sh r2h_csmall citation_small 0
