#!/bin/bash
# ncu captures of the final kernel source: the headline (both pair-kernel launches) and every other workload
bash profiles/capture.sh r2z2 person5_pipeline 10000000 2
bash profiles/capture.sh r2z2_c3 citation3 1000000
bash profiles/capture.sh r2z2_eh edit_heavy 1000000
bash profiles/capture.sh r2z2_p5 person5 1000000
bash profiles/capture.sh r2z2_lk linkage 1000000
bash profiles/capture.sh r2z2_p5parts person5_parts 1000000
bash profiles/capture.sh r2z2_c3parts citation3_parts 1000000
bash profiles/capture.sh r2z2_csmall citation_small 4591
rm -f gpurun_out/*_full.ncu-rep.tmp
ls -la gpurun_out | grep r2z2 | awk '{print $5, $9}'
