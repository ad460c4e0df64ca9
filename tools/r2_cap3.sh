#!/bin/bash
# captures of the current kernel source for the other BASELINE workloads (1M)
bash profiles/capture.sh r2v_c3 citation3 1000000
bash profiles/capture.sh r2v_eh edit_heavy 1000000
bash profiles/capture.sh r2v_p5 person5 1000000
bash profiles/capture.sh r2v_lk linkage 1000000
ls gpurun_out | grep r2v
