#!/bin/bash
TAG=$1; CFG=${2:-radio_b1}
mkdir -p gpurun_out
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:cgemm_b1 -s 2 -c 1 \
  -o gpurun_out/prof_${TAG}_${CFG} -f python tools/quick_time.py $CFG > gpurun_out/prof_${TAG}_${CFG}.log 2>&1
