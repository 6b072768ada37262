#!/bin/bash
# tools/prof_one.sh <tag> <shape> [variant]: ncu --set full of one beamform launch via sweep_f16
TAG=$1; SHAPE=${2:-radio}; V=${3:-1}
mkdir -p gpurun_out
VARIANTS=$V timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:cgemm -s 2 -c 1 \
  -o gpurun_out/prof_${TAG}_${SHAPE}_v${V} -f python tools/sweep_f16.py $SHAPE > gpurun_out/prof_${TAG}_${SHAPE}_v${V}.log 2>&1
