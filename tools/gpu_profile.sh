#!/bin/bash
# Usage (on the GPU box): tools/gpu_profile.sh <config> <tag>
# 1) launch list with per-launch device time (cold-cache, serialised) of a short bench run
# 2) one ncu --set full capture of the dominant kernel (the beamform GEMM)
set -u
CFG=${1:-radio_f16}; TAG=${2:-r01}
OUT=gpurun_out/prof_${TAG}_${CFG}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
# skip: 2 generator launches + weight pack + 3 warm-up steps x 2 launches; count: 10 timed steps x 2
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -s 9 -c 20 --csv \
  --log-file ${OUT}_launches.csv python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline \
  > ${OUT}_launches_bench.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:cgemm -s 4 -c 1 \
  -o ${OUT}_full -f python bench.py --config $CFG --steps 4 --warmup 3 --no-cpu-baseline \
  > ${OUT}_full.log 2>&1
echo "profile done: $CFG"
