#!/bin/bash
# Usage (on the GPU box): tools/gpu_profile.sh <config> <tag>
# 1) launch list: per-launch device time (cold-cache, serialised) of EVERY kernel of a short bench
#    run (generator, weight pack, warm-up, timed steps, e2e) -> kernel shares of the listed time
# 2) one ncu --set full capture of the dominant kernel (the beamform GEMM) inside the timed steps
set -u
CFG=${1:-radio_f16}; TAG=${2:-r01}
OUT=gpurun_out/prof_${TAG}_${CFG}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file ${OUT}_launches.csv python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --records "" --no-energy \
  > ${OUT}_launches_bench.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:cgemm -s 4 -c 1 \
  -o ${OUT}_full -f python bench.py --config $CFG --steps 4 --warmup 3 --no-cpu-baseline --records "" --no-energy \
  > ${OUT}_full.log 2>&1
echo "profile done: $CFG"
