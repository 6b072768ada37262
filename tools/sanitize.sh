#!/bin/bash
# compute-sanitizer pass over every kernel of libtcbf.so (tools/sanitize_cases.py), one log per
# tool x case group under gpurun_out/sanitize/.  Usage (GPU box): tools/sanitize.sh [tools...]
set -u
OUT=gpurun_out/sanitize
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
TOOLS=${*:-memcheck racecheck synccheck initcheck}
for tool in $TOOLS; do
  for grp in f16 b1 misc; do
    extra=""
    timeout 600 $CS --tool $tool $extra --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_cases.py $grp > $OUT/${tool}_${grp}.log 2>&1
    echo "$tool $grp rc=$?" | tee -a $OUT/summary.txt
  done
done
