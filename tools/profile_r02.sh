#!/bin/bash
# Round-2 profile set (GPU box): launch list + one ncu --set full capture per config.
for c in ${@:-radio_f16 radio_b1 ultrasound_f16 radio_f16i}; do
  bash tools/gpu_profile.sh $c r02
done
