#!/bin/bash
# LOFAR station sweep (Fig. 7): radio fp16, 1024 beams x 1024 samples x 256
# channels, K = 8 .. 512 stations; one bench line per K -> gpurun_out/lofar_<tag>.txt
TAG=${1:-r02}
mkdir -p gpurun_out
for k in 8 16 32 48 64 96 128 192 256 384 512; do
  timeout 300 python bench.py --config lofar_k$k --steps 50 --warmup 5 --no-cpu-baseline --no-energy --records "" 2>/dev/null | tail -1 > gpurun_out/lofar_${TAG}_k$k.json
  python - gpurun_out/lofar_${TAG}_k$k.json $k <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d["roofline"]; c = d["config"]
print(f"| {sys.argv[2]} | {d['value']:.1f} | {d['ms_per_step']:.4f} | {r['kernel']} | {r['bound']} {r['frac']} | {c['samples_per_s']/1e6:.1f} |")
PY
done
