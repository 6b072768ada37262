#!/bin/bash
# Run bench.py on every BASELINE config (N=1), one JSON line each -> gpurun_out/bench_<tag>_<cfg>.json
TAG=${1:-r01}; shift
CFGS=${@:-"tiny radio_f16 radio_b1 ultrasound_f16 square_f16_1024 square_f16_4096 square_f16_8192 square_f16_16384 square_b1_1024 square_b1_4096 square_b1_8192 square_b1_16384 m32_f16_4096 m32_f16_16384 m32_b1_16384 fig3_f16_small fig3_b1_small"}
mkdir -p gpurun_out
for c in $CFGS; do
  steps=100; [ "$c" = "tiny" ] && steps=2000
  case $c in square_*_16384|ultrasound_f16|square_*_8192) steps=20;; esac
  timeout 600 python bench.py --config $c --steps $steps --warmup 5 ${BENCH_FLAGS:---no-cpu-baseline --no-energy} 2>gpurun_out/bench_${TAG}_${c}.err | tail -1 > gpurun_out/bench_${TAG}_${c}.json
  python -c "import json,sys; d=json.load(open('gpurun_out/bench_${TAG}_${c}.json')); r=d['roofline']; print(f\"{d['config']['workload']:18s} {d['value']:9.2f} TOPS  step {d['ms_per_step']:.4f} ms  gemm {d['config']['gemm_ms']:.4f} pack {d['config']['pack_ms']:.4f}  {r['bound']} {r['achieved']} {r['unit']} frac {r['frac']}  e2e {d['e2e']['value']}  cpu {d.get('cpu_baseline',{}).get('value')}  clk {d['clocks'].get('sm_mhz')} {d['clocks'].get('reasons')}\")" 2>&1 | tail -1
done
