# upper bound of an early-TMEM-release epilogue in the fp4 1-bit kernel (TCBF_DEBUG=8, wrong values)
for cfg in square_b1_4096 square_b1_8192 radio_b1; do
for v in 0 8 0 8; do
  TCBF_B1_PACK16=0 TCBF_DEBUG=$v timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$cfg debug=$v', d['value'], d['config']['gemm_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
