# fp4 1-bit kernel with the expanded weights in TENSOR memory (TCBF_B1_ATMEM=1) vs smem; parity first
TCBF_B1_ATMEM=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "b1 and (f4] or f4-) and not f4pair" 2>&1 | tail -3
TCBF_B1_ATMEM=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "full_size_square_16384 or ultrasound_b1" 2>&1 | tail -1
for cfg in square_b1_4096 square_b1_8192 radio_b1 square_b1_16384; do for v in 0 1; do
  TCBF_B1_ATMEM=$v timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$cfg atmem=$v', d['value'], d['config']['gemm_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
