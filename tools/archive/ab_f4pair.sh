timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "b1 and f4pair" 2>&1 | tail -1
for d in 0 6 14 15 8; do
  TCBF_B1_KERNEL=f4pair TCBF_DEBUG=$d timeout 300 python bench.py --config square_b1_8192 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('f4pair debug=$d', d['config']['gemm_ms'])"
done
