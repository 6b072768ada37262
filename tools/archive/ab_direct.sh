TCBF_F16_DIRECT=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "f16_beamform_raw or radio_f16_raw" 2>&1 | tail -3
for r in 1 2; do
for v in "" "TCBF_F16_DIRECT=1" "TCBF_F16_MC=0" "TCBF_F16_DIRECT=1 TCBF_F16_MC=0"; do
  echo "== $v"; env $v timeout 300 python bench.py --config radio_f16 --steps 200 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print(d['value'], d['config']['gemm_ms'], d['roofline']['frac'], d['clocks'])"
done; done
