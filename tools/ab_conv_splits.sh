for cfg in m32_f16_4096 m32_f16_8192; do for sp in auto 4 5 8 9 16; do
  if [ $sp = auto ]; then unset TCBF_CONV_SPLITS; else export TCBF_CONV_SPLITS=$sp; fi
  timeout 300 python bench.py --config $cfg --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$cfg splits=$sp', d['ms_per_step'], d['config']['gemm_ms'], d['roofline']['frac'])"
done; done
