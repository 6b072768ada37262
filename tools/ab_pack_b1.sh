# 1-bit data pack (pack_b1_transpose): words-per-thread chunk A/B (TCBF_PACK_WPT = 32, 8, 2, 1 or the
# size-based default) on the configs whose step the pack dominates
for cfg in radio_b1 m32_b1_16384 m32_b1_4096 square_b1_1024; do for w in 32 8 2 1 auto; do
  if [ $w = auto ]; then unset TCBF_PACK_WPT; else export TCBF_PACK_WPT=$w; fi
  timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('$cfg wpt=$w', d['ms_per_step'], d['config']['pack_ms'], d['config']['gemm_ms'])"
done; done
