# b1 data pack: old (compile-time 32-word chunks) vs new (compile-time 32 / 8 / 2 / 1 word chunks)
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pack_b1 or full_size_m32_b1" 2>&1 | tail -1
cp paper_2505_03269_b200/lib/libtcbf.so /tmp/libtcbf_new.so
cp paper_2505_03269_b200/lib_old/libtcbf.so paper_2505_03269_b200/lib/libtcbf.so
for cfg in radio_b1 m32_b1_16384 m32_b1_4096 square_b1_1024; do
  timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('old $cfg', d['ms_per_step'], d['config']['pack_ms'], d['config']['gemm_ms'])"
done
cp /tmp/libtcbf_new.so paper_2505_03269_b200/lib/libtcbf.so
for cfg in radio_b1 m32_b1_16384 m32_b1_4096 square_b1_1024; do for w in 32 8 2 1 auto; do
  if [ $w = auto ]; then unset TCBF_PACK_WPT; else export TCBF_PACK_WPT=$w; fi
  timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.load(sys.stdin); print('new $cfg wpt=$w', d['ms_per_step'], d['config']['pack_ms'], d['config']['gemm_ms'])"
done; done
