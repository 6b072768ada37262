timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "f16i or ileave or next1" 2>&1 | tail -2
for rep in 1 2 3; do
for L in build/libtcbf_base.so paper_2505_03269_b200/lib/libtcbf.so; do
  echo "== $L"
  AB_LIB=$L AB_VARIANTS="f16i:,smaj:" python tools/ab_fused.py 1024 1024 256 256 200 2>&1 | grep -E "^f16i|^smaj" | head -4
done; done
