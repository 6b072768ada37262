for rep in 1 2; do
python bench.py --config m32_b1_16384 --steps 100 --warmup 5 --no-cpu-baseline --no-energy --records "" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new', d['config']['gemm_ms'])"
cp paper_2505_03269_b200/lib/libtcbf.so /tmp/new.so; cp build/libtcbf_head.so paper_2505_03269_b200/lib/libtcbf.so
python bench.py --config m32_b1_16384 --steps 100 --warmup 5 --no-cpu-baseline --no-energy --records "" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('head', d['config']['gemm_ms'])"
cp /tmp/new.so paper_2505_03269_b200/lib/libtcbf.so
done
