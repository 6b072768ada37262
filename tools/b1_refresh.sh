timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "b1" 2>&1 | tail -1
bash tools/bench_all.sh r01 radio_b1 square_b1_1024 square_b1_4096 square_b1_8192 square_b1_16384 m32_b1_16384 fig3_b1_small 2>&1 | tail -8
timeout 300 python bench.py --config ultrasound_b1_planes --steps 10 --warmup 3 > gpurun_out/bench_r01_ultrasound_b1_planes.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench_r01_ultrasound_b1_planes.json')); print('us_b1_planes', d['value'], d['roofline']['frac'], d['clocks'])"
for c in radio_b1 square_b1_8192; do
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:cgemm_b1 -s 4 -c 1 -o gpurun_out/prof_r01_${c}_full -f python bench.py --config $c --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/prof_r01_${c}_full.log 2>&1
done
