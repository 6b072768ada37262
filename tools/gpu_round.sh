set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_r02a.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gpu_tests_r02a.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02a.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/smoke_r02a.log | tail -2
timeout 600 python bench.py > gpurun_out/bench_r02a_default.json 2> gpurun_out/bench_r02a_default.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_r02a_default.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --dist-backend gloo --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r02a_gloo2.json 2> gpurun_out/bench_r02a_gloo2.err; echo "gloo2 rc=$?"
tail -c 1500 gpurun_out/bench_r02a_gloo2.json
