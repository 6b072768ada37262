#!/bin/bash
# GPU-box validation pass: the -m gpu suite, smoke(), the default bench line, optional extra configs.
# Usage: bash tools/gpu_round.sh <tag> [extra bench configs...]
TAG=${1:-r02}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/gpu_tests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}_default.json 2> gpurun_out/bench_${TAG}_default.err; echo "bench rc=$?"
python - gpurun_out/bench_${TAG}_default.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
recs = d.pop("records", {})
r = d["roofline"]
print("default", d["value"], d["unit"], d["ms_per_step"], "ms", r["kernel"], "frac", r["frac"], r.get("frac_kernel_bytes"), "e2e", d["e2e"]["value"], "clk", d["clocks"])
for k, v in recs.items():
    print("  rec", k, v["value"], v["ms_per_step"], v["roofline"]["kernel"], v["roofline"]["frac"])
PY
for c in "$@"; do
  timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline --no-energy --records "" 2>/dev/null | tail -1 > gpurun_out/bench_${TAG}_$c.json
  python - gpurun_out/bench_${TAG}_$c.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
c = d["config"]; r = d["roofline"]; g = r.get("gemm", r)
print(c["workload"], d["value"], d["ms_per_step"], "gemm", c["gemm_ms"], "pack", c["pack_ms"], r["kernel"], r["frac"], "| gemm", g["kernel"], g["frac"], g["achieved"], g["unit"])
PY
done
