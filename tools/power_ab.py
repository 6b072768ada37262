"""Dev tool: A/B of environment-selected variants of the radio fp16 step with the NVML energy
counter (300 ms loops): python tools/power_ab.py VAR=a,b [VAR2=c,d] -> ms, TeraOps/s, watts."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_03269_b200 as tcbf  # noqa: E402
import synth  # noqa: E402
from tools.tune import measure  # noqa: E402

M, N, K, B = 1024, 1024, 256, 256
plan = tcbf.Plan(M, N, K, B, "f16")
wp = plan.pack(tcbf.WEIGHTS, synth.generate_device("phase", 1, 0, B, M, K))
x = synth.generate_device("adc", 1, 1, B, K, N)
out = plan.alloc_output()
specs = [a.split("=") for a in sys.argv[1:]]
for rep in range(2):
    for var, vals in specs:
        for v in vals.split(","):
            os.environ[var] = v
            ms, j = measure(lambda: plan.beamform_raw(wp, x, out=out))
            print(f"{var}={v}: {ms:.4f} ms  {8 * M * N * K * B / ms / 1e9:.1f} TeraOps/s  "
                  f"{(j / (ms * 1e-3)) if j else float('nan'):.0f} W", flush=True)
            del os.environ[var]
