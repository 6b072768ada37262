"""Dev tool: timeline of the swapped small-M 1-bit kernel's first tile (TCBF_TRACE, dev build):
per K block when the packed words were requested, when the data expander got the stage / handed
its block over, when the weight expanders handed the stage (two K blocks) over, when the MMA
issuer got the stage."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_03269_b200 as tcbf  # noqa: E402
from paper_2505_03269_b200 import build as _b  # noqa: E402
import synth  # noqa: E402

tcbf.library_path = _b.build_tcbf(dev=True)
M, N, K = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (32, 16384, 16384)))
plan = tcbf.Plan(M, N, K, 1, "b1")
wp = plan.pack(tcbf.WEIGHTS, synth.generate_device("uniform", 5, 0, 1, M, K))
xp = plan.pack(tcbf.DATA, synth.generate_device("uniform", 5, 1, 1, K, N))
out = plan.alloc_output()
for _ in range(10):
    plan.beamform(wp, xp, out=out)
torch.cuda.synchronize()
os.environ["TCBF_TRACE"] = "/tmp/swap_trace.bin"
plan.beamform(wp, xp, out=out)
torch.cuda.synchronize()
t = np.fromfile("/tmp/swap_trace.bin", dtype=np.uint64).reshape(-1, 1024).astype(np.int64)
for cta in (0, 57):
    r = t[cta]
    t0 = min(v for v in (r[512], r[0]) if v > 0)
    f = lambda v: f"{(v - t0) / 1e3:7.2f}" if v > 0 else "      -"
    print(f"CTA {cta}: tile done at {f(r[1000])} us")
    print("  kb  tma-issue  pfull  xexp-empty  xexp-full  wexp-full  mma-got (stage = kb // 2 for M <= 32)")
    for kb in list(range(0, 12)) + list(range(28, 36)) + list(range(56, 64)):
        print(f"  {kb:2d}  {f(r[512 + kb // 4]) if kb % 4 == 0 else '       '}  "
              f"{f(r[128 + kb // 4]) if kb % 4 == 0 else '       '}  "
              f"{f(r[256 + kb])}  {f(r[384 + kb])}  {f(r[640 + kb // 2])}  {f(r[kb // 2])}")
