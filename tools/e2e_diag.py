"""Diagnose the end-to-end host pipeline: raw PCIe copy rates vs tcbf_beamform_host."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_03269_b200 as tcbf
import synth
M, N, K, B = 1024, 1024, 256, 256
plan = tcbf.Plan(M, N, K, B, "f16")
wp = plan.pack(tcbf.WEIGHTS, synth.generate_device("phase", 1, 0, B, M, K))
x = synth.generate_device("adc", 1, 1, B, K, N)
x_host = x.cpu().pin_memory()
out_host = torch.empty((B, 2, M, N), dtype=torch.float32).pin_memory()
out_dev = plan.alloc_output()
def t(fn, n=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3
h2d = t(lambda: x.copy_(x_host, non_blocking=True))
d2h = t(lambda: out_host.copy_(out_dev, non_blocking=True))
both = t(lambda: plan.beamform_host(wp, x_host, out_host))
print(f"H2D {x_host.numel()*4/1e9:.2f} GB: {h2d:.1f} ms ({x_host.numel()*4/h2d/1e6:.1f} GB/s); "
      f"D2H {out_host.numel()*4/1e9:.2f} GB: {d2h:.1f} ms ({out_host.numel()*4/d2h/1e6:.1f} GB/s); "
      f"beamform_host {both:.1f} ms")
