"""Quick CUDA-event timing of tcbf_beamform on a BASELINE config (dev tool, not the bench)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_03269_b200 as tcbf
import synth

def run(prec, M, N, K, B, wd, xd, iters=10):
    plan = tcbf.Plan(M, N, K, B, prec)
    w = synth.generate_device(wd, 1, 0, B, M, K); wp = plan.pack(tcbf.WEIGHTS, w); del w
    x = synth.generate_device(xd, 1, 1, B, K, N)
    xp = plan.pack(tcbf.DATA, x)
    out = plan.alloc_output()
    for _ in range(3): plan.beamform(wp, xp, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): plan.beamform(wp, xp, out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    ops = 8.0 * M * N * K * B
    byts = B * ((4 * M * K + 4 * K * N) if prec == "f16" else (M * K + K * N) / 4) + 8.0 * B * M * N
    # pack timing
    e0.record()
    for _ in range(iters): plan.pack(tcbf.DATA, x, out=xp)
    e1.record(); torch.cuda.synchronize()
    pms = e0.elapsed_time(e1) / iters
    print(f"{prec} M{M} N{N} K{K} B{B} [{plan.variant}]: {ms*1e3:.1f} us  {ops/ms/1e9:.1f} TeraOps/s  "
          f"{byts/ms/1e6:.1f} GB/s   pack(data) {pms*1e3:.1f} us {(B*K*N*8 + plan.x_bytes)/pms/1e6:.1f} GB/s", flush=True)

cfgs = sys.argv[1:] or ["radio_f16", "radio_b1", "sq8192", "ultra"]
for c in cfgs:
    if c == "radio_f16": run("f16", 1024, 1024, 256, 256, "phase", "adc")
    if c == "radio_b1": run("b1", 1024, 4096, 512, 256, "phase", "adc", iters=3)
    if c == "sq8192": run("f16", 8192, 8192, 8192, 1, "uniform", "uniform", iters=3)
    if c == "ultra": run("f16", 65536, 256, 8192, 8, "phase_amp", "adc_scaled", iters=3)
    if c == "sq_b1": run("b1", 8192, 8192, 8192, 1, "uniform", "uniform", iters=3)
