"""Time every fp16 kernel variant on a few BASELINE shapes (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_03269_b200 as tcbf
import synth

SHAPES = {"radio": (1024, 1024, 256, 256, "phase", "adc"), "sq8192": (8192, 8192, 8192, 1, "uniform", "uniform"),
          "ultra": (65536, 256, 8192, 8, "phase_amp", "adc_scaled"), "sq4096": (4096, 4096, 4096, 1, "uniform", "uniform"),
          "k512": (1024, 1024, 512, 256, "phase", "adc"), "k384": (1024, 1024, 384, 256, "phase", "adc"),
          "k1024": (1024, 1024, 1024, 64, "phase", "adc"), "sq2048": (2048, 2048, 2048, 1, "uniform", "uniform")}
variants = [int(v) for v in os.environ.get("VARIANTS", "0,1,2,3").split(",")]
for name in sys.argv[1:] or ["radio", "sq8192"]:
    M, N, K, B, wd, xd = SHAPES[name]
    base = tcbf.Plan(M, N, K, B, "f16")
    w = synth.generate_device(wd, 1, 0, B, M, K); wp = base.pack(tcbf.WEIGHTS, w); del w
    x = synth.generate_device(xd, 1, 1, B, K, N); xp = base.pack(tcbf.DATA, x)
    out = base.alloc_output()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(5): base.pack(tcbf.DATA, x, out=xp)
    e0.record()
    for _ in range(10): base.pack(tcbf.DATA, x, out=xp)
    e1.record(); torch.cuda.synchronize()
    pms = e0.elapsed_time(e1) / 10
    print(f"{name}: pack(data) {pms*1e3:.1f} us = {(B*K*N*8 + base.x_bytes)/pms/1e6:.0f} GB/s", flush=True)
    ref = None
    for v in variants:
        os.environ["TCBF_F16_VARIANT"] = str(v)
        plan = tcbf.Plan(M, N, K, B, "f16")
        for _ in range(3): plan.beamform(wp, xp, out)
        torch.cuda.synchronize()
        it = 20 if name == "radio" else 5
        e0.record()
        for _ in range(it): plan.beamform(wp, xp, out)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / it
        if ref is None: ref = out.clone()
        same = torch.equal(ref, out)
        ops = 8.0 * M * N * K * B
        byts = B * (4 * M * K + 4 * K * N + 8 * M * N)
        print(f"  v{v} {plan.variant:34s} {ms*1e3:8.1f} us {ops/ms/1e9:7.1f} TOPS {byts/ms/1e6:6.0f} GB/s same={same}", flush=True)
