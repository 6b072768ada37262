"""Time tcbf_beamform_raw (fused) vs pack + beamform on a config (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_03269_b200 as tcbf
import synth
SH = {"radio": (1024, 1024, 256, 256, "phase", "adc"), "fig3": (1024, 1024, 64, 256, "uniform", "uniform")}
for name in sys.argv[1:] or ["radio"]:
    M, N, K, B, wd, xd = SH[name]
    plan = tcbf.Plan(M, N, K, B, "f16")
    wp = plan.pack(tcbf.WEIGHTS, synth.generate_device(wd, 1, 0, B, M, K))
    x = synth.generate_device(xd, 1, 1, B, K, N)
    xp = plan.alloc_packed(tcbf.DATA); out = plan.alloc_output()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    def tm(fn, it=20):
        for _ in range(3): fn()
        torch.cuda.synchronize(); e0.record()
        for _ in range(it): fn()
        e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / it
    t_raw = tm(lambda: plan.beamform_raw(wp, x, out=out))
    t_two = tm(lambda: (plan.pack(tcbf.DATA, x, out=xp), plan.beamform(wp, xp, out)))
    ops = 8.0 * M * N * K * B
    print(f"{name}: fused raw {t_raw*1e3:.1f} us ({ops/t_raw/1e9:.0f} TOPS) | pack+gemm {t_two*1e3:.1f} us ({ops/t_two/1e9:.0f} TOPS)")
