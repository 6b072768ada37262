"""Time tcbf_beamform_raw (fused) vs pack + beamform on a config (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_03269_b200 as tcbf
import synth
SH = {"radio": (1024, 1024, 256, 256, "phase", "adc"), "fig3": (1024, 1024, 64, 256, "uniform", "uniform"),
      "m32": (32, 16384, 16384, 1, "uniform", "uniform"), "m32_8192": (32, 8192, 8192, 1, "uniform", "uniform"),
      "m128_k8192": (128, 16384, 8192, 2, "uniform", "uniform"),
      "m32_n8k16": (32, 8192, 16384, 1, "uniform", "uniform"), "m32_n16k8": (32, 16384, 8192, 1, "uniform", "uniform"),
      "m32_n32k8": (32, 32768, 8192, 1, "uniform", "uniform"), "m32_n4096": (32, 4096, 4096, 1, "uniform", "uniform")}
SPLITS = os.environ.pop("SWEEP_SPLITS", "").split(",") if os.environ.get("SWEEP_SPLITS") else []
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
    xb = 8.0 * B * K * N
    print(f"{name}: fused raw {t_raw*1e3:.1f} us ({ops/t_raw/1e9:.0f} TOPS, data {xb/t_raw/1e6:.0f} GB/s) | "
          f"pack+gemm {t_two*1e3:.1f} us ({ops/t_two/1e9:.0f} TOPS)", flush=True)
    for sp in SPLITS:
        os.environ["TCBF_CONV_SPLITS"] = sp
        t = tm(lambda: plan.beamform_raw(wp, x, out=out))
        print(f"   splits={sp}: {t*1e3:.1f} us ({ops/t/1e9:.0f} TOPS, data {xb/t/1e6:.0f} GB/s)", flush=True)
        os.environ.pop("TCBF_CONV_SPLITS")
