"""Variant tuning table (the analogue of the paper's Table III):
every kernel variant of the beamform GEMM on each BASELINE shape class, timed with CUDA events and
metered with the NVML energy counter -> TeraOps/s and TeraOps/J.  Writes JSON + a markdown table.

    python tools/tune.py [out_prefix]        (on the GPU box)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_03269_b200 as tcbf  # noqa: E402
import synth  # noqa: E402

SHAPES = [  # name, prec, M, N, K, B, wdist, xdist
    ("radio_f16", "f16", 1024, 1024, 256, 256, "phase", "adc"),
    ("lofar_k512", "f16", 1024, 1024, 512, 256, "phase", "adc"),
    ("ultrasound_f16", "f16", 65536, 256, 8192, 8, "phase_amp", "adc_scaled"),
    ("square_f16_8192", "f16", 8192, 8192, 8192, 1, "uniform", "uniform"),
    ("radio_b1", "b1", 1024, 4096, 512, 256, "phase", "adc"),
    ("square_b1_8192", "b1", 8192, 8192, 8192, 1, "uniform", "uniform"),
]
F16_VARIANTS = {"1cta_k64s3": "1", "1cta_coop": "11", "1cta_k32s4e8": "0", "2cta_256x128": "7", "2cta_256x256": "8"}
# 1-bit: fp4 with weights in TMEM (default), fp4 all-smem, fp4 CTA pair, int8, fp8, int8 pair,
# legacy b1 mma.sync, CUDA-core popc
B1_VARIANTS = {"f4": {"TCBF_B1_KERNEL": "f4"}, "f4_smem": {"TCBF_B1_KERNEL": "f4", "TCBF_B1_ATMEM": "0"},
               "f4pair": {"TCBF_B1_KERNEL": "f4pair"}, "i8": {"TCBF_B1_KERNEL": "i8"},
               "f8": {"TCBF_B1_KERNEL": "f8"}, "i8pair": {"TCBF_B1_KERNEL": "i8pair"},
               "bmma": {"TCBF_B1_KERNEL": "bmma"}, "popc": {"TCBF_B1_KERNEL": "popc"}}
ENV_KEYS = ("TCBF_F16_VARIANT", "TCBF_B1_KERNEL", "TCBF_B1_ATMEM")


def energy_mj():
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        return float(pynvml.nvmlDeviceGetTotalEnergyConsumption(h))
    except Exception:
        return None


def measure(fn, min_ms=300.0):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    once = max(e0.elapsed_time(e1), 1e-3)
    iters = max(5, int(min_ms / once))
    j0 = energy_mj()
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    j1 = energy_mj()
    ms = e0.elapsed_time(e1) / iters
    joules = (j1 - j0) / 1e3 / iters if (j0 is not None and j1 is not None) else None
    return ms, joules


def main():
    prefix = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/tune"
    rows = []
    for name, prec, M, N, K, B, wd, xd in SHAPES:
        base = tcbf.Plan(M, N, K, B, prec)
        wp = base.pack(tcbf.WEIGHTS, synth.generate_device(wd, 7, 0, B, M, K))
        x = synth.generate_device(xd, 7, 1, B, K, N)
        xp = base.pack(tcbf.DATA, x)
        out = base.alloc_output()
        ops = 8.0 * M * N * K * B
        variants = []
        if prec == "f16":
            for vname, v in F16_VARIANTS.items():
                variants.append((vname, {"TCBF_F16_VARIANT": v}, "gemm"))
            if base.raw_fused:
                variants.append(("fused_raw (pack+gemm)", {}, "raw"))
            variants.append(("pack+gemm default", {}, "two"))
        else:
            for v, env in B1_VARIANTS.items():
                variants.append((v, env, "gemm"))
        ref = None
        for vname, env, mode in variants:
            for k in ENV_KEYS:
                os.environ.pop(k, None)
            os.environ.update(env)
            plan = tcbf.Plan(M, N, K, B, prec)
            if mode == "gemm":
                fn = lambda: plan.beamform(wp, xp, out)  # noqa: E731
            elif mode == "raw":
                fn = lambda: plan.beamform_raw(wp, x, out=out)  # noqa: E731
            else:
                fn = lambda: (plan.pack(tcbf.DATA, x, out=xp), plan.beamform(wp, xp, out))  # noqa: E731
            ms, j = measure(fn)
            same = None
            if mode == "gemm":
                if ref is None:
                    ref = out.clone()
                same = bool(torch.equal(ref, out)) if prec == "b1" else None
            row = {"shape": name, "variant": vname, "kernel": plan.variant if mode == "gemm" else mode,
                   "ms": round(ms, 4), "teraops_s": round(ops / ms / 1e9, 1),
                   "teraops_per_joule": round(ops / j / 1e12, 3) if j else None,
                   "watts": round(j / (ms * 1e-3), 0) if j else None, "bit_identical_to_first": same}
            rows.append(row)
            print(json.dumps(row), flush=True)
        for k in ENV_KEYS:
            os.environ.pop(k, None)
        del wp, x, xp, out
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(prefix) or ".", exist_ok=True)
    with open(prefix + ".json", "w") as f:
        json.dump(rows, f, indent=1)
    with open(prefix + ".md", "w") as f:
        f.write("| shape | variant | kernel | ms | TeraOps/s | TeraOps/J | W |\n|---|---|---|---|---|---|---|\n")
        for r in rows:
            f.write(f"| {r['shape']} | {r['variant']} | {r['kernel']} | {r['ms']} | {r['teraops_s']} | "
                    f"{r['teraops_per_joule']} | {r['watts']} |\n")


if __name__ == "__main__":
    main()
