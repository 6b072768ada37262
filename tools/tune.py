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
    ("m32_f16_16384", "f16", 32, 16384, 16384, 1, "uniform", "uniform"),
    ("m32_b1_16384", "b1", 32, 16384, 16384, 1, "uniform", "uniform"),
    ("lofar_k512", "f16", 1024, 1024, 512, 256, "phase", "adc"),
    ("ultrasound_f16", "f16", 65536, 256, 8192, 8, "phase_amp", "adc_scaled"),
    ("square_f16_8192", "f16", 8192, 8192, 8192, 1, "uniform", "uniform"),
    ("radio_b1", "b1", 1024, 4096, 512, 256, "phase", "adc"),
    ("square_b1_8192", "b1", 8192, 8192, 8192, 1, "uniform", "uniform"),
]
# packed-operand GEMM variants (tcbf::F16_V_*): 1-CTA 128x128 BK32 / BK64, 1-CTA 128x64, CTA pairs
F16_VARIANTS = {"1cta_k32s4e8": "0", "1cta_k64s3": "1", "1cta_n64": "2", "2cta_256x128": "3", "2cta_256x256": "4"}
# 1-bit: fp4 resident-data TMEM kernel (short K), fp4 (+-1 e2m1, weights in TMEM; the swapped
# small-M kernel for M <= 64), fp4 forced
# unswapped / forced swapped, int8 AND form, legacy b1 mma.sync, CUDA-core popc
B1_VARIANTS = {"tmem": {"TCBF_B1_KERNEL": "tmem"},  # resident data in TMEM (default for Kw <= 24, M > 64)
               "f4": {"TCBF_B1_KERNEL": "f4"}, "f4_noswap": {"TCBF_B1_KERNEL": "f4", "TCBF_NO_SWAP": "1"},
               "f4_swap64": {"TCBF_B1_KERNEL": "f4", "TCBF_B1_SWAP": "64"}, "i8": {"TCBF_B1_KERNEL": "i8"},
               "bmma": {"TCBF_B1_KERNEL": "bmma"}, "popc": {"TCBF_B1_KERNEL": "popc"}}


def _nvml_handle():
    """NVML handle of the current CUDA device, looked up by PCI bus id (NVML ignores
    CUDA_VISIBLE_DEVICES)."""
    try:
        import pynvml
        pynvml.nvmlInit()
        props = torch.cuda.get_device_properties(torch.cuda.current_device())
        bus = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
        try:
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
    except Exception:
        return None, None


NV, NVH = None, None


def energy_mj():
    try:
        return float(NV.nvmlDeviceGetTotalEnergyConsumption(NVH))
    except Exception:
        return None


def measure(fn, min_ms=1000.0):   # >= 1 s per variant: the energy counter's resolution
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
    global NV, NVH
    NV, NVH = _nvml_handle()
    prefix = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/tune"
    only = set(sys.argv[2].split(",")) if len(sys.argv) > 2 else None
    rows = []
    for name, prec, M, N, K, B, wd, xd in SHAPES:
        if only and name not in only:
            continue
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
                variants.append(("fused_raw (conversion inside the GEMM)", {}, "raw"))
                if base.kernel("raw").startswith("f16_tcgen05_fused_tmem"):
                    variants.append(("fused_raw sample-major, data in smem", {"TCBF_F16_FUSED": "smaj"}, "raw"))
            if base.N % 4 == 0 and base.k_packed <= 256:
                variants.append(("fp16 interleaved data, resident (NEXT-1)", {}, "f16i"))
                variants.append(("fp16 interleaved data, streaming (NEXT-1)", {"TCBF_F16I_STREAM": "1"}, "f16i"))
            variants.append(("pack+gemm default", {}, "two"))
        else:
            for v, env in B1_VARIANTS.items():
                variants.append((v, env, "gemm"))
        ref = None
        x16 = x.half() if prec == "f16" else None
        for vname, env, mode in variants:
            for k in [k for k in os.environ if k.startswith("TCBF_")]:
                os.environ.pop(k, None)
            os.environ.update(env)
            plan = tcbf.Plan(M, N, K, B, prec)
            if mode == "gemm":
                fn = lambda: plan.beamform(wp, xp, out)  # noqa: E731
            elif mode == "raw":
                fn = lambda: plan.beamform_raw(wp, x, out=out)  # noqa: E731
            elif mode == "f16i":
                fn = lambda: plan.beamform_f16i(wp, x16, out=out)  # noqa: E731
            else:
                fn = lambda: (plan.pack(tcbf.DATA, x, out=xp), plan.beamform(wp, xp, out))  # noqa: E731
            ms, j = measure(fn)
            same = None
            if mode == "gemm":
                if ref is None:
                    ref = out.clone()
                same = bool(torch.equal(ref, out)) if prec == "b1" else None
            kname = plan.variant if mode == "gemm" else (plan.kernel("raw") if mode == "raw" else
                                                          plan.kernel("f16i") if mode == "f16i" else "pack + " + plan.variant)
            row = {"shape": name, "variant": vname, "kernel": kname,
                   "ms": round(ms, 4), "teraops_s": round(ops / ms / 1e9, 1),
                   "teraops_per_joule": round(ops / j / 1e12, 3) if j else None,
                   "watts": round(j / (ms * 1e-3), 0) if j else None, "bit_identical_to_first": same}
            rows.append(row)
            print(json.dumps(row), flush=True)
        for k in [k for k in os.environ if k.startswith("TCBF_")]:
            os.environ.pop(k, None)
        del wp, x, xp, out, x16
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
