"""A/B of the fused fp32-data 16-bit kernels on a radio-shaped workload (dev tool, not the bench):
sample-major (coalesced line stores from TMEM, 8 or 4 epilogue warps) vs the beam-major TMA-store
kernel, each against pack + beamform (max abs difference and bitwise equality) and CUDA-event timed.

    python tools/ab_fused.py [M N K B] [iters]
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402  (ClockSampler: NVML SM clock / power during each variant)

import paper_2505_03269_b200 as tcbf  # noqa: E402
import synth  # noqa: E402

if os.environ.get("AB_LIB"):       # a specific build (e.g. a compile-time variant under /tmp)
    tcbf.library_path = os.environ["AB_LIB"]
elif os.environ.get("AB_DEV_LIB"):   # ablation studies: the TCBF_DEV build (TCBF_DEBUG honoured)
    from paper_2505_03269_b200 import build as _b
    tcbf.library_path = _b.build_tcbf(dev=True)

VARIANTS = [("tmem", {}), ("tmem64", {"TCBF_F16_FUSED": "tmem"}), ("tmem_nomc", {"TCBF_F16_MC": "0"}),
            ("smaj", {"TCBF_F16_FUSED": "smaj"})]   # tmem = the plan default (32-beam tiles at K16 = 256)
if os.environ.get("AB_VARIANTS"):   # e.g. "smaj8:,nostore:TCBF_DEBUG=1,nomma:TCBF_DEBUG=2"
    VARIANTS = []
    for item in os.environ["AB_VARIANTS"].split(","):
        name, _, envs = item.partition(":")
        VARIANTS.append((name, dict(e.split("=") for e in envs.split(";") if e)))


def main():
    a = [int(v) for v in sys.argv[1:5]] if len(sys.argv) >= 5 else [1024, 1024, 256, 256]
    iters = int(sys.argv[5]) if len(sys.argv) > 5 else 50
    M, N, K, B = a
    seed = synth.SEED_BASE + 1
    w = synth.generate_device("phase", seed, 0, B, M, K)
    x = synth.generate_device("adc", seed, 1, B, K, N)
    ref_plan = tcbf.Plan(M, N, K, B, "f16")
    wp = ref_plan.pack(tcbf.WEIGHTS, w)
    ref = ref_plan.beamform(wp, ref_plan.pack(tcbf.DATA, x))
    torch.cuda.synchronize()
    ops = 8.0 * M * N * K * B
    byts = B * (4 * M * K + 8 * K * N + 8 * M * N)
    reps = int(os.environ.get("AB_REPS", "2"))
    for name, env in VARIANTS * reps:    # interleaved repeats: the board heats up over a run
        for k in [k for k in os.environ if k.startswith("TCBF_")]:   # every override of the previous variant
            os.environ.pop(k, None)
        os.environ.update(env)
        plan = tcbf.Plan(M, N, K, B, "f16")
        out = plan.alloc_output()
        f16i = name.startswith("f16i")   # fp16 interleaved data, tcbf_beamform_f16i (NEXT-1)
        if f16i:
            xh = x.half()
            call = lambda: plan.beamform_f16i(wp, xh, out=out)          # noqa: E731
        else:
            call = lambda: plan.beamform_raw(wp, x, out=out)            # noqa: E731
        call()
        torch.cuda.synchronize()
        diff = (out - ref).abs().max().item()
        same = torch.equal(out, ref)
        for _ in range(5):
            call()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        cs = bench.ClockSampler(torch.device("cuda", 0))
        cs.start()
        mj0 = cs.energy_mj()
        t0 = time.perf_counter()
        e0.record()
        for _ in range(iters):
            call()
        e1.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        mj1 = cs.energy_mj()
        cs.stop()
        ms = e0.elapsed_time(e1) / iters
        clk = statistics.median(cs.samples) if cs.samples else 0
        watts = (mj1 - mj0) * 1e-3 / wall if (mj0 is not None and mj1 is not None) else 0.0
        kname = plan.kernel("f16i") if f16i else plan.raw_variant
        byts_v = byts - (4 * B * K * N if f16i else 0)   # fp16 data: 4 B per complex sample
        print(f"{name:10s} {kname:38s} {ms * 1e3:8.1f} us  {ops / ms / 1e9:7.1f} TeraOps/s  "
              f"{byts_v / ms / 1e6:7.1f} GB/s (algorithmic)  {clk:5.0f} MHz {watts:5.0f} W  bitwise={same} maxdiff={diff:.3g}", flush=True)


if __name__ == "__main__":
    main()
