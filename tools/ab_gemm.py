"""A/B of the beamform GEMM alone (packed operands) under environment variants (dev tool).

    AB_VARIANTS="full:,nostore:TCBF_DEBUG=1" python tools/ab_gemm.py b1 32 16384 16384 1 [iters]

AB_DEV_LIB=1 loads the TCBF_DEV build (TCBF_DEBUG ablations honoured: wrong values, timing only).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_03269_b200 as tcbf  # noqa: E402
import synth  # noqa: E402

if os.environ.get("AB_LIB"):       # a specific build (e.g. the previous commit's, for an A/B)
    tcbf.library_path = os.environ["AB_LIB"]
elif os.environ.get("AB_DEV_LIB"):
    from paper_2505_03269_b200 import build as _b
    tcbf.library_path = _b.build_tcbf(dev=True)


def main():
    prec = sys.argv[1]
    M, N, K, B = (int(v) for v in sys.argv[2:6])
    iters = int(sys.argv[6]) if len(sys.argv) > 6 else 50
    seed = synth.SEED_BASE + 4
    w = synth.generate_device("uniform", seed, 0, B, M, K)
    x = synth.generate_device("uniform", seed, 1, B, K, N)
    variants = [("full", {})]
    if os.environ.get("AB_VARIANTS"):
        variants = []
        for item in os.environ["AB_VARIANTS"].split(","):
            name, _, envs = item.partition(":")
            variants.append((name, dict(e.split("=") for e in envs.split(";") if e)))
    ops = 8.0 * M * N * K * B
    byts = B * ((M * K + K * N) / 4.0 + 8 * M * N) if prec == "b1" else B * (4 * M * K + 4 * K * N + 8 * M * N)
    ref = None
    for name, env in variants * int(os.environ.get("AB_REPS", "1")):
        for k in [k for k in os.environ if k.startswith("TCBF_")]:   # every override of the previous variant
            os.environ.pop(k, None)
        os.environ.update(env)
        plan = tcbf.Plan(M, N, K, B, prec)
        wp, xp = plan.pack(tcbf.WEIGHTS, w), plan.pack(tcbf.DATA, x)
        out = plan.alloc_output()
        plan.beamform(wp, xp, out=out)
        torch.cuda.synchronize()
        if ref is None:
            ref = out.clone()
        same = torch.equal(out, ref)
        for _ in range(5):
            plan.beamform(wp, xp, out=out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            plan.beamform(wp, xp, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        print(f"{name:12s} {plan.kernel('beamform'):40s} {ms * 1e3:9.2f} us  {ops / ms / 1e9:9.1f} TeraOps/s  "
              f"{byts / ms / 1e6:8.1f} GB/s  same_as_first={same}", flush=True)


if __name__ == "__main__":
    main()
