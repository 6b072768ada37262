#!/usr/bin/env python
"""Benchmark of the B200 Tensor-Core Beamformer hot path (BASELINE.json metric:
"beamforming TeraOps/s (fp16 and 1-bit) at 1/2/4/8 B200 vs roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config radio_f16] [--impl tcbf|reference]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N --steps K --warmup W

A step = one pass of the hot path over one batch of synthetic data resident in HBM:
the fp32 data -> packed operand conversion (§8 a1/a2) + the beamform GEMM (§8 a3-a6), i.e.
tcbf_beamform_raw -- one fused kernel for short-K fp16 plans (each data element converted
once inside the GEMM), otherwise tcbf_pack(DATA) + tcbf_beamform.  The weights are packed
once before timing (the model matrix is prepared once;
PAPER.md:48: weights constant over a period).  Useful ops = 8*B*M*N*K.
Multi-GPU: STRONG scaling of the fixed config -- the global batch is split into
contiguous slices (radio: 256 channels -> 32 per rank at N=8), or, when the batch is smaller than
the world (square / M=32 sweeps), the samples N are split in multiples of 4 with the weights
replicated; K is never split, so there is no data-path collective.  Inputs are generated from
global indices, so every N computes the same global problem.  value = global useful ops / (max
over ranks of the CUDA-event step time).  The optional NCCL output gather (--gather) is timed
separately and never enters `value`.
Default workload = BASELINE configs[1] (radio astronomy fp16, LOFAR-shaped); the
same run also times radio 1-bit (configs[2]) and ultrasound fp16 (configs[3]) under `records`,
so the driver-timed line carries both precisions of the metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

L2_BYTES = 126 * 2 ** 20


def _cfg(prec, M, N, K, B, wd, xd, idx, desc):
    return dict(prec=prec, M=M, N=N, K=K, B=B, wd=wd, xd=xd, idx=idx, desc=desc)


CONFIGS = {
    "tiny": _cfg("f16", 8, 64, 32, 2, "uniform", "uniform", 0,
                 "tiny fp16: M=8 beams, K=32 receivers, N=64 samples, batch=2"),
    "radio_f16": _cfg("f16", 1024, 1024, 256, 256, "phase", "adc", 1,
                      "radio astronomy fp16: M=1024 beams, K=256 stations, N=1024 samples, batch=256 channels"),
    "radio_b1": _cfg("b1", 1024, 4096, 512, 256, "phase", "adc", 2,
                     "radio astronomy 1-bit: M=1024 beams, K=512 stations, N=4096 samples, batch=256 channels"),
    "ultrasound_f16": _cfg("f16", 65536, 256, 8192, 8, "phase_amp", "adc_scaled", 3,
                           "computational ultrasound fp16: M=65536 pixels, K=8192, N=256 frames, batch=8"),
    # ultrasound 1-bit real-time pipeline (Fig. 5): three orthogonal 128^2 planes,
    # K = 128 frequencies x 64 transceivers x 32 transmissions, a block of 1024 frames per step
    "ultrasound_b1_planes": _cfg("b1", 3 * 128 * 128, 1024, 128 * 64 * 32, 1, "phase_amp", "adc_scaled", 3,
                                 "ultrasound 1-bit: M=49152 voxels (3 planes), K=262144, N=1024 frames"),
    # NEXT-1: the radio shape with the data already fp16 interleaved (an fp16 producer,
    # PAPER.md:103), beamformed with no data pack by tcbf_beamform_f16i
    "radio_f16i": dict(_cfg("f16", 1024, 1024, 256, 256, "phase", "adc", 1,
                            "radio fp16, data delivered as interleaved fp16 (no pack): M=1024, K=256, N=1024, "
                            "batch=256"), src="f16i"),
    # Fig. 3 extra rows
    "fig3_f16_small": _cfg("f16", 1024, 1024, 64, 256, "uniform", "uniform", 4, "fp16 small 256x1024x1024x64"),
    "fig3_b1_small": _cfg("b1", 1024, 1024, 256, 256, "uniform", "uniform", 4, "int1 small 256x1024x1024x256"),
}
# LOFAR station sweep (Fig. 7): 1024 beams, 1024 samples, batch 256, K = 8..512
for _k in (8, 16, 32, 48, 64, 96, 128, 192, 256, 384, 512):
    CONFIGS[f"lofar_k{_k}"] = _cfg("f16", 1024, 1024, _k, 256, "phase", "adc", 1,
                                   f"LOFAR station sweep fp16: M=1024 beams, K={_k} stations, N=1024, batch=256")
for _n in (1024, 2048, 4096, 8192, 16384):
    CONFIGS[f"square_f16_{_n}"] = _cfg("f16", _n, _n, _n, 1, "uniform", "uniform", 4, f"square fp16 M=N=K={_n}")
    CONFIGS[f"square_b1_{_n}"] = _cfg("b1", _n, _n, _n, 1, "uniform", "uniform", 4, f"square 1-bit M=N=K={_n}")
    CONFIGS[f"m32_f16_{_n}"] = _cfg("f16", 32, _n, _n, 1, "uniform", "uniform", 4, f"M=32 fp16 N=K={_n}")
    CONFIGS[f"m32_b1_{_n}"] = _cfg("b1", 32, _n, _n, 1, "uniform", "uniform", 4, f"M=32 1-bit N=K={_n}")


def useful_ops(c):
    return 8.0 * c["M"] * c["N"] * c["K"] * c["B"]


def gemm_bytes(c, fused=False):
    """Algorithmic bytes of one beamform launch (PAPER.md:319 'theoretical amount
    of bytes'): logical inputs read once, output written once.  The fused kernel reads the data
    as fp32 complex (8 B) instead of the packed fp16 operand (4 B)."""
    B, M, N, K = c["B"], c["M"], c["N"], c["K"]
    if c["prec"] == "f16":
        return B * (4 * M * K + (8 if fused else 4) * K * N + 8 * M * N)
    return B * ((M * K + K * N) / 4.0 + 8 * M * N)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return dict(hbm=float(d["hbm_gbs"]), bf16=float(d["bf16_tflops"]),
                    bf16_sus=float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), src="measured")
    except Exception:
        return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, src="fallback")


def roofline_for(c, gemm_ms, peaks, long_step, variant="", fused=False):
    """Dominant kernel = the beamform GEMM.  Binding roof = the slower of the HBM time
    (algorithmic bytes / measured copy bandwidth) and the tensor time (useful ops / peak):
    fp16 tensor peak = measured bf16 peak (same nominal rate); the 1-bit tensor-core kernels
    run fp4 (default, 4x fp16 nominal) or int8 / fp8 MMAs (2x) -> 4x or 2x measured bf16.  The
    CUDA-core popc kernel (TCBF_B1_KERNEL=popc) reports 'alu' against 16 POPC/clk/SM."""
    ops = useful_ops(c)
    byts = gemm_bytes(c, fused)
    bw = peaks["hbm"]
    t_ms = gemm_ms * 1e-3
    if c["prec"] == "b1" and "mma_sync" in variant:
        # legacy b1 mma.sync (emulated on sm_100a): its register-only peak measured by peaks.cu
        # (profiles/r01/peaks.json); single-AND form = 4 binary MACs per complex MAC, useful = raw
        try:
            with open(os.path.join(ROOT, "profiles", "r01", "peaks.json")) as f:
                bpeak = float(json.load(f)["peaks"]["b1_mma_sync_and_popc"]["tera_ops_per_s"])
            bsrc = "measured (peaks.cu register-only mma.sync .and.popc, profiles/r01/peaks.json)"
        except Exception:
            bpeak, bsrc = 413.0, "fallback (round-1 peaks.cu measurement)"
        ach = ops / t_ms / 1e12
        return dict(bound="b1_mma_sync", achieved=round(ach, 1), peak=bpeak, unit="TOP/s",
                    frac=round(ach / bpeak, 4), peak_src=bsrc)
    if c["prec"] == "b1" and "popc" in variant:
        alu_peak = 16 * 148 * 1.965e9 * 32 * 2 / 1e12
        ach = ops / t_ms / 1e12
        return dict(bound="alu", achieved=round(ach, 1), peak=round(alu_peak, 1), unit="TOP/s",
                    frac=round(ach / alu_peak, 4), peak_src="derived (16 POPC/clk/SM x 148 x 1965 MHz)")
    # fp16: 1x bf16; 1-bit on int8 MMAs (i8 / i8pair): 2x; on +-1 e4m3 (f8): 2x; on +-1 e2m1
    # with unit block scales (mxf4): 4x -- B200 nominal dense 2.25 / 4.5 / 4.5 / 9 P(FL)OP/s
    ratio = 1.0 if c["prec"] == "f16" else (4.0 if "mxf4" in variant else 2.0)
    # sustained = cuBLAS bf16 back to back at the board's power cap; the narrow-precision 1-bit
    # kernels draw less power per op than that, so a long step of theirs keeps the burst base
    # (x ratio) -- with the sustained base the fp4 planes workload read 1.13 of its "peak"
    base = peaks["bf16_sus"] if (long_step and ratio == 1.0) else peaks["bf16"]
    tpeak = base * ratio
    t_hbm = byts / (bw * 1e9)
    t_tc = ops / (tpeak * 1e12)
    src = peaks["src"] + (" sustained" if (long_step and ratio == 1.0) else " burst") + {
        1.0: "", 2.0: " x2 (int8/fp8 nominal ratio)", 4.0: " x4 (fp4 nominal ratio)"}[ratio]
    if t_hbm >= t_tc:
        # achieved = SURVEY.md §8(d)'s per-unit bytes as written (fp16: data counted at its packed
        # size, 4 B per complex sample, even for the fused kernel that reads it as fp32)
        b8 = gemm_bytes(c, False)
        ach = b8 / t_ms / 1e9
        r = dict(bound="hbm", achieved=round(ach, 1), peak=bw, unit="GB/s", frac=round(ach / bw, 4),
                 peak_src=peaks["src"], tensor_frac=round(ops / t_ms / 1e12 / tpeak, 4))
        if fused:
            # the bytes this launch must move (fp32 data read, 8 B per complex sample): context
            r["frac_kernel_bytes"] = round(byts / t_ms / 1e9 / bw, 4)
            r["kernel_bytes_per_launch"] = byts
        return r
    ach = ops / t_ms / 1e12
    return dict(bound="tensor", achieved=round(ach, 1), peak=round(tpeak, 1), unit="TOP/s" if ratio > 1 else "TFLOP/s",
                frac=round(ach / tpeak, 4), peak_src=src, hbm_frac=round(byts / t_ms / 1e9 / bw, 4))


def pack_roofline(c, pack_ms, packed_bytes, peaks):
    """tcbf_pack(DATA) as the dominant kernel: HBM-bound stream, algorithmic bytes = the fp32
    complex source read once (8 B per element) + the packed operand written once."""
    byts = c["B"] * c["K"] * c["N"] * 8 + packed_bytes
    ach = byts / (pack_ms * 1e-3) / 1e9
    bw = peaks["hbm"]
    return dict(bound="hbm", achieved=round(ach, 1), peak=bw, unit="GB/s", frac=round(ach / bw, 4),
                peak_src=peaks["src"], kernel="pack_b1_transpose" if c["prec"] == "b1" else "pack_f16_rows",
                kernel_ms=round(pack_ms, 4), algorithmic_bytes_per_launch=byts)


def traffic_for(c_name, kernel):
    """dram bytes per launch from the committed ncu --set full capture (profiles/traffic.json) of
    the same config and kernel, or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d.get(c_name)
        if e and e.get("kernel") == kernel:
            return e.get("dram_bytes_per_launch")
    except Exception:
        pass
    return None


class ClockSampler:
    """NVML sampling of SM clock and clock-event reasons during the timed region."""
    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
             0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
             0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device, sample=True):
        """device: the torch CUDA device this rank runs on.  NVML ignores CUDA_VISIBLE_DEVICES, so
        the NVML handle is looked up by the device's PCI bus id, not by the CUDA ordinal."""
        self.samples, self.reasons, self.ok = [], 0, False
        self.max_mhz = None
        self.sample = sample
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            self.nv = pynvml
            props = torch.cuda.get_device_properties(device)
            bus = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
            try:
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.01)

    def energy_mj(self):
        """Total energy counter in mJ (NVML; PAPER.md:278 measures TOPs/J the same way via PMT)."""
        try:
            return float(self.nv.nvmlDeviceGetTotalEnergyConsumption(self.h))
        except Exception:
            return None

    def start(self):
        if self.ok:
            self.e0 = self.energy_mj()
            if self.sample:
                self.t = threading.Thread(target=self._run, daemon=True)
                self.t.start()

    def stop(self):
        if self.ok:
            if self.sample:
                self._stop.set()
                self.t.join()
            self.e1 = self.energy_mj()

    def joules(self):
        if not self.ok or getattr(self, "e0", None) is None or getattr(self, "e1", None) is None:
            return None
        return (self.e1 - self.e0) / 1e3

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        active = [n for bit, n in self.NAMES.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": active,
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------- CPU oracle
def oracle_sample(c, seconds, rank_b0=0, budget_rows=None):
    """Time the oracle (as it stands) on a bounded sample of the workload: the first `rows`
    beams of batch entry 0 (all N samples, all K receivers).  Returns (ops/s, rows, sec)."""
    import numpy as np
    import oracle
    import synth
    seed = synth.SEED_BASE + c["idx"]
    M, N, K, B = c["M"], c["N"], c["K"], c["B"]
    x = synth.to_interleaved(synth.generate(c["xd"], seed, 1, B, K, N, b_sel=[rank_b0]))

    def run(rows):
        w = synth.to_interleaved(synth.generate(c["wd"], seed, 0, B, M, K, b_sel=[rank_b0], r_sel=slice(0, rows)))
        t0 = time.perf_counter()
        if c["prec"] == "f16":
            oracle.cgemm_f16(w, x, 0, rows, N, K, 1)
        else:
            oracle.cgemm_b1(w, x, 0, rows, N, K, 1)
        return time.perf_counter() - t0

    rows = budget_rows or min(M, 4)
    t = run(rows)
    if budget_rows is None:
        while t < seconds * 0.25 and rows < M:
            rows = min(M, max(rows + 1, int(rows * min(8.0, seconds / max(t, 1e-4)))))
            t = run(rows)
    ops = 8.0 * rows * N * K
    return ops / t, rows, t


def cpu_baseline(c, seconds=10.0):
    """The oracle as it stands, on the box's host cores, over a bounded sample of the workload:
    whole batch entries (all M beams, N samples, K receivers) in order until ~`seconds` of oracle
    time (or the whole workload); rows of entry 0 only if one entry alone exceeds the budget."""
    os.environ["OMP_NUM_THREADS"] = str(os.cpu_count())   # before liboracle (libgomp) loads
    import oracle
    import synth
    rate, rows, t = oracle_sample(c, seconds)
    if rows < c["M"]:
        desc = f"beams 0..{rows - 1} of batch entry 0 (all N={c['N']}, K={c['K']})"
        tot_ops, tot_t = 8.0 * rows * c["N"] * c["K"], t
    else:
        seed = synth.SEED_BASE + c["idx"]
        M, N, K, B = c["M"], c["N"], c["K"], c["B"]
        tot_ops, tot_t, nb = 0.0, 0.0, 0
        while nb < B and tot_t < seconds:
            w = synth.to_interleaved(synth.generate(c["wd"], seed, 0, B, M, K, b_sel=[nb]))
            x = synth.to_interleaved(synth.generate(c["xd"], seed, 1, B, K, N, b_sel=[nb]))
            t0 = time.perf_counter()
            if c["prec"] == "f16":
                oracle.cgemm_f16(w, x, 0, M, N, K, 1)
            else:
                oracle.cgemm_b1(w, x, 0, M, N, K, 1)
            tot_t += time.perf_counter() - t0
            tot_ops += 8.0 * M * N * K
            nb += 1
        desc = f"batch entries 0..{nb - 1} of {B} (all M={M}, N={N}, K={K})"
    return {"value": round(tot_ops / tot_t / 1e12, 6), "unit": "TeraOps/s", "cores": os.cpu_count(),
            "kind": "oracle",
            "sample": f"oracle (C, fp64/int64 triple loop, OpenMP {os.cpu_count()} threads) on {desc}; "
                      f"{tot_t:.1f} s of oracle time"}


def run_reference(args, c):
    """--impl reference: the oracle as it stands is this tier's reference arm."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    # torchrun exports OMP_NUM_THREADS=1; the oracle is timed on all host cores (reported below)
    os.environ["OMP_NUM_THREADS"] = str(os.cpu_count())
    import numpy as np  # noqa: F401
    budget = max(0.05, min(0.5, 150.0 / max(1, args.steps + args.warmup)))
    rate, rows, t = oracle_sample(c, budget * 4)
    # rows chosen so one step ~ budget seconds
    rows = max(1, min(c["M"], int(rows * budget / max(t, 1e-6))))
    for _ in range(args.warmup):
        oracle_sample(c, 0, budget_rows=rows)
    times = []
    for s in range(args.steps):
        r, _, tt = oracle_sample(c, 0, budget_rows=rows)
        times.append(tt)
    tot = sum(times)
    ops = 8.0 * rows * c["N"] * c["K"] * args.steps
    val = ops / tot / 1e12
    sample = (f"each step: oracle on beams 0..{rows - 1} of batch entry 0 (N={c['N']}, K={c['K']}), "
              f"{os.cpu_count()} OpenMP threads")
    line = {"metric": "beamforming TeraOps/s (fp16 and 1-bit) at 1/2/4/8 B200 vs roofline", "impl": "reference",
            "value": round(val, 6), "unit": "TeraOps/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(tot / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64" if c["prec"] == "f16" else "int64",
            "data": "synthetic (seeded counter-based generator, synth/)",
            "config": {"workload": args.config, "desc": c["desc"], "M": c["M"], "N": c["N"], "K": c["K"],
                       "global_batch": c["B"], "batch_per_gpu": c["B"],
                       "note": "rank 0 alone runs the oracle on a bounded sample of the global problem"},
            "cpu_baseline": {"value": round(val, 6), "unit": "TeraOps/s", "cores": os.cpu_count(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": round(val, 6), "unit": "TeraOps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------- GPU arm
def pack_weights(plan, c, seed, dev, b0, max_src_bytes=8 << 30):
    """Generate + pack the weights once (outside the timed region).  Model matrices whose fp32
    source would not fit comfortably (ultrasound 1-bit: 103 GB) are generated and packed in row
    slices of the same global index space and copied into the plan's [B][2][M][Kp] layout."""
    import torch

    import paper_2505_03269_b200 as tcbf
    import synth
    B, M, K = c["B"], c["M"], c["K"]
    if B * M * K * 8 <= max_src_bytes:
        wsrc = synth.generate_device(c["wd"], seed, 0, B, M, K, device=dev, b0=b0)
        return plan.pack(tcbf.WEIGHTS, wsrc)
    wp = plan.alloc_packed(tcbf.WEIGHTS, dev)
    rows = max(1, max_src_bytes // (K * 8))
    for b in range(B):
        for m0 in range(0, M, rows):
            mr = min(rows, M - m0)
            sub = tcbf.Plan(mr, c["N"], K, 1, c["prec"])
            # rows m0..m0+mr of entry b0+b of the global [*, M, K] weight tensor
            src = synth.generate_device(c["wd"], seed, 0, 1, mr, K, device=dev, b0=0,
                                        offset_elems=((b0 + b) * M + m0) * K)
            part = sub.pack(tcbf.WEIGHTS, src)
            del src
            wp[b, :, m0:m0 + mr].copy_(part[0])
            del part
    torch.cuda.synchronize()
    return wp


def setup_dist(args):
    """One process per GPU (torchrun env), NCCL; --dist-backend gloo is the single-GPU test mode in
    which every rank shares cuda:0 (exercises the N>1 code path on one device)."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dist_backend == "gloo":
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return world, rank, local, torch.device("cuda", local)


def shard_inputs(c, sh, seed, dev):
    """This rank's plan, packed weights and fp32 data of the GLOBAL problem c:
    batch slices b0..b0+nb (inputs generated from the global index space), or -- batch smaller
    than the world -- sample columns n0..n0+nn of every batch entry with the weights replicated.
    K is never split, so no rank needs another rank's partial sums."""
    import paper_2505_03269_b200 as tcbf
    import synth
    M, N, K = c["M"], c["N"], c["K"]
    if sh.mode == "samples":
        plan = tcbf.Plan(M, sh.nn, K, c["B"], c["prec"])
        wp = pack_weights(plan, dict(c, N=sh.nn), seed, dev, 0)
        xfull = synth.generate_device(c["xd"], seed, 1, c["B"], K, N, device=dev, b0=0)
        xsrc = xfull[:, :, sh.n0:sh.n0 + sh.nn].contiguous()
        del xfull
    else:
        plan = tcbf.Plan(M, N, K, sh.nb, c["prec"])
        wp = pack_weights(plan, dict(c, B=sh.nb), seed, dev, sh.b0)
        xsrc = synth.generate_device(c["xd"], seed, 1, sh.nb, K, N, device=dev, b0=sh.b0)
    return plan, wp, xsrc


def measure(args, name, c, world, rank, local, dev, steps, warmup, e2e=False, energy=False, sample_clocks=True):
    """Time `steps` steps of workload c (the global problem, sharded over the world) and return
    its record: ms_per_step (max over ranks), whole-job TeraOps/s, the dominant kernel's roofline,
    clocks, optionally e2e through the host-buffer API and a >= 1 s energy loop."""
    import torch
    import torch.distributed as dist

    import paper_2505_03269_b200 as tcbf
    import synth
    from paper_2505_03269_b200.shard import max_over_ranks, plan_shard

    sh = plan_shard(c["B"], c["N"], rank, world)
    seed = synth.SEED_BASE + c["idx"]
    plan, wp, xsrc = shard_inputs(c, sh, seed, dev)
    lc = dict(c, B=plan.batch, N=plan.N)   # this rank's share
    f16i = c.get("src") == "f16i"
    if f16i:   # the producer delivers interleaved fp16 (conversion outside the timed region)
        xsrc = xsrc.half()
    fused = plan.raw_fused and not f16i
    xp = plan.alloc_packed(tcbf.DATA, dev)
    out = plan.alloc_output(dev)
    torch.cuda.synchronize()

    working = xsrc.numel() * xsrc.element_size() + plan.x_bytes + plan.w_bytes + plan.out_bytes
    flush = working < 4 * L2_BYTES
    flush_buf = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device=dev) if flush else None
    stream = torch.cuda.current_stream(dev)

    def step(ev=None):
        if f16i:
            if ev: ev[1].record(stream)
            plan.beamform_f16i(wp, xsrc, out=out, stream=stream)
        elif fused:
            if ev: ev[1].record(stream)
            plan.beamform_raw(wp, xsrc, out=out, stream=stream)
        else:
            plan.pack(tcbf.DATA, xsrc, out=xp, stream=stream)
            if ev: ev[1].record(stream)
            plan.beamform(wp, xp, out, stream=stream)

    for _ in range(warmup):
        if flush:
            flush_buf.fill_(1.0)
        step()
    torch.cuda.synchronize()
    # kernels per step, as the library counts them (pack: 1; beamform: 1, or memset + kernel on split K)
    launches_per_step = tcbf.Plan.last_launch_count() + (0 if (f16i or fused) else 1)

    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    sampler = ClockSampler(dev) if sample_clocks else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
    for i in range(steps):
        if flush:
            flush_buf.fill_(float(i))   # evict L2 between timed steps (not inside the timed spans)
        ev[i][0].record(stream)
        step(ev[i])
        ev[i][2].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    if sampler:
        sampler.stop()
    if flush:
        total_ms = sum(e[0].elapsed_time(e[2]) for e in ev)
    else:
        total_ms = ev[0][0].elapsed_time(ev[-1][2])
    gemm_ms = sum(e[1].elapsed_time(e[2]) for e in ev) / steps
    pack_ms = sum(e[0].elapsed_time(e[1]) for e in ev) / steps
    ms_step = max_over_ranks(total_ms / steps, dev)
    gemm_ms_max = max_over_ranks(gemm_ms, dev)
    value = useful_ops(c) / (ms_step * 1e-3) / 1e12      # the global problem / slowest rank

    peaks = load_peaks()
    # roofline of the dominant kernel on the slowest rank's share (each rank runs the same kernel)
    kern = plan.kernel("f16i" if f16i else ("raw" if fused else "beamform"))
    roof = roofline_for(lc, gemm_ms_max, peaks, long_step=(steps * ms_step > 1000.0), variant=kern, fused=fused)
    roof["kernel"] = kern
    roof["traffic"] = traffic_for(name, kern) if world == 1 else None
    roof["kernel_ms"] = round(gemm_ms_max, 4)
    roof["algorithmic_bytes_per_launch"] = gemm_bytes(lc, False)
    roof["useful_ops_per_launch"] = useful_ops(lc)
    pack_ms_max = max_over_ranks(pack_ms, dev) if not (fused or f16i) else 0.0
    if pack_ms_max > gemm_ms_max:
        # the data pack dominates the step (few beams: M=32 sweeps): report ITS roofline as the
        # dominant kernel, the GEMM's beside it
        pk = pack_roofline(lc, pack_ms_max, plan.x_bytes, peaks)
        pk["gemm"] = roof
        pk["traffic"] = traffic_for(name, pk["kernel"]) if world == 1 else None
        roof = pk

    rec = {
        "workload": name, "desc": c["desc"], "precision": c["prec"],
        "value": round(value, 2), "unit": "TeraOps/s", "ms_per_step": round(ms_step, 4), "steps": steps,
        "M": c["M"], "N": c["N"], "K": c["K"], "global_batch": c["B"],
        "shard": {"mode": sh.mode, "batch_per_rank": plan.batch, "samples_per_rank": plan.N},
        "step": ("tcbf_beamform_f16i (fp16 interleaved data, no pack)" if f16i else
                 "tcbf_beamform_raw (data pack fused into the GEMM)" if fused else
                 "tcbf_pack(data) + tcbf_beamform") + "; weights packed once",
        "l2": ("flushed between steps (256 MiB write)" if flush else
               f"working set {working / 2 ** 30:.2f} GiB > L2 (126 MiB), no flush"),
        "pack_ms": round(pack_ms, 4), "gemm_ms": round(gemm_ms, 4),
        "samples_per_s": round(c["N"] * c["B"] / (ms_step * 1e-3), 1),
        "roofline": roof,
        "gpu_launches": launches_per_step * steps,
    }
    if sampler:
        rec["clocks"] = sampler.summary()

    if energy:
        rec["energy"] = energy_loop(step, stream, c, dev, world,
                                    shared_device=(world > 1 and args.dist_backend == "gloo"))

    if e2e:
        # through the public API with HOST buffers (pinned), copies inside the timed region
        x_host = xsrc.cpu().pin_memory()
        out_host = torch.empty(tuple(out.shape), dtype=out.dtype).pin_memory()
        e2e_steps = max(1, min(steps, 5))

        def e2e_call():
            if f16i:   # H2D of the fp16 data, beamform_f16i, D2H of the output (binding-level API)
                xsrc.copy_(x_host, non_blocking=True)
                plan.beamform_f16i(wp, xsrc, out=out, stream=stream)
                out_host.copy_(out, non_blocking=True)
                torch.cuda.synchronize()
            else:
                plan.beamform_host(wp, x_host, out_host)

        e2e_call()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_call()
        e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_steps, dev)
        rec["e2e"] = {"value": round(useful_ops(c) / e2e_s / 1e12, 3), "unit": "TeraOps/s",
                      "h2d_bytes_per_step": int(x_host.numel() * x_host.element_size()) * world,
                      "d2h_bytes_per_step": int(plan.out_bytes) * world,
                      "api": ("Plan.beamform_f16i with pinned-host copies in and out" if f16i else
                              "tcbf_beamform_host (pinned host buffers)"),
                      "steps": e2e_steps}

    if args.gather and world > 1 and sh.mode == "batch" and c["B"] % world == 0:
        # the optional output gather: timed separately, never part of `value`
        from paper_2505_03269_b200.shard import gather_outputs
        gather_outputs(out)
        torch.cuda.synchronize()
        dist.barrier()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        full = gather_outputs(out)
        g1.record(stream)
        torch.cuda.synchronize()
        rec["gather"] = {"ms": round(max_over_ranks(g0.elapsed_time(g1), dev), 3),
                         "bytes_per_rank_received": int(full.numel() * full.element_size() - plan.out_bytes),
                         "collective": f"all_gather_into_tensor ({args.dist_backend})"}
        del full
    del wp, xsrc, xp, out, flush_buf
    torch.cuda.empty_cache()
    return rec


def energy_loop(step, stream, c, dev, world, min_s=1.0, shared_device=False):
    """NVML energy over a separate loop of >= `min_s` seconds of back-to-back steps (the counter's
    granularity makes short timed regions meaningless).  Board energy of this GPU; TeraOps/J of the
    whole job = global ops / (joules summed over ranks).  shared_device (the gloo test mode, every
    rank on cuda:0): all ranks read the same board over the same loop, so the max is taken."""
    import torch
    from paper_2505_03269_b200.shard import sum_over_ranks
    s = ClockSampler(dev, sample=False)
    if not s.ok:
        return {"unavailable": "NVML not available"}
    # calibrate the step count for ~min_s
    t0 = time.perf_counter()
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    per = max(1e-5, (time.perf_counter() - t0) / 3)
    n = max(10, int(min_s / per) + 1)
    s.start()
    t0 = time.perf_counter()
    for _ in range(n):
        step()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    s.stop()
    j = s.joules()
    if j is None or j <= 0:
        return {"unavailable": "NVML energy counter returned no delta"}
    if shared_device:
        from paper_2505_03269_b200.shard import max_over_ranks
        j_all = max_over_ranks(j, dev)
    else:
        j_all = sum_over_ranks(j, dev)
    watts = j / wall
    rec = {"joules_per_step": round(j_all / n, 6), "teraops_per_joule": round(useful_ops(c) * n / j_all / 1e12, 3),
           "loop_s": round(wall, 3), "steps": n, "avg_board_w": round(watts, 1),
           "source": "NVML total energy counter over a separate >= 1 s loop of back-to-back steps"}
    if watts > 1200.0:   # a B200 board cannot sustain this: counter artefact, do not report
        return {"unavailable": f"implausible average power {watts:.0f} W over {wall:.2f} s"}
    return rec


def run_tcbf(args, c):
    import torch.distributed as dist
    world, rank, local, dev = setup_dist(args)
    main = measure(args, args.config, c, world, rank, local, dev, args.steps, args.warmup, e2e=True,
                   energy=not args.no_energy)
    records = {}
    extra = [r for r in (args.records.split(",") if args.records else []) if r and r != args.config]
    for r in extra:
        records[r] = measure(args, r, CONFIGS[r], world, rank, local, dev, args.steps, args.warmup)
    line = {
        "metric": "beamforming TeraOps/s (fp16 and 1-bit) at 1/2/4/8 B200 vs roofline",
        "value": main["value"], "unit": "TeraOps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": main["ms_per_step"], "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": c["prec"],
        "data": "synthetic (seeded counter-based generator, synth/)",
        "config": {"workload": args.config, "desc": c["desc"], "M": c["M"], "N": c["N"], "K": c["K"],
                   "global_batch": c["B"], "batch_per_gpu": main["shard"]["batch_per_rank"],
                   "samples_per_gpu": main["shard"]["samples_per_rank"], "precision": c["prec"],
                   "step": main["step"], "l2": main["l2"],
                   "parallelism": (f"{main['shard']['mode']}-sharded x{world} (SURVEY.md §8e strong scaling of "
                                   f"the fixed config), no data-path collective"),
                   "pack_ms": main["pack_ms"], "gemm_ms": main["gemm_ms"], "samples_per_s": main["samples_per_s"]},
        "roofline": main["roofline"],
        "e2e": main["e2e"],
        "gpu_launches": main["gpu_launches"],
        "clocks": main["clocks"],
    }
    if "energy" in main:
        line["energy"] = main["energy"]
    if "gather" in main:
        line["gather"] = main["gather"]
    if records:
        line["records"] = records
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(c)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="radio_f16", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="tcbf", choices=["tcbf", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo = test mode, all ranks share cuda:0 (production runs use nccl)")
    ap.add_argument("--records", default=None,
                    help="comma-separated extra workloads timed in the same run and reported under 'records' "
                         "(default for radio_f16: radio_b1,ultrasound_f16,radio_f16i -- both precisions of the "
                         "metric and the NEXT-1 interleaved-fp16 path)")
    ap.add_argument("--no-energy", action="store_true", help="skip the >= 1 s NVML energy loop")
    ap.add_argument("--gather", action="store_true", help="also time the optional NCCL output gather (N > 1)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    c = CONFIGS[args.config]
    if args.records is None:
        args.records = "radio_b1,ultrasound_f16,radio_f16i" if args.config == "radio_f16" else ""
    if args.impl == "reference":
        return run_reference(args, c)
    return run_tcbf(args, c)


if __name__ == "__main__":
    sys.exit(main())
