"""CPU checks of bench.py's contract: the reference arm (the oracle, this tier's reference) prints
one well-formed JSON line, alone and under torchrun (rank 0 only), and the roofline / work-count
helpers follow SURVEY.md §8(d) (8·M·N·K useful ops, algorithmic bytes, binding roof)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _run(cmd, env=None):
    e = dict(os.environ, **(env or {}))
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300, env=e)
    assert r.returncode == 0, r.stderr[-2000:]
    return [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]


def test_reference_arm_json_line():
    lines = _run([sys.executable, "bench.py", "--impl", "reference", "--config", "tiny", "--steps", "2",
                  "--warmup", "1"])
    assert len(lines) == 1
    d = lines[0]
    assert KEYS <= set(d) and d["impl"] == "reference"
    assert d["metric"] == json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
    assert d["value"] > 0 and d["unit"] == "TeraOps/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["config"]["workload"] == "tiny" and d["steps"] == 2 and d["warmup"] == 3  # W >= 3 enforced


def test_reference_arm_under_torchrun_rank0_only():
    lines = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                  "--master-addr", "127.0.0.1", "--master-port", "29561", "bench.py", "--impl", "reference",
                  "--gpus", "2", "--config", "tiny", "--steps", "2", "--warmup", "1"])
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"


def test_useful_ops_and_bytes():
    c = bench.CONFIGS["radio_f16"]
    assert bench.useful_ops(c) == 8 * 1024 * 1024 * 256 * 256
    B, M, N, K = 256, 1024, 1024, 256
    assert bench.gemm_bytes(c) == B * (4 * M * K + 4 * K * N + 8 * M * N)
    assert bench.gemm_bytes(c, fused=True) == B * (4 * M * K + 8 * K * N + 8 * M * N)
    c1 = bench.CONFIGS["radio_b1"]
    B, M, N, K = 256, 1024, 4096, 512
    assert bench.gemm_bytes(c1) == B * ((M * K + K * N) / 4 + 8 * M * N)


@pytest.mark.parametrize("name", sorted(bench.CONFIGS))
def test_configs_well_formed(name):
    c = bench.CONFIGS[name]
    assert c["prec"] in ("f16", "b1") and min(c["M"], c["N"], c["K"], c["B"]) >= 1
    assert c["wd"] in ("uniform", "adc", "phase", "phase_amp", "adc_scaled")


def test_roofline_binding_roof_and_kind():
    peaks = dict(hbm=6000.0, bf16=1600.0, bf16_sus=1300.0, src="test")
    radio = bench.CONFIGS["radio_f16"]
    t_hbm_ms = bench.gemm_bytes(radio) / 6000e9 * 1e3
    r = bench.roofline_for(radio, 2 * t_hbm_ms, peaks, long_step=False, variant="f16_x")
    assert r["bound"] == "hbm" and abs(r["frac"] - 0.5) < 1e-3 and r["peak"] == 6000.0
    sq = bench.CONFIGS["square_f16_8192"]
    t_tc_ms = bench.useful_ops(sq) / 1600e12 * 1e3
    r = bench.roofline_for(sq, t_tc_ms / 0.8, peaks, long_step=False, variant="f16_x")
    assert r["bound"] == "tensor" and abs(r["frac"] - 0.8) < 1e-3
    r = bench.roofline_for(sq, t_tc_ms / 0.8, peaks, long_step=True, variant="f16_x")
    assert abs(r["peak"] - 1300.0) < 1e-6   # sustained peak for long timed regions
    sqb = bench.CONFIGS["square_b1_8192"]
    r4 = bench.roofline_for(sqb, 1.0, peaks, long_step=False, variant="b1_tcgen05_mxf4pm1_128x128_tma")
    r8 = bench.roofline_for(sqb, 1.0, peaks, long_step=False, variant="b1_tcgen05_i8_128x128_tma")
    assert r4["peak"] == 4 * 1600.0 and r8["peak"] == 2 * 1600.0
    rp = bench.roofline_for(sqb, 1.0, peaks, long_step=False, variant="b1_popc_xor_64x64")
    assert rp["bound"] == "alu"
    rm = bench.roofline_for(sqb, 1.0, peaks, long_step=False, variant="b1_mma_sync_and_128x64")
    assert rm["bound"] == "b1_mma_sync" and rm["peak"] > 100.0   # measured peaks.cu value


def test_peaks_record_committed():
    """profiles/r01/peaks.json (peaks.cu on the B200) holds every kind tools/peaks.py measures."""
    import json
    with open(os.path.join(ROOT, "profiles", "r01", "peaks.json")) as f:
        d = json.load(f)["peaks"]
    for k in ("b1_mma_sync_and_popc", "b1_mma_sync_xor_popc", "cuda_core_xor_popc", "tcgen05_f16", "tcgen05_i8",
              "tcgen05_mxf4"):
        assert d[k]["tera_ops_per_s"] > 0


def test_pack_roofline_when_pack_dominates():
    """M=32 1-bit: the fp32 data pack is the step's dominant kernel; its roofline counts the fp32
    read plus the packed write."""
    c = bench.CONFIGS["m32_b1_16384"]
    peaks = dict(hbm=6000.0, bf16=1600.0, bf16_sus=1300.0, src="test")
    packed = 2 * c["N"] * (c["K"] // 32) * 4
    byts = c["K"] * c["N"] * 8 + packed
    r = bench.pack_roofline(c, byts / 6000e9 * 1e3 / 0.5, packed, peaks)
    assert r["bound"] == "hbm" and abs(r["frac"] - 0.5) < 1e-3 and r["kernel"] == "pack_b1_transpose"
