"""Multi-process sharded beamform on the CUDA path (PAPER.md:101 batch option,
PAPER.md:393 batch = polarizations x channels): world size 2 over gloo with both ranks on cuda:0
(the one-GPU stand-in for one process per GPU).  Each rank builds its shard exactly as bench.py
does (batch slices from global indices, or sample columns when the batch is smaller than the
world; K never split) and runs it through libtcbf.so; the reassembled result must equal the
unsharded run bit for bit, and sampled rows must match the oracle."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CASES = [
    # name, prec, M, N, K, B  (B >= world -> batch slices; B < world -> sample columns)
    ("batch_f16_fused", "f16", 256, 512, 256, 5),
    ("batch_b1", "b1", 200, 300, 700, 3),
    ("samples_f16", "f16", 300, 1000, 300, 1),
    ("samples_b1", "b1", 100, 260, 1000, 1),
]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cfg(prec, M, N, K, B):
    return dict(prec=prec, M=M, N=N, K=K, B=B, wd="phase", xd="adc", idx=1, desc="shard test")


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        import synth
        from paper_2505_03269_b200.shard import max_over_ranks, plan_shard
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        res = {}
        for name, prec, M, N, K, B in CASES:
            c = _cfg(prec, M, N, K, B)
            sh = plan_shard(B, N, rank, world)
            plan, wp, xsrc = bench.shard_inputs(c, sh, synth.SEED_BASE + c["idx"], dev)
            y = plan.beamform_raw(wp, xsrc)   # the call bench.py times
            torch.cuda.synchronize()
            res[name] = (sh, y.cpu().numpy())
        t = max_over_ranks(float(rank), dev)
        q.put((rank, res, t))
    finally:
        dist.destroy_process_group()


def test_sharded_equals_unsharded_on_cuda():
    import oracle
    import paper_2505_03269_b200 as tcbf
    import synth
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((r, (res, t)) for r, res, t in (q.get(timeout=600) for _ in procs))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got[0][1] == 1.0 and got[1][1] == 1.0   # max over ranks through the process group
    for name, prec, M, N, K, B in CASES:
        (sh0, y0), (sh1, y1) = got[0][0][name], got[1][0][name]
        if sh0.mode == "batch":
            assert (sh0.b0, sh0.b0 + sh0.nb) == (0, sh1.b0) and sh1.b0 + sh1.nb == B
            full = np.concatenate([y0, y1], axis=0)
        else:
            assert sh0.mode == "samples" and sh0.n0 == 0 and sh1.n0 == sh0.nn and sh0.nn % 4 == 0
            full = np.concatenate([y0, y1], axis=3)
        seed = synth.SEED_BASE + 1
        plan = tcbf.Plan(M, N, K, B, prec)
        wp = plan.pack(tcbf.WEIGHTS, synth.generate_device("phase", seed, 0, B, M, K))
        ref = plan.beamform_raw(wp, synth.generate_device("adc", seed, 1, B, K, N)).cpu().numpy()
        assert np.array_equal(full, ref), name                     # sharded == unsharded, bitwise
        rows = [0, M // 2, M - 1]
        for b in sorted({0, B - 1}):
            w = synth.to_interleaved(synth.generate("phase", seed, 0, B, M, K, b_sel=[b], r_sel=rows))
            x = synth.to_interleaved(synth.generate("adc", seed, 1, B, K, N, b_sel=[b]))
            got_rows = full[b][:, rows][None]
            if prec == "b1":
                assert np.array_equal(got_rows, oracle.cgemm_b1(w, x, 0, len(rows), N, K, 1)), name
            else:
                ref_rows = oracle.cgemm_f16(w, x, 0, len(rows), N, K, 1)
                err = np.linalg.norm(got_rows.astype(np.float64) - ref_rows)
                assert err <= 2e-3 * np.linalg.norm(ref_rows), name


def test_bench_two_ranks_strong_scaling_line():
    """bench.py's N > 1 path end to end (the driver's torchrun launch, gloo, both ranks on cuda:0):
    one JSON line from rank 0, the FIXED global radio batch split into two 128-channel slices
    (strong scaling), timing reduced over ranks."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--dist-backend", "gloo", "--config", "radio_f16", "--steps", "3", "--warmup", "3",
           "--no-cpu-baseline", "--no-energy", "--records", ""]
    r = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["global_batch"] == 256 and d["config"]["batch_per_gpu"] == 128
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] >= 3
