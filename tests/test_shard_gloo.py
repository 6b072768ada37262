"""Multi-process host logic of the batch sharder on CPU (gloo, world_size 2): the batch
slices cover the problem exactly once, and the sharded beamform (oracle per shard, gathered
with the sharder's collective) equals the unsharded one bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_03269_b200.shard import (contiguous_slice, gather_outputs, max_over_ranks, plan_shard,
                                         sum_over_ranks)


def test_contiguous_slices_cover_once():
    for total in (1, 7, 256, 1000):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                s, n = contiguous_slice(total, r, world)
                seen += list(range(s, s + n))
            assert seen == list(range(total))


def test_plan_shard_modes():
    assert plan_shard(256, 1024, 3, 8) == plan_shard(256, 1024, 3, 8)
    s = plan_shard(256, 1024, 3, 8)
    assert (s.mode, s.b0, s.nb, s.nn) == ("batch", 96, 32, 1024)
    cols = []
    for r in range(8):                      # B=1 < world: split samples, multiples of 4
        s = plan_shard(1, 16384, r, 8)
        assert s.mode == "samples" and s.n0 % 4 == 0
        cols += list(range(s.n0, s.n0 + s.nn))
    assert cols == list(range(16384))
    s = plan_shard(8, 256, 5, 8)            # ultrasound 8 frames on 8 GPUs: one each
    assert (s.mode, s.b0, s.nb) == ("batch", 5, 1)
    s = plan_shard(8, 256, 2, 3)            # unequal slices: 3, 3, 2
    assert (s.b0, s.nb) == (6, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        B, M, N, K = 6, 9, 12, 40
        sh = plan_shard(B, N, rank, world)
        w = synth.to_interleaved(synth.generate("adc", 77, 0, B, M, K, b_sel=slice(sh.b0, sh.b0 + sh.nb)))
        x = synth.to_interleaved(synth.generate("adc", 77, 1, B, K, N, b_sel=slice(sh.b0, sh.b0 + sh.nb)))
        local = torch.from_numpy(oracle.cgemm_b1(w, x, 0, M, N, K, sh.nb))
        full = gather_outputs(local)
        t = max_over_ranks(float(rank + 1))
        tot = sum_over_ranks(float(rank + 1))
        if rank == 0:
            q.put((full.numpy(), t, tot))
    finally:
        dist.destroy_process_group()


def test_sharded_equals_unsharded_gloo():
    import oracle
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, tmax, tsum = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    B, M, N, K = 6, 9, 12, 40
    w = synth.to_interleaved(synth.generate("adc", 77, 0, B, M, K))
    x = synth.to_interleaved(synth.generate("adc", 77, 1, B, K, N))
    assert np.array_equal(full, oracle.cgemm_b1(w, x, 0, M, N, K, B))
    assert tmax == 2.0 and tsum == 3.0
