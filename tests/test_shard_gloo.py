"""Frame-range sharding with a one-frame halo and the record all-gather
(SURVEY section 8(e)), exercised on CPU with torch.distributed/gloo at
world_size 2.  The per-rank analyser here is the CPU oracle, so this pins the
host logic (plan, halo, POCs, padding, gather order): sharded + gathered
records must equal the unsharded run bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2304_12384_b200 import shard

W, H = 96, 64


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _frames(first, n):
    from paper_2304_12384_b200 import synth

    return synth.as_numpy_planes(*synth.g_frames(12, W, H, n, 8, first_t=first))


def _records_tensor(rec):
    return torch.from_numpy(np.ascontiguousarray(rec).view(np.float64).reshape(-1, 8).copy())


def _worker(rank, world, port, n_total, lowpass, q):
    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = shard.plan(n_total, world, rank)
        Y, U, V = _frames(sh.first_frame, sh.n_frames)
        rec = oracle.analyze(Y, U, V, 8, 32, lowpass, n_halo=sh.n_halo, first_poc=sh.first_poc)
        assert len(rec) == sh.count
        allrec = shard.gather_records(_records_tensor(rec), world)
        if rank == 0:
            q.put(allrec.numpy().copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_total,lowpass", [(6, True), (7, False)])
def test_sharded_equals_unsharded_gloo(oracle_mod, n_total, lowpass):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_total, lowpass, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    Y, U, V = _frames(0, n_total)
    ref = oracle_mod.analyze(Y, U, V, 8, 32, lowpass)
    want = np.ascontiguousarray(ref).view(np.float64).reshape(-1, 8)
    assert np.array_equal(got.view(np.int64)[:, 0], np.arange(n_total))
    assert np.array_equal(got, want)


def test_plan():
    assert shard.plan(4800, 8, 0) == shard.Shard(0, 8, 0, 600, 0, 600, 0)
    s3 = shard.plan(4800, 8, 3)
    assert (s3.first_poc, s3.count, s3.first_frame, s3.n_frames, s3.n_halo) == (1800, 600, 1799, 601, 1)
    # uneven split covers every POC exactly once
    cov = []
    for r in range(3):
        s = shard.plan(10, 3, r)
        cov += list(range(s.first_poc, s.first_poc + s.count))
        assert s.n_frames == s.count + s.n_halo
    assert cov == list(range(10))
    with pytest.raises(ValueError):
        shard.plan(2, 3, 0)


def test_config5_strong_scaling_plan():
    """bench.py at N > 1 (config 5, strong scaling): 4800 frames in contiguous ranges of 4800 / N,
    every rank after the first behind a one-frame halo, every rank start on a 600-frame segment
    boundary for N = 2, 4, 8 (so each rank's halo is the previous segment's last frame)."""
    for world in (1, 2, 4, 8):
        plans = [shard.plan(4800, world, r) for r in range(world)]
        assert sum(p.count for p in plans) == 4800
        assert [p.first_poc for p in plans] == [r * 4800 // world for r in range(world)]
        for r, p in enumerate(plans):
            assert p.count == 4800 // world and p.n_halo == (1 if r else 0)
            assert p.first_frame == p.first_poc - p.n_halo and p.n_frames == p.count + p.n_halo
            assert p.first_poc % 600 == 0
