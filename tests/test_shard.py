"""Multi-rank host logic of the batch-sharded path, world_size 2 over gloo on
the CPU: slice table, weight replication, max-over-ranks timing, and that the
ranks' slices reassemble the single-rank result (the per-slice conv here is
the oracle -- the checker stands in for the GPU kernel, which needs a B200)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2006_02230_b200.shard import (gather_images, max_over_ranks, replicate_, shard_images,
                                         shard_table)


def test_shard_table_covers_batch():
    for n in (0, 1, 5, 256, 257):
        for world in (1, 2, 3, 8):
            t = shard_table(n, world)
            assert sum(c for _, c in t) == n
            pos = 0
            for s, c in t:
                assert s == pos and c >= 0
                pos += c
            assert max(c for _, c in t) - min(c for _, c in t) <= 1
    assert shard_images(256, 8, 3) == (96, 32)
    with pytest.raises(ValueError):
        shard_images(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_global, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import conv2d_np
        rng = np.random.default_rng(0)
        x = rng.uniform(-1, 1, size=(n_global, 1, 6, 6, 16)).astype(np.float32)
        w = torch.from_numpy(rng.uniform(-1, 1, size=(2, 1, 3, 3, 16, 16)).astype(np.float32))
        if rank != 0:
            w.zero_()           # must come from rank 0
        replicate_([w])
        s, c = shard_images(n_global, world, rank)
        y = conv2d_np(x[s:s + c], w.numpy(), stride=1, pad=1) if c else \
            np.zeros((0, 2, 6, 6, 16))
        full = gather_images(torch.from_numpy(np.ascontiguousarray(y)), n_global)
        t = max_over_ranks(1.5 + rank)
        if rank == 0:
            ref = conv2d_np(x, w.numpy(), stride=1, pad=1)
            q.put((float(np.abs(full.numpy() - ref).max()), t, float(w.abs().sum())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_global", [4, 3, 1])
def test_two_rank_gloo_roundtrip(n_global):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_global, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    err, t, wsum = q.get(timeout=5)
    assert err == 0.0 and t == 2.5 and wsum > 0
