"""Multi-process (gloo, world size 2) coverage of the sharded-evaluation host logic."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2102_08518_b200.dist import gather_results, max_over_ranks, replicate_arrays, shard_range  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(100 + rank)          # ranks start with different data
        arrays = [rng.random((5, 6, 7)).astype(np.float32) for _ in range(2)]
        rep = replicate_arrays(arrays)
        t = max_over_ranks(1.5 + rank)
        n_total = 11
        lo, hi = shard_range(n_total, rank, world)
        local = torch.arange(lo, hi, dtype=torch.float32) * 2
        full = gather_results(local, n_total)
        q.put((rank, [r.numpy() for r in rep], t, full.numpy()))
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions():
    for n in (0, 1, 7, 1 << 20):
        for w in (1, 2, 3, 8):
            got = [shard_range(n, r, w) for r in range(w)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            assert max(h - l for l, h in got) - min(h - l for l, h in got) <= 1


def test_gloo_world2_replicate_reduce_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    res.sort(key=lambda r: r[0])
    rng = np.random.default_rng(100)
    want = [rng.random((5, 6, 7)).astype(np.float32) for _ in range(2)]
    for rank, rep, t, full in res:
        for a, b in zip(rep, want):
            assert np.array_equal(a, b)          # every rank holds rank 0's volume
        assert t == 2.5                          # max over ranks
        assert np.array_equal(full, np.arange(11, dtype=np.float32) * 2)
