"""World-size-2 gloo test of the multi-GPU exchange step (CPU only).

The per-rank match is stood in for by the oracle on that rank's ranges (the
GPU shard partition itself is covered by the gpu tests, including
tests/test_sharding_gpu.py, which runs the real library shard path in two
processes); what is tested here is the host-side exchange: each rank contributes only
the ranges it owns (zeros elsewhere) to two all-reduces -- which must
reproduce the 1-process result byte for byte, for even and uneven shards,
and reject a partition with a hole or an overlap.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fic_oracle as orc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _owner(n_r, world, mode):
    r = np.arange(n_r)
    if mode == "even":
        return r % world
    if mode == "uneven":       # rank 0 owns the first 5 ranges only
        return np.where(r < 5, 0, 1 + r % (world - 1))
    if mode == "hole":         # range 7 owned by nobody
        return np.where(r == 7, -1, r % world)
    return r % world           # "overlap": range 3 owned by every rank (below)


def _worker(rank, world, port, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1206_4880_b200.sharding import gather_shards

    img = np.random.default_rng(5).integers(0, 256, (64, 64), dtype=np.uint8)
    n_r = 64
    own = _owner(n_r, world, mode)
    mine = np.flatnonzero((own == rank) | ((mode == "overlap") & (np.arange(n_r) == 3)))
    res = orc.encode(img, "dynamic_fd", stride=4, isometries=True, range_ids=mine)
    rec = torch.from_numpy(res.records.view(np.uint8).reshape(-1, 7).copy())
    rec[np.setdiff1d(np.arange(n_r), mine)] = 0
    pre = torch.full((n_r,), -1.0, dtype=torch.float64)
    post = torch.full((n_r,), -1.0, dtype=torch.float64)
    pre[mine] = torch.from_numpy(res.pre_rms[mine])
    post[mine] = torch.from_numpy(res.post_rms[mine])
    try:
        r2, p2, q2 = gather_shards(rec, pre, post)
        q.put((rank, r2.numpy().tobytes(), p2.numpy().tobytes(), q2.numpy().tobytes()))
    except RuntimeError as e:
        q.put((rank, "error", str(e), None))
    dist.destroy_process_group()


def _run(world, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return got


@pytest.mark.parametrize("world,mode", [(2, "even"), (3, "uneven")])
def test_gather_shards_matches_single_process(world, mode):
    got = _run(world, mode)
    img = np.random.default_rng(5).integers(0, 256, (64, 64), dtype=np.uint8)
    full = orc.encode(img, "dynamic_fd", stride=4, isometries=True)
    for _, rec, pre, post in got:
        assert rec == full.records.tobytes()
        assert pre == full.pre_rms.tobytes()
        assert post == full.post_rms.tobytes()


@pytest.mark.parametrize("mode", ["hole", "overlap"])
def test_gather_shards_rejects_bad_partitions(mode):
    got = _run(2, mode)
    for _, tag, msg, _ in got:
        assert tag == "error"
        assert "no rank or by several" in msg or "range entries for" in msg
