"""World-size-2 gloo test of the multi-GPU exchange step (CPU only).

The per-rank match is stood in for by the oracle on that rank's ranges (the
GPU shard partition itself is covered by the gpu tests); what is tested here
is the host-side exchange: all-gather of per-rank record shards and owner
selection, which must reproduce the 1-process result byte for byte.
"""

import os
import socket

import numpy as np
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


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1206_4880_b200.sharding import gather_shards

    img = np.random.default_rng(5).integers(0, 256, (64, 64), dtype=np.uint8)
    n_r = 64
    mine = np.arange(n_r)[np.arange(n_r) % world == rank]
    res = orc.encode(img, "dynamic_fd", stride=4, isometries=True, range_ids=mine)
    rec = torch.from_numpy(res.records.view(np.uint8).reshape(-1, 7).copy())
    pre = torch.full((n_r,), -1.0, dtype=torch.float64)
    post = torch.full((n_r,), -1.0, dtype=torch.float64)
    pre[mine] = torch.from_numpy(res.pre_rms[mine])
    post[mine] = torch.from_numpy(res.post_rms[mine])
    r2, p2, q2 = gather_shards(rec, pre, post)
    q.put((rank, r2.numpy().tobytes(), p2.numpy().tobytes(), q2.numpy().tobytes()))
    dist.destroy_process_group()


def test_gather_shards_world2_matches_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    img = np.random.default_rng(5).integers(0, 256, (64, 64), dtype=np.uint8)
    full = orc.encode(img, "dynamic_fd", stride=4, isometries=True)
    for _, rec, pre, post in got:
        assert rec == full.records.tobytes()
        assert pre == full.pre_rms.tobytes()
        assert post == full.post_rms.tobytes()
