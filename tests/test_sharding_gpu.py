"""The real multi-rank shard path on one GPU: two processes, each running the
library's own shard cut (fic_params_t.shard_index/count) and the packed
all-gather of its own ranges (gloo carries the exchange: the two ranks'
kernels never wait on each other, so one GPU is enough), must give bytes
identical to a one-process encode (SURVEY.md §8e correctness gate)."""

import hashlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _digest(*ts):
    h = hashlib.sha256()
    for t in ts:
        h.update(t.cpu().contiguous().numpy().tobytes())
    return h.hexdigest()


def _worker(rank, world, port, cname, strategy, q):
    import torch.distributed as dist

    from paper_1206_4880_b200 import codec, synth
    from paper_1206_4880_b200.sharding import encode_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c = synth.CONFIGS[cname]
    img = torch.from_numpy(c.make()).cuda()
    kw = dict(range_size=c.range_size, domain_size=c.domain_size, stride=c.stride,
              isometries=True, delta=c.delta if strategy == "dynamic_fd" else None)
    recs, pre, post, pools, st = encode_sharded(img, strategy, **kw)
    full = codec.encode_device(img, strategy, **kw)
    q.put((rank, _digest(recs, pre, post), _digest(full.records, full.pre_rms, full.post_rms),
           bool(torch.equal(pools, full.pool_sizes))))
    dist.destroy_process_group()


@pytest.mark.parametrize("cname,strategy,world", [("cfg2", "dynamic_fd", 2),
                                                  ("cfg2", "exhaustive", 2),
                                                  ("cfg1", "dynamic_fd", 3)])
def test_two_process_shards_equal_one_process(cname, strategy, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cname, strategy, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for _, sharded, single, pools_ok in got:
        assert sharded == single
        assert pools_ok
