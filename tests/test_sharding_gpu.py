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


def _worker(rank, world, port, cname, strategy, q, backend="gloo"):
    import torch.distributed as dist

    from paper_1206_4880_b200 import codec, synth
    from paper_1206_4880_b200.sharding import encode_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=torch.device("cuda", 0))
    else:
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


@pytest.mark.parametrize("cname", ["cfg2", "cfg3"])
def test_nccl_exchange_one_rank_equals_one_process(cname):
    """The NCCL branch of the exchange (all_gather of the counts,
    all_gather_into_tensor of the packed entries on the device, as bench.py
    --gpus N runs it) over a one-rank group -- the only NCCL group one GPU
    allows -- returns the one-process encode byte for byte."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(0, 1, _free_port(), cname, "dynamic_fd", q, "nccl"))
    p.start()
    _, sharded, single, pools_ok = q.get(timeout=600)
    p.join(timeout=120)
    assert p.exitcode == 0
    assert sharded == single and pools_ok


def test_shard_pack_unpack_kernels_round_trip_and_flag_holes():
    """fic_shard_pack_v1 / fic_shard_unpack_v1 on one rank (no reduction):
    owned ranges come back byte for byte, a range nobody owns is counted."""
    import ctypes

    from paper_1206_4880_b200 import _lib

    lib = _lib.load()
    n = 1000
    g = torch.Generator().manual_seed(5)
    rec = torch.randint(0, 256, (n, 7), dtype=torch.uint8, generator=g).cuda()
    pre = torch.rand(n, dtype=torch.float64, generator=g).cuda() * 40
    post = pre + 1.0
    post[17] = -1.0                     # not matched by this rank: a hole
    buf = torch.empty((n, 3), dtype=torch.int64, device="cuda")
    out_rec = torch.empty_like(rec)
    out_pre = torch.empty_like(pre)
    out_post = torch.empty_like(post)
    bad = torch.empty(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    vp = ctypes.c_void_p
    _lib.check(lib.fic_shard_pack_v1(vp(rec.data_ptr()), vp(pre.data_ptr()), vp(post.data_ptr()), n,
                                     vp(buf.data_ptr()), vp(s)))
    _lib.check(lib.fic_shard_unpack_v1(vp(buf.data_ptr()), n, vp(out_rec.data_ptr()),
                                       vp(out_pre.data_ptr()), vp(out_post.data_ptr()),
                                       vp(bad.data_ptr()), vp(s)))
    keep = torch.arange(n, device="cuda") != 17
    assert int(bad.item()) == 1
    assert torch.equal(out_rec[keep], rec[keep])
    assert torch.equal(out_pre[keep], pre[keep]) and torch.equal(out_post[keep], post[keep])
    assert int(out_rec[17].sum()) == 0 and float(out_post[17]) == 0.0
