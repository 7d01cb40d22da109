"""Where the sharded path's extra time goes (one-rank NCCL group, cfg3):
device time (CUDA events) and host wall time of encode_device with and
without shard=(0, 1), and of gather_shards alone.
    python -m torch.distributed.run --nproc-per-node 1 --master-addr 127.0.0.1 tools/dist_overhead.py"""
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth  # noqa: E402
from paper_1206_4880_b200.sharding import encode_sharded, gather_shards  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
img = torch.from_numpy(synth.cfg3_image()).cuda()
kw = dict(range_size=8, domain_size=16, stride=1, isometries=True, delta=0.05)


def timed(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    dev, wall = [], []
    for _ in range(n):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        wall.append((time.perf_counter() - t0) * 1e3)
        dev.append(e0.elapsed_time(e1))
    return sum(dev) / n, sum(wall) / n


print("encode_device        dev %.3f wall %.3f ms" % timed(lambda: codec.encode_device(img, "dynamic_fd", **kw)))
print("encode_device shard  dev %.3f wall %.3f ms" % timed(lambda: codec.encode_device(img, "dynamic_fd", shard=(0, 1), **kw)))
print("encode_sharded       dev %.3f wall %.3f ms" % timed(lambda: encode_sharded(img, "dynamic_fd", **kw)))
r = codec.encode_device(img, "dynamic_fd", **kw)
print("gather_shards        dev %.3f wall %.3f ms" % timed(lambda: gather_shards(r.records, r.pre_rms, r.post_rms)))
buf = torch.zeros((16384, 3), dtype=torch.int64, device="cuda")
print("all_reduce alone     dev %.3f wall %.3f ms" % timed(lambda: dist.all_reduce(buf)))
print("check (.all() sync)  dev %.3f wall %.3f ms" % timed(lambda: bool((buf[:, 0] == 1).all())))
pre, post, rec = r.pre_rms, r.post_rms, r.records


def pack():
    owned = post >= 0
    b = torch.zeros((16384, 3), dtype=torch.int64, device="cuda")
    b8 = b.view(torch.uint8).view(16384, 24)
    b8[:, :7] = rec
    b8[:, 7] = 1
    b[:, 1] = pre.view(torch.int64)
    b[:, 2] = post.view(torch.int64)
    b.mul_(owned.to(torch.int64)[:, None])


print("pack ops             dev %.3f wall %.3f ms" % timed(pack))
dist.destroy_process_group()
