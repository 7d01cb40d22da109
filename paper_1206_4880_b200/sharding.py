"""Range sharding across GPUs: one process per GPU, one all-gather of records.

Every rank holds the whole image (<= 64 MB) and recomputes FD, the FD index
and the pool (sub-millisecond), so every rank derives the same FD-sorted,
cost-balanced partition of ranges without communication (the
library sorts the ranges deterministically when sharded, fic_api.cu
k_range_scatter_stable).  Each rank matches only its shard
(``fic_params_t.shard_index/count``) and writes only its ranges' outputs.
The exchange is one all-gather of each rank's OWN entries -- (range id,
7-byte record, pre RMS, post RMS) packed in 32 bytes, padded to the largest
shard -- followed by a scatter by range id on the device.  No other
collective is needed: ranges are independent (codec.py:386-397 writes
disjoint slots).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

ENTRY = 32  # bytes per exchanged range: id u32 | record 7 B | pad 5 | pre f64 | post f64


def pack_owned(records: torch.Tensor, pre_rms: torch.Tensor, post_rms: torch.Tensor):
    """(n, 32) uint8 entries of the ranges this rank matched (post_rms >= 0;
    unmatched ranges hold the -1 sentinel ``encode_sharded`` fills in)."""
    ids = torch.nonzero(post_rms >= 0).squeeze(1)
    n = ids.numel()
    buf = torch.zeros((n, ENTRY), dtype=torch.uint8, device=records.device)
    buf[:, 0:4] = ids.to(torch.int32).view(torch.uint8).view(n, 4)
    buf[:, 4:11] = records[ids]
    buf[:, 16:24] = pre_rms[ids].contiguous().view(torch.uint8).view(n, 8)
    buf[:, 24:32] = post_rms[ids].contiguous().view(torch.uint8).view(n, 8)
    return buf


def gather_shards(records: torch.Tensor, pre_rms: torch.Tensor, post_rms: torch.Tensor,
                  group=None):
    """Exchange every rank's own ranges; returns the full (records, pre, post).

    records (R, 7) uint8, pre_rms/post_rms (R,) float64 with post_rms < 0 on
    ranges this rank did not match.  NCCL (CUDA tensors) or gloo (the
    exchange then runs on host copies).  Raises if a range is owned by no
    rank or by more than one.
    """
    world = dist.get_world_size(group)
    dev = records.device
    host = dist.get_backend(group) == "gloo"
    mine = pack_owned(records, pre_rms, post_rms)
    xdev = torch.device("cpu") if host else dev
    cnt = torch.tensor([mine.shape[0]], dtype=torch.int64, device=xdev)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    counts = [int(c) for c in counts]
    mx = max(counts)
    send = torch.zeros((mx, ENTRY), dtype=torch.uint8, device=xdev)
    send[:mine.shape[0]] = mine.to(xdev)
    if host:
        parts = [torch.empty_like(send) for _ in range(world)]
        dist.all_gather(parts, send, group=group)
        allb = torch.cat(parts)
    else:
        allb = torch.empty((world * mx, ENTRY), dtype=torch.uint8, device=xdev)
        dist.all_gather_into_tensor(allb, send, group=group)
    keep = torch.cat([torch.arange(k * mx, k * mx + c) for k, c in enumerate(counts)])
    ent = allb[keep.to(allb.device)].to(dev)
    n_r = records.shape[0]
    if ent.shape[0] != n_r:
        raise RuntimeError(f"shards cover {ent.shape[0]} range entries for {n_r} ranges")
    ids = ent[:, 0:4].contiguous().view(torch.int32).view(-1).to(torch.int64)
    seen = torch.zeros(n_r, dtype=torch.int32, device=dev)
    seen.index_add_(0, ids, torch.ones_like(ids, dtype=torch.int32))
    if not bool((seen == 1).all()):
        raise RuntimeError("some ranges were matched by no rank or by several")
    out_rec = torch.empty_like(records)
    out_pre = torch.empty_like(pre_rms)
    out_post = torch.empty_like(post_rms)
    out_rec[ids] = ent[:, 4:11]
    out_pre[ids] = ent[:, 16:24].contiguous().view(torch.float64).view(-1)
    out_post[ids] = ent[:, 24:32].contiguous().view(torch.float64).view(-1)
    return out_rec, out_pre, out_post


def encode_sharded(image_dev: torch.Tensor, strategy: str = "dynamic_fd", *, group=None,
                   **kwargs):
    """Encode on every rank of ``group`` (one GPU each) and all-gather.

    Returns (records (R,7) uint8, pre_rms, post_rms, pool_sizes, stats) as
    CUDA tensors, identical on every rank and byte-identical to a 1-GPU run.
    """
    from .codec import DeviceResult, encode_device, validate

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    rs = kwargs.get("range_size", 8)
    _, h, w = validate(image_dev, strategy, rs, kwargs.get("domain_size", 16),
                       kwargs.get("stride", 1), kwargs.get("fd_source", "original"))
    n_r = (h // rs) * (w // rs)
    dev = image_dev.device
    out = DeviceResult(
        torch.zeros((n_r, 7), dtype=torch.uint8, device=dev),
        torch.full((n_r,), -1.0, dtype=torch.float64, device=dev),
        torch.full((n_r,), -1.0, dtype=torch.float64, device=dev),
        torch.zeros(n_r, dtype=torch.int64, device=dev), {})
    res = encode_device(image_dev, strategy, shard=(rank, world), out=out, **kwargs)
    recs, pre, post = gather_shards(res.records, res.pre_rms, res.post_rms, group)
    return recs, pre, post, res.pool_sizes, res.stats
