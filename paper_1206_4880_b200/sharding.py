"""Range sharding across GPUs: one process per GPU, NCCL all-gather of records.

Every rank holds the whole image (<= 64 MB) and recomputes FD, the FD index
and the pool (sub-millisecond), so every rank derives the same FD-sorted,
cost-balanced partition of ranges without communication.
Each rank matches only its shard (``fic_params_t.shard_index/count``); the
per-range transforms are then exchanged with one all-gather and each range
takes the value of the rank that owns it.  No other collective is needed:
ranges are independent (codec.py:386-397 writes disjoint slots).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def gather_shards(records: torch.Tensor, pre_rms: torch.Tensor, post_rms: torch.Tensor,
                  group=None):
    """All-gather per-rank shard outputs and keep each range's owner value.

    records (R, 7) uint8, pre_rms/post_rms (R,) float64, with post_rms < 0 on
    ranges this rank did not match.  Works with NCCL (CUDA tensors) and gloo
    (CPU tensors); returns the full (records, pre_rms, post_rms).
    """
    world = dist.get_world_size(group)
    rms = torch.stack([pre_rms, post_rms], dim=1).contiguous()
    rec_list = [torch.empty_like(records) for _ in range(world)]
    rms_list = [torch.empty_like(rms) for _ in range(world)]
    dist.all_gather(rec_list, records.contiguous(), group=group)
    dist.all_gather(rms_list, rms, group=group)
    recs = torch.stack(rec_list)            # (world, R, 7)
    rmss = torch.stack(rms_list)            # (world, R, 2)
    owned = rmss[:, :, 1] >= 0              # (world, R)
    if not bool(owned.any(dim=0).all()):
        raise RuntimeError("some ranges were matched by no rank")
    owner = owned.to(torch.int8).argmax(dim=0)          # (R,)
    idx = torch.arange(records.shape[0], device=records.device)
    return recs[owner, idx], rmss[owner, idx, 0], rmss[owner, idx, 1]


def encode_sharded(image_dev: torch.Tensor, strategy: str = "dynamic_fd", *, group=None,
                   **kwargs):
    """Encode on every rank of ``group`` (one GPU each) and all-gather.

    Returns (records (R,7) uint8, pre_rms, post_rms, pool_sizes, stats) as
    CUDA tensors, identical on every rank and byte-identical to a 1-GPU run.
    """
    from .codec import DeviceResult, encode_device, validate

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    _, h, w = validate(image_dev, strategy, kwargs.get("range_size", 8),
                       kwargs.get("domain_size", 16), kwargs.get("stride", 1),
                       kwargs.get("fd_source", "original"))
    n_r = (h // kwargs.get("range_size", 8)) * (w // kwargs.get("range_size", 8))
    dev = image_dev.device
    out = DeviceResult(
        torch.zeros((n_r, 7), dtype=torch.uint8, device=dev),
        torch.full((n_r,), -1.0, dtype=torch.float64, device=dev),
        torch.full((n_r,), -1.0, dtype=torch.float64, device=dev),
        torch.zeros(n_r, dtype=torch.int64, device=dev), {})
    res = encode_device(image_dev, strategy, shard=(rank, world), out=out, **kwargs)
    recs, pre, post = gather_shards(res.records, res.pre_rms, res.post_rms, group)
    return recs, pre, post, res.pool_sizes, res.stats
