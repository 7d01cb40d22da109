"""Range sharding across GPUs: one process per GPU, one reduction of records.

Every rank holds the whole image (<= 64 MB) and recomputes FD, the FD index
and the pool (sub-millisecond), so every rank derives the same FD-sorted,
cost-balanced partition of ranges without communication (the
library sorts the ranges deterministically when sharded, fic_api.cu
k_range_scatter_stable).  Each rank matches only its shard
(``fic_params_t.shard_index/count``) and writes only its ranges' outputs.
The exchange is one all-reduce (SUM) of the full-length outputs packed in
an int64 (R, 3) buffer with zeros outside the rank's own ranges -- the
record bytes plus an owner-count byte, and the bits of the RMS pair -- so
every range has exactly one non-zero contribution and the sum reproduces
its bytes.  No compaction, no count exchange: the
only host synchronisation is the check that every range has exactly one
owner.  Ranges are independent (codec.py:386-397 writes disjoint slots).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def _pack_host(records, pre_rms, post_rms):
    """The pack of fic_shard_pack_v1 in torch ops (host tensors)."""
    n_r = records.shape[0]
    owned = post_rms >= 0
    buf = torch.zeros((n_r, 3), dtype=torch.int64, device=records.device)
    b8 = buf.view(torch.uint8).view(n_r, 24)
    b8[:, :7] = records
    b8[:, 7] = 1
    buf[:, 1] = pre_rms.view(torch.int64)
    buf[:, 2] = post_rms.view(torch.int64)
    return buf.mul_(owned.to(torch.int64)[:, None])


def gather_shards(records: torch.Tensor, pre_rms: torch.Tensor, post_rms: torch.Tensor,
                  group=None):
    """Combine every rank's own ranges; returns the full (records, pre, post).

    records (R, 7) uint8, pre_rms/post_rms (R,) float64 with post_rms < 0 on
    ranges this rank did not match.  One all-reduce (SUM) of an int64 (R, 3)
    buffer: the 7 record bytes plus an owner-count byte, and the bits of the
    two RMS values -- zero outside the rank's own ranges, so each range has
    one non-zero contribution and the integer sum reproduces its bytes.  On
    CUDA tensors the pack and the unpack are one library kernel each
    (fic_shard_pack_v1 / fic_shard_unpack_v1).  NCCL, or gloo (host copies).
    Raises if a range is owned by no rank or by more than one (its count
    byte is then 0 or >= 2: record carries add at most the number of owners).
    """
    import ctypes

    from . import _lib
    from .codec import _stream

    dev = records.device
    host = dist.get_backend(group) == "gloo"
    n_r = records.shape[0]
    cuda = dev.type == "cuda"
    if cuda:
        lib = _lib.load()
        stream = _stream(torch, dev)
        records, pre_rms, post_rms = records.contiguous(), pre_rms.contiguous(), post_rms.contiguous()
        buf = torch.empty((n_r, 3), dtype=torch.int64, device=dev)
        _lib.check(lib.fic_shard_pack_v1(
            ctypes.c_void_p(records.data_ptr()), ctypes.c_void_p(pre_rms.data_ptr()),
            ctypes.c_void_p(post_rms.data_ptr()), n_r, ctypes.c_void_p(buf.data_ptr()), stream))
    else:
        buf = _pack_host(records, pre_rms, post_rms)
    x = buf.cpu() if host and cuda else buf
    dist.all_reduce(x, op=dist.ReduceOp.SUM, group=group)
    if x is not buf:
        buf.copy_(x)
    if cuda:
        out_rec = torch.empty((n_r, 7), dtype=torch.uint8, device=dev)
        out_pre = torch.empty(n_r, dtype=torch.float64, device=dev)
        out_post = torch.empty(n_r, dtype=torch.float64, device=dev)
        bad = torch.empty(1, dtype=torch.int32, device=dev)
        _lib.check(lib.fic_shard_unpack_v1(
            ctypes.c_void_p(buf.data_ptr()), n_r, ctypes.c_void_p(out_rec.data_ptr()),
            ctypes.c_void_p(out_pre.data_ptr()), ctypes.c_void_p(out_post.data_ptr()),
            ctypes.c_void_p(bad.data_ptr()), stream))
        ok = int(bad.item()) == 0
    else:
        b8 = buf.view(torch.uint8).view(n_r, 24)
        ok = bool((b8[:, 7] == 1).all())
        out_rec = b8[:, :7].contiguous()
        out_pre = buf[:, 1].contiguous().view(torch.float64)
        out_post = buf[:, 2].contiguous().view(torch.float64)
    if not ok:
        raise RuntimeError("some ranges were matched by no rank or by several")
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
    # only post RMS needs a value outside the rank's ranges (the -1 the
    # exchange reads as "not mine"); the library writes the rest
    out = DeviceResult(
        torch.empty((n_r, 7), dtype=torch.uint8, device=dev),
        torch.empty(n_r, dtype=torch.float64, device=dev),
        torch.full((n_r,), -1.0, dtype=torch.float64, device=dev),
        torch.zeros(n_r, dtype=torch.int64, device=dev), {})
    res = encode_device(image_dev, strategy, shard=(rank, world), out=out, **kwargs)
    recs, pre, post = gather_shards(res.records, res.pre_rms, res.post_rms, group)
    return recs, pre, post, res.pool_sizes, res.stats
