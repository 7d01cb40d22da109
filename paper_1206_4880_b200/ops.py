"""``torch.ops.fic.encode``: the PyTorch operator SURVEY.md §8(b) names for the
encoder boundary, registered with ``torch.library`` on import.

    records_u8[R,7], pre_rms_f64[R], post_rms_f64[R], pool_sizes_i64[R], stats_f64[S] =
        torch.ops.fic.encode(image_u8[H,W] (cuda), range_size, domain_size, stride,
                             isometries, strategy_id, delta, fd_source)

It is backed by the same C ABI as ``codec.encode_device`` (``fic_encode_v1``,
include/fic_b200.h), on the image's device and current stream; the outputs
stay on the device except ``stats`` (host float64, fields ``STATS_FIELDS``).
``strategy_id`` follows the reference's numbering (codec.py:17-18: 0
exhaustive, 1 nosearch, 2 static2, 3 dynamic_fd); ``delta`` None is the
reference's D_f rule; ``fd_source`` 0 = "original", 1 = "downsampled"
(codec.py:320-321).  Errors raise the reference's ValueError texts.
"""

from __future__ import annotations

import torch

from . import _lib, codec

STATS_FIELDS = tuple(name for name, _ in _lib.FicStats._fields_)
FD_SOURCES = ("original", "downsampled")


@torch.library.custom_op("fic::encode", mutates_args=())
def encode(image: torch.Tensor, range_size: int, domain_size: int, stride: int, isometries: bool,
           strategy_id: int, delta: float | None, fd_source: int
           ) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor]:
    if not 0 <= strategy_id < len(codec.STRATEGIES):
        raise ValueError(f"unknown strategy id {strategy_id}")
    if fd_source not in (0, 1):
        raise ValueError(f"unknown fd_source id {fd_source}")
    res = codec.encode_device(image, codec.STRATEGIES[strategy_id], range_size=range_size,
                              domain_size=domain_size, stride=stride, isometries=isometries,
                              fd_source=FD_SOURCES[fd_source], delta=delta)
    stats = torch.tensor([float(res.stats[k]) for k in STATS_FIELDS], dtype=torch.float64)
    return res.records, res.pre_rms, res.post_rms, res.pool_sizes, stats


@encode.register_fake
def _(image, range_size, domain_size, stride, isometries, strategy_id, delta, fd_source):
    h, w = image.shape
    n_r = (h // range_size) * (w // range_size)
    new = image.new_empty
    return (new((n_r, 7), dtype=torch.uint8), new(n_r, dtype=torch.float64),
            new(n_r, dtype=torch.float64), new(n_r, dtype=torch.int64),
            torch.empty(len(STATS_FIELDS), dtype=torch.float64, device="cpu"))
