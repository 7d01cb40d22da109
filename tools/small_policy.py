"""Device ms per encode (median of 7) with the default matcher choice and
with every range on the exact (CUDA-core) matcher, for the small configs:
    python tools/small_policy.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth  # noqa: E402

for name in ("cfg1", "cfg2"):
    c = synth.CONFIGS[name]
    img = torch.from_numpy(c.make()).cuda()
    for strat in (c.strategy, "exhaustive"):
        for matcher in ("auto", "exact"):
            kw = dict(range_size=c.range_size, domain_size=c.domain_size, stride=c.stride,
                      isometries=True, delta=c.delta if strat == c.strategy else None, matcher=matcher)
            codec.encode_device(img, strat, **kw)
            ms = sorted(codec.encode_device(img, strat, **kw).stats["ms_total"] for _ in range(7))[3]
            st = codec.encode_device(img, strat, **kw).stats
            print(name, strat, matcher, "%.3f ms" % ms, "comparisons %.3g" % st["comparisons"],
                  "tensor_tiles", st["tensor_tiles"], flush=True)
