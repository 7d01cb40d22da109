"""Per-rank device time of the range-sharded encode at N GPUs, measured on
one GPU: encode_device(shard=(k, N)) is exactly the work rank k does (full
FD / pool / planning, its cost-balanced shard of the matcher); the max over
k, plus the measured exchange, bounds the N-GPU step.  Not a multi-GPU run.
    python tools/shard_projection.py [cfg3]"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
c = synth.CONFIGS[name]
img = torch.from_numpy(c.make()).cuda()
kw = dict(range_size=c.range_size, domain_size=c.domain_size, stride=c.stride, isometries=True,
          delta=c.delta)
reps = 5 if name != "cfg5" else 1


def med(shard):
    codec.encode_device(img, c.strategy, shard=shard, **kw)
    v = sorted(codec.encode_device(img, c.strategy, shard=shard, **kw).stats["ms_total"]
               for _ in range(reps))
    return v[len(v) // 2]


one = med((0, 1))
for n in (2, 4, 8):
    per = [med((k, n)) for k in range(n)]
    print(json.dumps({"config": name, "n": n, "ms_one_gpu": one, "ms_per_rank_max": max(per),
                      "ms_per_rank": per, "projected_efficiency_no_exchange": one / (n * max(per))}),
          flush=True)
