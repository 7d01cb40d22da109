"""Worst-rank device ms of the range-sharded cfg3 encode against the matcher's segment length (max_segment; 0 = the default 131072):
    python tools/seg_probe.py"""
import sys, torch
sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth
c = synth.CONFIGS["cfg3"]
img = torch.from_numpy(c.make()).cuda()
kw = dict(range_size=8, domain_size=16, stride=1, isometries=True, delta=0.05)
def med(shard, seg):
    codec.encode_device(img, c.strategy, shard=shard, max_segment=seg, **kw)
    v = sorted(codec.encode_device(img, c.strategy, shard=shard, max_segment=seg, **kw).stats["ms_total"] for _ in range(5))
    return v[2]
import os
for n in (1, 8):
    for seg in (0, 98304, 196608, 262144, 393216, 524288, 1048576):
        worst = max(med((k, n), seg) for k in range(n))
        print("N", n, "max_segment", seg, "worst rank ms %.3f" % worst, flush=True)
