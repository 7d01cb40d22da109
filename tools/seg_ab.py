"""Interleaved A/B of the work-item segment length on cfg3 (ms_tensor mean/min)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth  # noqa: E402

c = synth.CONFIGS["cfg3"]
img = torch.from_numpy(c.make()).cuda()
kw = dict(range_size=8, domain_size=16, stride=1, isometries=True, delta=c.delta)
segs = [int(x) for x in sys.argv[1:]]
res = {s: [] for s in segs}
for _ in range(2):
    codec.encode_device(img, "dynamic_fd", **kw)
for r in range(6):
    for seg in segs:
        out = codec.encode_device(img, "dynamic_fd", max_segment=seg, **kw)
        torch.cuda.synchronize()
        res[seg].append(out.stats["ms_tensor"])
for seg in segs:
    t = res[seg]
    print(seg, "mean %.3f min %.3f" % (sum(t) / len(t), min(t)), "items", out.stats["work_items"])
