"""ms_tensor at cfg3 for a few segment lengths (work-item granularity)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth  # noqa: E402

c = synth.CONFIGS["cfg3"]
img = torch.from_numpy(c.make()).cuda()
kw = dict(range_size=8, domain_size=16, stride=1, isometries=True, delta=c.delta)
segs = [int(x) for x in sys.argv[1:]] or [32768, 65536, 98304, 131072, 196608]
for _ in range(2):
    codec.encode_device(img, "dynamic_fd", **kw)
for seg in segs:
    ts = []
    for _ in range(4):
        r = codec.encode_device(img, "dynamic_fd", max_segment=seg, **kw)
        torch.cuda.synchronize()
        ts.append(r.stats["ms_tensor"])
    print(seg, "ms_tensor %.3f min %.3f" % (sum(ts[1:]) / 3, min(ts)), "items", r.stats["work_items"], flush=True)
