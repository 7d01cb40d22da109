"""cfg3 encodes with a variant library (FIC_B200_LIB), printing the library's stderr counters."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth  # noqa: E402

c = synth.CONFIGS["cfg3"]
img = torch.from_numpy(c.make()).cuda()
kw = dict(range_size=8, domain_size=16, stride=1, isometries=True, delta=c.delta)
for _ in range(3):
    r = codec.encode_device(img, "dynamic_fd", **kw)
    torch.cuda.synchronize()
    print("ms_tensor", r.stats["ms_tensor"], "items", r.stats["work_items"], flush=True)
