"""A/B timing of an env knob read per call by the library: alternates the
settings on cfg3 encodes in one process, prints mean/min ms_tensor and ms_total.

    python tools/ab_env.py FIC_TC_SPLIT 1 4 [rounds]
"""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth  # noqa: E402

var, vals = sys.argv[1], sys.argv[2:]
rounds = 8
if vals and vals[-1].startswith("x"):
    rounds = int(vals.pop()[1:])
c = synth.CONFIGS["cfg3"]
img = torch.from_numpy(c.make()).cuda()
kw = dict(range_size=8, domain_size=16, stride=1, isometries=True, delta=c.delta)
ref = None
res = {v: ([], []) for v in vals}
for _ in range(2):
    codec.encode_device(img, "dynamic_fd", **kw)
for r in range(rounds):
    for v in vals:
        os.environ[var] = v
        out = codec.encode_device(img, "dynamic_fd", **kw)
        torch.cuda.synchronize()
        res[v][0].append(out.stats["ms_tensor"])
        res[v][1].append(out.stats["ms_total"])
        if ref is None:
            ref = out.records.clone()
        assert torch.equal(ref, out.records), (var, v)
for v in vals:
    t, tt = res[v]
    print(f"{var}={v}: ms_tensor mean {sum(t)/len(t):.3f} min {min(t):.3f} | ms_total mean {sum(tt)/len(tt):.3f} min {min(tt):.3f}")
