"""Encodes of one config with a variant library (FIC_B200_LIB), for the
FIC_TC_PROF / FIC_PLAN_TIMING stderr counters:  python tools/tc_prof_cfg.py cfg4"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth  # noqa: E402

c = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
img = torch.from_numpy(c.make()).cuda()
kw = dict(range_size=c.range_size, domain_size=c.domain_size, stride=c.stride, isometries=True,
          delta=c.delta)
for _ in range(2):
    r = codec.encode_device(img, c.strategy, **kw)
    torch.cuda.synchronize()
    print("ms_tensor", r.stats["ms_tensor"], "exact_evals", r.stats["exact_evals"], flush=True)
