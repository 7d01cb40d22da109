"""cfg3 encodes with the FIC_PLAN_TIMING phase timer (prints per-phase ms to stderr)."""
import os
import sys

os.environ.setdefault("FIC_PLAN_TIMING", "1")
import torch

sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 5
c = synth.CONFIGS[name]
img = torch.from_numpy(c.make()).cuda()
for _ in range(n):
    res = codec.encode_device(img, c.strategy, range_size=c.range_size, domain_size=c.domain_size,
                              stride=c.stride, isometries=True, delta=c.delta)
    torch.cuda.synchronize()
    print({k: round(res.stats[k], 4) if isinstance(res.stats[k], float) else res.stats[k]
           for k in ("ms_total", "ms_fd", "ms_pool", "ms_tensor", "ms_exact")}, flush=True)
