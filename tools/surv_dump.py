"""Per-range survivor counts of the tensor screen (FIC_SURV_DUMP) next to
each range's V and pool, for tuning the bulk hand-over:
    python tools/surv_dump.py cfg4 [FIC_BULK_MIN] [FIC_BULK_SHIFT]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth  # noqa: E402

name = sys.argv[1]
os.environ["FIC_BULK_MIN"] = sys.argv[2] if len(sys.argv) > 2 else "2000000000"
os.environ["FIC_BULK_SHIFT"] = sys.argv[3] if len(sys.argv) > 3 else "0"
out = f"gpurun_out/surv_{name}_{os.environ['FIC_BULK_MIN']}_{os.environ['FIC_BULK_SHIFT']}.npz"
os.environ["FIC_SURV_DUMP"] = "/tmp/surv.bin"
c = synth.CONFIGS[name]
img = c.make()
d = torch.from_numpy(img).cuda()
kw = dict(range_size=c.range_size, domain_size=c.domain_size, stride=c.stride, isometries=True,
          delta=c.delta)
res = codec.encode_device(d, c.strategy, **kw)
torch.cuda.synchronize()
h = np.fromfile("/tmp/surv.bin", dtype=np.uint32)
R = len(h) // 2
rs = c.range_size
blk = img.reshape(img.shape[0] // rs, rs, img.shape[1] // rs, rs).transpose(0, 2, 1, 3).reshape(R, -1)
blk = blk.astype(np.float64)
V = (blk * blk).sum(1) - blk.sum(1) ** 2 / blk.shape[1]
np.savez_compressed(out, surv=h[:R], bulk=h[R:], V=V, pool=res.pool_sizes.cpu().numpy(),
                    post=res.post_rms.cpu().numpy())
st = res.stats
print(name, {k: st[k] for k in ("ms_total", "ms_tensor", "ms_bulk", "exact_evals", "bulk_ranges")})
s = h[:R]
for q in (0, 100, 1000, 10000, 100000, 1000000):
    print(f"  ranges with > {q} survivors: {(s > q).sum()}  (sum {s[s > q].sum():.3g})")
