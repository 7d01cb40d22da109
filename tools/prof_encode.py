"""One cfg3 encode for profiling (ncu launch list / --set full of k_match_tc)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
c = synth.CONFIGS[name]
img = torch.from_numpy(c.make()).cuda()
res = codec.encode_device(img, c.strategy, range_size=c.range_size, domain_size=c.domain_size,
                          stride=c.stride, isometries=True, delta=c.delta)
torch.cuda.synchronize()
print({k: res.stats[k] for k in ("ms_total", "ms_tensor", "exact_evals", "comparisons")})
