"""One cfg5 encode-plan for profiling the pool builder (ncu -k regex:k_pool)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_1206_4880_b200 import codec, synth
name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
c = synth.CONFIGS[name]
img = torch.from_numpy(c.make()).cuda()
res = codec.encode_device(img, c.strategy, range_size=c.range_size, domain_size=c.domain_size,
                          stride=c.stride, isometries=True, delta=c.delta, max_segment=256)
torch.cuda.synchronize()
print(res.stats["ms_pool"], res.stats["ms_fd"])
