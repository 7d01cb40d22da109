import sys, time; sys.path.insert(0, ".")
import torch
from paper_1206_4880_b200 import codec, synth
c = synth.CONFIGS["cfg5"]
t = time.time(); im = c.make(); print("gen", time.time() - t, im.shape, flush=True)
img = torch.from_numpy(im).cuda()
for i in range(2):
    res = codec.encode_device(img, c.strategy, range_size=c.range_size, domain_size=c.domain_size, stride=c.stride, isometries=True, delta=c.delta)
    torch.cuda.synchronize()
    st = res.stats
    print({k: st[k] for k in ("ms_total", "ms_fd", "ms_pool", "ms_tensor", "ms_exact", "exact_evals", "comparisons", "work_items")}, "matches/s %.3g" % (st["comparisons"] / st["ms_total"] * 1e3), flush=True)
