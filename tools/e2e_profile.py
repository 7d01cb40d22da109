import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
from paper_1206_4880_b200 import codec, synth
c = synth.CONFIGS["cfg3"]
im = c.make()
kw = dict(range_size=c.range_size, domain_size=c.domain_size, stride=c.stride, isometries=True, delta=c.delta)
for i in range(3): codec.encode(im, c.strategy, **kw)
torch.cuda.synchronize()
import cProfile, pstats
t = time.perf_counter()
for i in range(10): codec.encode(im, c.strategy, **kw)
print("e2e ms", (time.perf_counter() - t) / 10 * 1e3)
img = torch.from_numpy(im).cuda()
torch.cuda.synchronize()
t = time.perf_counter()
for i in range(10):
    r = codec.encode_device(img, c.strategy, **kw)
torch.cuda.synchronize()
print("device-call ms", (time.perf_counter() - t) / 10 * 1e3, "ms_total", r.stats["ms_total"])
t = time.perf_counter()
for i in range(20): codec.make_params(c.strategy, 8, 16, 1, True, "original", 0.05, "auto", (0, 1))
print("make_params ms", (time.perf_counter() - t) / 20 * 1e3)
t = time.perf_counter()
for i in range(20):
    x = torch.from_numpy(np.ascontiguousarray(im)).cuda(); torch.cuda.synchronize()
print("h2d ms", (time.perf_counter() - t) / 20 * 1e3)
t = time.perf_counter()
for i in range(20):
    a = r.records.cpu(); b = r.pre_rms.cpu(); cc = r.post_rms.cpu(); d = r.pool_sizes.cpu()
print("4 d2h ms", (time.perf_counter() - t) / 20 * 1e3)
pr = cProfile.Profile(); pr.enable()
for i in range(5): codec.encode(im, c.strategy, **kw)
pr.disable(); pstats.Stats(pr).sort_stats("cumtime").print_stats(12)
