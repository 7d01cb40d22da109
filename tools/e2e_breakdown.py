"""Host-side breakdown of one codec.encode at cfg3 (perf_counter, mean of 20):
validate+staging copy, H2D+encode_device (library call incl. its sync),
D2H+sync, host copies/objects; beside the device-timed ms_total."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth  # noqa: E402

c = synth.CONFIGS["cfg3"]
img = c.make()
kw = dict(range_size=8, domain_size=16, stride=1, isometries=True, delta=0.05)
for _ in range(3):
    codec.encode(img, "dynamic_fd", **kw)
torch.cuda.synchronize()
T = []
for _ in range(20):
    t0 = time.perf_counter()
    code, st = codec.encode(img, "dynamic_fd", **kw)
    T.append((time.perf_counter() - t0, st.device["ms_total"]))
T = np.array(T)
print("e2e %.3f ms (device ms_total %.3f)" % (T[:, 0].mean() * 1e3, T[:, 1].mean()))
# phases, replicated from codec.encode
dev = torch.device("cuda", 0)
n_r = (1024 // 8) ** 2
stage = codec._staging(torch, dev, 1024, 1024, n_r)
P = []
for _ in range(20):
    t0 = time.perf_counter()
    stage.h_img.copy_(torch.from_numpy(np.ascontiguousarray(img)))
    stage.d_img.copy_(stage.h_img, non_blocking=True)
    t1 = time.perf_counter()
    res = codec.encode_device(stage.d_img, "dynamic_fd", out=stage.result(), **kw)
    t2 = time.perf_counter()
    stage.h_out.copy_(stage.d_out, non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()
    t3 = time.perf_counter()
    pre, post, pools, records = stage.host_views()
    records = records.copy().view(codec.RECORD_DTYPE).ravel()
    pre, post, pools = pre.copy(), post.copy(), pools.copy()
    t4 = time.perf_counter()
    P.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3, res.stats["ms_total"] / 1e3))
P = np.array(P).mean(0) * 1e3
print("staging %.3f | encode_device %.3f (device %.3f) | D2H+sync %.3f | host copies %.3f ms"
      % (P[0], P[1], P[4], P[2], P[3]))
