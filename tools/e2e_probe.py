"""Per-stage host timing of codec.encode on cfg3 (same steps as the function)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth  # noqa: E402

c = synth.CONFIGS["cfg3"]
im = c.make()
kw = dict(range_size=8, domain_size=16, stride=1, isometries=True, delta=c.delta)
for _ in range(3):
    codec.encode(im, "dynamic_fd", **kw)
dev = torch.device("cuda", 0)
T = {}
N = 10
for _ in range(N):
    ts = [time.perf_counter()]
    image, h, w = codec.validate(im, "dynamic_fd", 8, 16, 1, "original"); ts.append(time.perf_counter())
    st = codec._staging(torch, dev, h, w, 16384); ts.append(time.perf_counter())
    st.h_img.numpy()[...] = image; ts.append(time.perf_counter())
    st.d_img.copy_(st.h_img, non_blocking=True); ts.append(time.perf_counter())
    res = codec.encode_device(st.d_img, "dynamic_fd", out=st.result(), **kw); ts.append(time.perf_counter())
    st.h_out.copy_(st.d_out, non_blocking=True); torch.cuda.current_stream(dev).synchronize(); ts.append(time.perf_counter())
    pre, post, pools, records = st.host_views()
    records = records.copy().view(codec.RECORD_DTYPE).ravel(); pre, post, pools = pre.copy(), post.copy(), pools.copy()
    ts.append(time.perf_counter())
    for k, (a, b) in zip(["validate", "staging", "pinned copy", "h2d issue", "encode_device", "d2h+sync", "numpy"], zip(ts, ts[1:])):
        T[k] = T.get(k, 0) + (b - a)
    T["total"] = T.get("total", 0) + ts[-1] - ts[0]
    T["ms_total(dev)"] = T.get("ms_total(dev)", 0) + res.stats["ms_total"] / 1e3
for k, v in T.items():
    print(f"{k:16s} {v / N * 1e3:.3f} ms")
t0 = time.perf_counter()
for _ in range(N):
    codec.encode(im, "dynamic_fd", **kw)
print("codec.encode    %.3f ms" % ((time.perf_counter() - t0) / N * 1e3))
