"""Host-side phases of one public codec.encode call at cfg3 (median of 20):
validation, pinned staging copy, the library call (enqueue + its final
stats sync), output D2H + sync, host copies.
    python tools/e2e_probe.py"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth  # noqa: E402

CFG = dict(range_size=8, domain_size=16, stride=1, isometries=True, delta=0.05)
img = synth.cfg3_image()
for _ in range(3):
    codec.encode(img, "dynamic_fd", **CFG)
torch.cuda.synchronize()
ph = {k: [] for k in ("validate", "stage", "lib_call", "d2h", "host_copy", "total", "ms_total_dev")}
dev = torch.device("cuda", 0)
for _ in range(20):
    t0 = time.perf_counter()
    image, h, w = codec.validate(img, "dynamic_fd", 8, 16, 1, "original")
    n_r = (h // 8) * (w // 8)
    st = codec._staging(torch, dev, h, w, n_r)
    t1 = time.perf_counter()
    st.h_img.copy_(torch.from_numpy(np.ascontiguousarray(image)))
    st.d_img.copy_(st.h_img, non_blocking=True)
    t2 = time.perf_counter()
    res = codec.encode_device(st.d_img, "dynamic_fd", out=st.result(), **CFG)
    t3 = time.perf_counter()
    st.h_out.copy_(st.d_out, non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()
    t4 = time.perf_counter()
    pre, post, pools, records = st.host_views()
    records = records.copy().view(codec.RECORD_DTYPE).ravel()
    pre, post, pools = pre.copy(), post.copy(), pools.copy()
    t5 = time.perf_counter()
    for k, v in zip(ph, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t5 - t0)):
        ph[k].append(1e3 * v)
    ph["ms_total_dev"].append(res.stats["ms_total"])
print(json.dumps({k: float(np.median(v)) for k, v in ph.items()}))
t = []
for _ in range(20):
    t0 = time.perf_counter()
    codec.encode(img, "dynamic_fd", **CFG)
    t.append(1e3 * (time.perf_counter() - t0))
print(json.dumps({"codec.encode_ms_median": float(np.median(t))}))
