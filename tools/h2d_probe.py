"""Time the host->device staging of codec.encode: pinned copy, H2D, clear."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth  # noqa: E402

im = synth.CONFIGS["cfg3"].make()
dev = torch.device("cuda", 0)
st = codec._staging(torch, dev, 1024, 1024, 16384)
for _ in range(3):
    st.d_img.copy_(st.h_img, non_blocking=True)
torch.cuda.synchronize()
T = {}
for _ in range(20):
    t0 = time.perf_counter(); st.h_img.numpy()[...] = im; t1 = time.perf_counter()
    st.d_img.copy_(st.h_img, non_blocking=True); t2 = time.perf_counter()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    st.d_out.zero_(); torch.cuda.synchronize(); t4 = time.perf_counter()
    for k, v in (("pinned copy", t1 - t0), ("h2d issue", t2 - t1), ("h2d wait", t3 - t2), ("zero+sync", t4 - t3)):
        T[k] = T.get(k, 0) + v
for k, v in T.items():
    print(f"{k:12s} {v / 20 * 1e3:.3f} ms")
print("pinned:", st.h_img.is_pinned())
