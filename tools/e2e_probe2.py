"""Which part of codec.encode's Python wrapper costs time (cfg3)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth  # noqa: E402

c = synth.CONFIGS["cfg3"]
im = c.make()
kw = dict(range_size=8, domain_size=16, stride=1, isometries=True, delta=c.delta)
for _ in range(3):
    codec.encode(im, "dynamic_fd", **kw)
dev = torch.device("cuda", 0)
N = 200


def t(name, f):
    t0 = time.perf_counter()
    for _ in range(N):
        f()
    print(f"{name:28s} {(time.perf_counter() - t0) / N * 1e6:8.1f} us")


t("torch.cuda.is_available", torch.cuda.is_available)
t("current_device", torch.cuda.current_device)
t("device ctx enter/exit", lambda: torch.cuda.device(dev).__enter__() or None)


def ctx():
    with torch.cuda.device(dev):
        pass


t("with torch.cuda.device", ctx)
t("current_stream", lambda: torch.cuda.current_stream(dev).cuda_stream)
st = codec._staging(torch, dev, 1024, 1024, 16384)
t("host_views+copies", lambda: [x.copy() for x in st.host_views()])
N = 10
t0 = time.perf_counter()
for _ in range(N):
    codec.encode(im, "dynamic_fd", **kw)
print("codec.encode %.3f ms" % ((time.perf_counter() - t0) / N * 1e3))
t0 = time.perf_counter()
for _ in range(N):
    codec.encode_device(st.d_img, "dynamic_fd", out=st.result(), **kw)
    torch.cuda.synchronize()
print("encode_device %.3f ms" % ((time.perf_counter() - t0) / N * 1e3))
