"""Time the steps of codec.encode() on cfg3 (host image in, host results out)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1206_4880_b200 import codec, synth

c = synth.CONFIGS["cfg3"]
im = c.make()
kw = dict(range_size=c.range_size, domain_size=c.domain_size, stride=c.stride, isometries=True, delta=c.delta)
for _ in range(3):
    codec.encode(im, c.strategy, **kw)
torch.cuda.synchronize()
dev = torch.device("cuda", 0)
h, w = im.shape
n_r = (h // 8) * (w // 8)
T = {}
def t(name, t0):
    T[name] = T.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
for _ in range(10):
    t0 = time.perf_counter(); img, hh, ww = codec.validate(im, c.strategy, 8, 16, 1, "original"); t("validate", t0)
    t0 = time.perf_counter(); st = codec._staging(torch, dev, h, w, n_r); t("staging lookup", t0)
    t0 = time.perf_counter(); st.h_img.numpy()[...] = im; t("host copy to pinned", t0)
    t0 = time.perf_counter(); st.d_img.copy_(st.h_img, non_blocking=True); st.d_out.zero_(); t("h2d issue + zero", t0)
    t0 = time.perf_counter(); res = codec.encode_device(st.d_img, c.strategy, out=st.result(), **kw); t("encode_device", t0)
    t0 = time.perf_counter(); st.h_out.copy_(st.d_out, non_blocking=True); torch.cuda.current_stream(dev).synchronize(); t("d2h + sync", t0)
    t0 = time.perf_counter()
    pre, post, pools, records = st.host_views()
    records = records.copy().view(codec.RECORD_DTYPE).ravel(); pre, post, pools = pre.copy(), post.copy(), pools.copy(); t("numpy views/copies", t0)
for k, v in T.items():
    print(f"{k:24s} {v / 10:.3f} ms")
print("ms_total (GPU events)", res.stats["ms_total"])

# inside encode_device: Python parts vs the library call
import ctypes
from paper_1206_4880_b200 import _lib
lib = _lib.load()
T2 = {}
def t2(name, t0):
    T2[name] = T2.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
out = st.result()
for _ in range(10):
    t0 = time.perf_counter(); prm = codec.make_params(c.strategy, 8, 16, 1, True, "original", c.delta, "auto", (0, 1)); t2("make_params", t0)
    t0 = time.perf_counter(); s_ = _lib.FicStats(); strm = torch.cuda.current_stream(dev).cuda_stream; t2("stats+stream", t0)
    t0 = time.perf_counter()
    rc = lib.fic_encode_v1(ctypes.c_void_p(st.d_img.data_ptr()), h, w, ctypes.byref(prm),
                           ctypes.c_void_p(out.records.data_ptr()), ctypes.c_void_p(out.pre_rms.data_ptr()),
                           ctypes.c_void_p(out.post_rms.data_ptr()), ctypes.c_void_p(out.pool_sizes.data_ptr()),
                           ctypes.byref(s_), ctypes.c_void_p(strm))
    t2("library call", t0)
    t0 = time.perf_counter(); d = s_.as_dict(); t2("as_dict", t0)
for k, v in T2.items():
    print(f"{k:24s} {v / 10:.3f} ms")
print("ms_total", d["ms_total"])
