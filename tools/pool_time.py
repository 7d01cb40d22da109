"""K1 device time alone (FIC_POOL_SERIAL: the pool builder on the main
stream, nothing beside it): median of 5 encodes' ms_pool_main (k_pool) and
ms_pool (whole K1), and the SURVEY 8(d) roofline fraction of each.
    python tools/pool_time.py cfg3 cfg5"""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
os.environ["FIC_POOL_SERIAL"] = "1"
from paper_1206_4880_b200 import codec, synth  # noqa: E402

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6552.3
import bench  # noqa: E402
wpeak = bench._write_stream_gbs()
for name in sys.argv[1:] or ["cfg3"]:
    c = synth.CONFIGS[name]
    img = torch.from_numpy(c.make()).cuda()
    kw = dict(range_size=c.range_size, domain_size=c.domain_size, stride=c.stride, isometries=True,
              delta=c.delta)
    codec.encode_device(img, c.strategy, **kw)
    st = [codec.encode_device(img, c.strategy, **kw).stats for _ in range(5)]
    mm = sorted(s["ms_pool_main"] for s in st)[2]
    m1 = sorted(s["ms_pool"] for s in st)[2]
    D = int(st[0]["n_domains"])
    K = c.range_size ** 2
    nbytes = img.numel() + D * (2 * K + 16)
    print(json.dumps({"config": name, "bytes": nbytes, "k_pool_ms": mm, "k1_ms": m1,
                      "k_pool_frac": nbytes / (mm * 1e-3) / 1e9 / peak,
                      "k1_frac": nbytes / (m1 * 1e-3) / 1e9 / peak,
                      "write_stream_gbs": wpeak,
                      "k_pool_frac_of_write_stream": D * (2 * K + 16) / (mm * 1e-3) / 1e9 / wpeak}),
          flush=True)
