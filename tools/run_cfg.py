"""Encode one BASELINE config on the GPU a few times and print the device stats:
    python tools/run_cfg.py cfg4 [reps]"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
c = synth.CONFIGS[name]
t = time.time()
im = c.make()
print(name, "gen %.1fs" % (time.time() - t), im.shape, c.strategy, flush=True)
img = torch.from_numpy(im).cuda()
for i in range(reps):
    res = codec.encode_device(img, c.strategy, range_size=c.range_size, domain_size=c.domain_size,
                              stride=c.stride, isometries=True, delta=c.delta)
    torch.cuda.synchronize()
    st = res.stats
    keys = ("ms_total", "ms_fd", "ms_pool", "ms_tensor", "ms_sl", "ms_exact", "exact_evals",
            "sl_entries", "hl_entries", "hl_tests", "comparisons", "work_items")
    print({k: st[k] for k in keys}, "matches/s %.3g" % (st["comparisons"] / st["ms_total"] * 1e3),
          flush=True)
