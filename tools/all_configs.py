"""One line per BASELINE config (plus cfg2 exhaustive and cfg1/cfg3 with the
reference's own D_f rule): device ms per encode (median of 3 after a
warm-up), matches/s, exact rescorings, tensor fraction.  Writes JSON lines
to stdout; `profiles/r01_configs.jsonl` holds the committed run."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth  # noqa: E402

RUNS = [("cfg1", None), ("cfg1", "ref_Df"), ("cfg2", None), ("cfg2", "exhaustive"), ("cfg3", None),
        ("cfg3", "ref_Df"), ("cfg4", None), ("cfg5", None)]
for name, variant in RUNS:
    c = synth.CONFIGS[name]
    img = torch.from_numpy(c.make()).cuda()
    strat, delta = c.strategy, c.delta
    if variant == "exhaustive":
        strat, delta = "exhaustive", None
    elif variant == "ref_Df":
        delta = None
    kw = dict(range_size=c.range_size, domain_size=c.domain_size, stride=c.stride, isometries=True,
              delta=delta)
    codec.encode_device(img, strat, **kw)
    torch.cuda.synchronize()
    ms, st = [], None
    for _ in range(3):
        r = codec.encode_device(img, strat, **kw)
        torch.cuda.synchronize()
        ms.append(r.stats["ms_total"])
        st = r.stats
    m = float(np.median(ms))
    print(json.dumps({"config": name, "variant": variant or "baseline", "strategy": strat,
                      "delta": delta, "image": list(img.shape), "range_size": c.range_size,
                      "domain_size": c.domain_size, "stride": c.stride,
                      "comparisons": int(st["comparisons"]), "ms": m,
                      "matches_per_s": st["comparisons"] / (m / 1e3),
                      "ms_tensor": st["ms_tensor"], "ms_fd": st["ms_fd"],
                      "exact_evals": int(st["exact_evals"]), "tensor_tiles": int(st["tensor_tiles"])}),
          flush=True)
