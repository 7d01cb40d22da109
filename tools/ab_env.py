"""A/B device timing of env variants on one config:
    python tools/ab_env.py cfg4 "" "FIC_SL_ALL=1" "FIC_NO_SL=1"
Each variant runs in its own process (the library reads env per call, but
a fresh process keeps the variants independent); prints median ms."""
import json
import os
import subprocess
import sys

name, variants = sys.argv[1], sys.argv[2:] or [""]
code = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth
c = synth.CONFIGS[sys.argv[1]]
img = torch.from_numpy(c.make()).cuda()
kw = dict(range_size=c.range_size, domain_size=c.domain_size, stride=c.stride, isometries=True, delta=c.delta)
codec.encode_device(img, c.strategy, **kw)
st = [codec.encode_device(img, c.strategy, **kw).stats for _ in range(int(sys.argv[2]))]
ms = sorted(s["ms_total"] for s in st)
s = st[-1]
print(json.dumps({"ms": ms[len(ms) // 2], "ms_tensor": s["ms_tensor"], "ms_sl": s["ms_sl"],
                  "exact_evals": s["exact_evals"], "sl_entries": s["sl_entries"]}))
'''
for v in variants:
    env = dict(os.environ)
    for kv in v.split():
        k, val = kv.split("=", 1)
        env[k] = val
    reps = "3" if name != "cfg5" else "1"
    out = subprocess.run([sys.executable, "-c", code, name, reps], env=env, capture_output=True,
                         text=True)
    line = [l for l in out.stdout.splitlines() if l.startswith("{")]
    print(name, repr(v), line[-1] if line else out.stderr[-800:], flush=True)
