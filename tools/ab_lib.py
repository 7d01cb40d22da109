"""A/B of library builds on one config, alternating processes:
    python tools/ab_lib.py cfg3 ROUNDS A.so B.so ...
A directory argument is a whole package snapshot (DIR/paper_1206_4880_b200
with its own library, e.g. an older round's build), imported instead of the
in-tree package.
Each process does a warm-up encode then 5 timed ones; prints the median
device ms (ms_total, ms_tensor) per build and round."""
import json
import os
import subprocess
import sys

name, rounds, libs = sys.argv[1], int(sys.argv[2]), sys.argv[3:]
code = r'''
import os, sys, json, torch
sys.path.insert(0, os.environ.get("AB_PKG_ROOT", "."))
from paper_1206_4880_b200 import codec, synth
c = synth.CONFIGS[sys.argv[1]]
img = torch.from_numpy(c.make()).cuda()
kw = dict(range_size=c.range_size, domain_size=c.domain_size, stride=c.stride, isometries=True, delta=c.delta)
codec.encode_device(img, c.strategy, **kw)
st = [codec.encode_device(img, c.strategy, **kw).stats for _ in range(5)]
print(json.dumps({k: sorted(s[k] for s in st)[2] for k in ("ms_total", "ms_tensor")}))
print("#", codec.__file__, file=sys.stderr)
'''
res = {lib: [] for lib in libs}
for _ in range(rounds):
    for lib in libs:
        if os.path.isdir(lib):
            env = dict(os.environ, AB_PKG_ROOT=os.path.abspath(lib))
            env.pop("FIC_B200_LIB", None)
        else:
            env = dict(os.environ, FIC_B200_LIB=os.path.abspath(lib))
        out = subprocess.run([sys.executable, "-c", code, name], env=env, capture_output=True,
                             text=True)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        d = json.loads(line[-1]) if line else {"error": out.stderr[-300:]}
        res[lib].append(d)
        print(os.path.basename(lib), d, flush=True)
for lib, v in res.items():
    t = sorted(x.get("ms_tensor", 0) for x in v)
    print("median", os.path.basename(lib), t[len(t) // 2])
