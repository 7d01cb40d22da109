import sys, os
import numpy as np
sys.path.insert(0, ".")
from oracle import fic_oracle as orc
from paper_1206_4880_b200 import codec
img = np.random.default_rng(42).integers(0, 256, (96, 96), dtype=np.uint8)
ref = orc.encode(img, "exhaustive", stride=2, isometries=False)
code, st = codec.encode(img, "exhaustive", stride=2, isometries=False)
bad = np.flatnonzero(code.records != ref.records)
print("debug", os.environ.get("FIC_TC_DEBUG"), "bad", len(bad), bad[:20], "evals", st.device["exact_evals"])
for i in bad[:5]:
    print(i, code.records[i], ref.records[i], st.post_rms[i], ref.post_rms[i])
