cat > /tmp/pt.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch
from paper_1206_4880_b200 import codec, synth
c = synth.CONFIGS["cfg3"]
img = torch.from_numpy(c.make()).cuda()
t = []
for i in range(4):
    res = codec.encode_device(img, c.strategy, range_size=c.range_size, domain_size=c.domain_size, stride=c.stride, isometries=True, delta=c.delta)
    torch.cuda.synchronize()
    t.append(res.stats["ms_tensor"])
print("ms_tensor", ["%.3f" % x for x in t], "evals", res.stats["exact_evals"], "items", res.stats["work_items"])
PY
FIC_TC_CG=2 timeout 120 python tools/gpu_check.py 2>&1 | tail -3
for v in 1 2; do echo -n "CG=$v "; FIC_TC_CG=$v timeout 60 python /tmp/pt.py 2>&1 | tail -1; done
