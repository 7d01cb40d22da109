cat > /tmp/pt.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch
from paper_1206_4880_b200 import codec, synth
c = synth.CONFIGS["cfg3"]
img = torch.from_numpy(c.make()).cuda()
for i in range(4):
    res = codec.encode_device(img, c.strategy, range_size=c.range_size, domain_size=c.domain_size, stride=c.stride, isometries=True, delta=c.delta)
    torch.cuda.synchronize()
PY
python tools/gpu_check.py 2>&1 | tail -2
FIC_PLAN_TIMING=1 python /tmp/pt.py 2>&1 | tail -3
timeout 120 python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-250
