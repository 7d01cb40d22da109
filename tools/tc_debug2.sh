cat > /tmp/pt2.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch
from paper_1206_4880_b200 import codec, synth
c = synth.CONFIGS["cfg3"]
img = torch.from_numpy(c.make()).cuda()
for seg in (32768, 65536, 131072, 262144):
    t = []
    for i in range(4):
        res = codec.encode_device(img, c.strategy, range_size=c.range_size, domain_size=c.domain_size, stride=c.stride, isometries=True, delta=c.delta, max_segment=seg)
        torch.cuda.synchronize()
        t.append(res.stats["ms_tensor"])
    print(seg, "ms_tensor", ["%.3f" % x for x in t], "evals", res.stats["exact_evals"], "items", res.stats["work_items"])
PY
python /tmp/pt2.py
