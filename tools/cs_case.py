import sys, torch
sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth
img = torch.from_numpy(synth.CONFIGS["cfg2"].make()[:256, :256].copy()).cuda()
r = codec.encode_device(img, "dynamic_fd", range_size=8, domain_size=16, stride=2, isometries=True, delta=0.1)
torch.cuda.synchronize()
print("ok", r.stats["exact_evals"], r.stats["work_items"])
