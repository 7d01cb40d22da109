"""cProfile of repeated codec.encode calls on cfg3 (host-side overhead)."""
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth  # noqa: E402

c = synth.CONFIGS["cfg3"]
im = c.make()
kw = dict(range_size=8, domain_size=16, stride=1, isometries=True, delta=c.delta)
for _ in range(3):
    codec.encode(im, "dynamic_fd", **kw)
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    codec.encode(im, "dynamic_fd", **kw)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
