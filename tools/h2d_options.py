"""Time host->device options for a 1 MB uint8 image (pinned staging vs direct)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1206_4880_b200 import synth  # noqa: E402

im = synth.CONFIGS["cfg3"].make()
h_pin = torch.empty(im.shape, dtype=torch.uint8, pin_memory=True)
d = torch.empty(im.shape, dtype=torch.uint8, device="cuda")
t_im = torch.from_numpy(im)


def bench(name, f, n=50):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
        torch.cuda.synchronize()
    print(f"{name:32s} {(time.perf_counter() - t0) / n * 1e3:.3f} ms")


bench("numpy->pinned, H2D async", lambda: (h_pin.numpy().__setitem__(Ellipsis, im), d.copy_(h_pin, non_blocking=True)))
bench("torch copy_ ->pinned, H2D", lambda: (h_pin.copy_(t_im), d.copy_(h_pin, non_blocking=True)))
bench("pageable H2D (torch)", lambda: d.copy_(t_im))
bench("pageable H2D non_blocking", lambda: d.copy_(t_im, non_blocking=True))
