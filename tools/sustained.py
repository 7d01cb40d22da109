"""Back-to-back cfg3 encodes (graph replays, no gaps) against spaced ones
(an L2 flush and a synchronise between encodes, as in bench.py): device ms
per encode with the SM clock and board power sampled by NVML meanwhile.
    python tools/sustained.py [n]"""
import sys
import threading
import time

import numpy as np
import pynvml
import torch

sys.path.insert(0, ".")
from paper_1206_4880_b200 import codec, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
c = synth.CONFIGS["cfg3"]
img = torch.from_numpy(c.make()).cuda()
kw = dict(range_size=8, domain_size=16, stride=1, isometries=True, delta=0.05)
n_r = 16384
out = codec.DeviceResult(torch.empty((n_r, 7), dtype=torch.uint8, device="cuda"),
                         torch.empty(n_r, dtype=torch.float64, device="cuda"),
                         torch.empty(n_r, dtype=torch.float64, device="cuda"),
                         torch.empty(n_r, dtype=torch.int64, device="cuda"), {})
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)


class Sampler(threading.Thread):
    def __init__(self):
        super().__init__(daemon=True)
        self.stop, self.clk, self.pw = False, [], []

    def run(self):
        while not self.stop:
            self.clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            self.pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1e3)
            time.sleep(0.005)


def run(spaced):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(4):
        codec.encode_device(img, "dynamic_fd", out=out, **kw)
    torch.cuda.synchronize()
    s = Sampler()
    s.start()
    t, tt = [], []
    for _ in range(n):
        if spaced:
            flush.zero_()
            torch.cuda.synchronize()
            time.sleep(0.02)
        st = codec.encode_device(img, "dynamic_fd", out=out, **kw).stats
        t.append(st["ms_total"])
        tt.append(st["ms_tensor"])
    torch.cuda.synchronize()
    s.stop = True
    s.join()
    t, tt = np.array(t), np.array(tt)
    print("%s: ms_total first10 %.3f last10 %.3f median %.3f | ms_tensor median %.3f | SM MHz median %.0f min %.0f | W median %.0f max %.0f"
          % ("spaced" if spaced else "back-to-back", t[:10].mean(), t[-10:].mean(), np.median(t),
             np.median(tt), np.median(s.clk), np.min(s.clk), np.median(s.pw), np.max(s.pw)), flush=True)


run(True)
run(False)
run(True)
