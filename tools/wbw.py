"""HBM write / copy bandwidth probe: torch fill_ and copy_ of n bytes (CUDA events, best of 10)."""
import sys, torch
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else int(2.4e9)
a = torch.empty(n, dtype=torch.uint8, device="cuda"); b = torch.empty_like(a)
for name, fn, nb in (("fill", lambda: a.fill_(1), n), ("copy", lambda: b.copy_(a), 2 * n)):
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(name, "%.0f GB/s" % (nb / best / 1e6))
