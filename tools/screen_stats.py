"""Design probe: survivor rate of the tensor-core lower-bound screen.

Simulates the matcher's epilogue on CPU: B = fp16(centered, unit-normalised
decimated domain), A = permuted range minus round(mean) (exact in fp16),
u = A.B in fp32; a candidate survives when |u| >= sqrt(V - thr - eta) - eps,
with thr the running best exact post-quantisation error of the range (shared
by its 8 isometries), updated after every 32-column chunk.
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import fic_oracle as orc  # noqa: E402
from paper_1206_4880_b200 import synth  # noqa: E402


def run(cfg_name, n_sample=64, seed=0, chunk=32):
    cfg = synth.CONFIGS[cfg_name]
    img = cfg.make()
    rs, ds = cfg.range_size, cfg.domain_size
    r_blk = orc.range_blocks(img, rs)
    d_blk = orc.domain_blocks(img, ds, cfg.stride)
    d_dec = orc.decimate(d_blk)
    strat = cfg.strategy
    plan = orc.plan_pools(img, strat, rs, ds, cfg.stride, "original", cfg.delta,
                          r_blk, d_blk, d_dec)
    d = d_dec.reshape(len(d_dec), -1).astype(np.float64)[plan.order]
    sd, sdd, inv = orc.domain_sums(d)
    cen = d - sd[:, None] / 64.0
    nrm = np.sqrt((cen * cen).sum(1))
    B = np.where(nrm[:, None] > 0, cen / np.where(nrm > 0, nrm, 1)[:, None], 0).astype(np.float16)
    perms = orc.iso_perms(rs)
    invp = np.stack([np.argsort(p) for p in perms])
    rng = np.random.default_rng(seed)
    sample = rng.choice(len(r_blk), n_sample, replace=False)
    tot = surv = 0
    lowv = 0
    per_range = []
    for r in sample:
        row = r_blk[r].reshape(-1).astype(np.float64)
        sr, srr = row.sum(), row @ row
        V = srr - sr * sr / 64.0
        rho = np.rint(sr / 64.0)
        lo, hi = int(plan.lo[r]), int(plan.hi[r])
        rv = row[invp]                                       # (8, 64)
        A = (rv - rho).astype(np.float16).astype(np.float32)
        u = A @ B[lo:hi].astype(np.float32).T                # (8, m)
        cross = rv @ d[lo:hi].T
        n = 64.0
        s = cross * n - sd[lo:hi] * sr
        s *= inv[lo:hi]
        s = np.clip(s, -1, 1)
        o = (sr - s * sd[lo:hi]) / n
        o = np.clip(o, -255, 255)
        sq = np.rint((s + 1) * orc.S_MUL)
        oq = np.rint((o + 255) * orc.O_MUL)
        sh, oh = sq * orc.S_DEQ - 1, oq * orc.O_DEQ - 255
        err = orc._sq_err(sh, oh, sd[lo:hi], sdd[lo:hi], cross, sr, srr, n)
        eps = (2.0 ** -11 + 2.0 ** -12) * np.sqrt(V + 16.0) + 2e-3
        thr = np.inf
        m = hi - lo
        cnt = 0
        for c0 in range(0, m, chunk):
            c1 = min(m, c0 + chunk)
            c = V - thr - 1e-3
            sr_ = -1.0 if not np.isfinite(c) or c <= 0 else np.sqrt(c) * (1 - 1e-6) - eps
            mask = np.abs(u[:, c0:c1]) >= sr_
            cnt += int(mask.sum())
            if mask.any():
                thr = min(thr, float(err[:, c0:c1][mask].min()))
        tot += 8 * m
        surv += cnt
        per_range.append(cnt / (8 * m))
        if V < 2000:
            lowv += 1
    pr = np.array(per_range)
    print(f"{cfg_name}: sample {n_sample} ranges, candidates {tot}, survivors {surv} "
          f"({100 * surv / tot:.4f}%), ranges with V<2000: {lowv}, "
          f"per-range survivor frac p50 {np.median(pr):.4%} p90 {np.quantile(pr, .9):.4%} "
          f"max {pr.max():.4%}")


if __name__ == "__main__":
    for name in sys.argv[1:] or ["cfg1", "cfg2"]:
        t = time.time()
        run(name)
        print(f"  {time.time() - t:.1f}s")
