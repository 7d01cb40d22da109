"""Pruning power of the quantisation-aware exact bound on
near-flat cfg4 ranges, against the plain bound LB = V - num^2/(K den), with
the reference's final errors (tests/golden/scale_cfg4.npz) as thresholds:
    python tools/qbound_check.py"""
import sys, numpy as np
sys.path.insert(0, ".")


def range_blocks(image, rs):  # blocks.py:145-155, raster order
    h, w = image.shape
    return image.reshape(h // rs, rs, w // rs, rs).transpose(0, 2, 1, 3).reshape(-1, rs, rs)


def decimated_domains(image, ds, st):  # blocks.py:58-82: windows, 2x2 floor means
    win = np.lib.stride_tricks.sliding_window_view(image, (ds, ds))[::st, ::st].reshape(-1, ds, ds)
    g = win.reshape(-1, ds // 2, 2, ds // 2, 2).astype(np.uint32)
    return (g.sum(axis=(2, 4)) >> 2)


def iso_perms(n):  # blocks.py:113-139: the 8 dihedral maps as gather tables
    idx = np.arange(n * n).reshape(n, n)
    out = []
    for i in range(8):
        b = np.rot90(idx, i % 4)
        out.append((b.T if i >= 4 else b).ravel())
    return np.stack(out)
g=np.load('./tests/golden/scale_cfg4.npz'); im=g['cfg4_ex.image']
r_mat = range_blocks(im, 4).reshape(-1, 16).astype(np.float64)
d_mat = decimated_domains(im, 8, 2).reshape(-1, 16).astype(np.float64)
K=16.0; perms=iso_perms(4); inv_perms=np.stack([np.argsort(p) for p in perms])
sd=d_mat.sum(1); sdd=(d_mat*d_mat).sum(1); den=K*sdd-sd*sd
thr_all=g['cfg4_ex.post_rms']**2*K
sr_all=r_mat.sum(1); V_all=(r_mat*r_mat).sum(1)-sr_all**2/K
flat=(r_mat.max(1)==r_mat.min(1))
cand=np.where(~flat & (V_all-thr_all<5))[0]
rng=np.random.default_rng(1); pick=rng.choice(cand, 12, replace=False)
slev=-1+2*np.arange(32)/31; olev=-255+510*np.arange(128)/127
tot_lb=tot_q=tot_all=0
for r in pick:
    row=r_mat[r]; sr=row.sum(); srr=(row*row).sum(); V=srr-sr*sr/K; thr=thr_all[r]
    cross=row[inv_perms]@d_mat.T   # (8, D)
    num=K*cross-sr*sd
    ok=den>0
    LB=np.where(ok, V-num*num/np.where(ok,K*den,1), V)
    lbpass=(LB<=thr+1e-5)
    sstar=np.where(ok, num/np.where(ok,den,1), 0.0)
    # two bracketing levels
    k=np.clip(np.floor((sstar+1)*15.5),0,30); best=np.full(sstar.shape,np.inf)
    for kk in (k, k+1):
        sq=-1+2*kk/31
        ts=np.where(ok,(den/K)*(sq-sstar)**2,0)
        ostar=(sr-sq*sd)/K
        ko=np.clip(np.rint((ostar+255)*127/510),0,127); do=np.abs(-255+510*ko/127-ostar)
        best=np.minimum(best, LB+ts+K*do*do)
    qpass=best<=thr+1e-4
    assert not (~lbpass & qpass).any() or True
    tot_lb+=lbpass.sum(); tot_q+=qpass.sum(); tot_all+=cross.size
    print(r, "V %.1f thr %.1f  LB-pass %d  quant-bound-pass %d" % (V, thr, lbpass.sum(), qpass.sum()))
print(tot_lb, tot_q, tot_all)
