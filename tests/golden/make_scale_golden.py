"""At-scale golden fixtures from the REFERENCE itself (build container only).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_scale_golden.py [cfg2 cfg3 cfg4 cfg5 k1]

Every record here comes from the reference package's own matcher
``fic.codec._search_chunk`` (codec.py:184-264) run on the reference's own
setup (``_SearchContext``, ``dbc_grid``, ``AvlTree``; the harness in
make_golden.py, with the BASELINE configs' fixed ``delta`` in place of D_f).
The setup is built once per config; the ranges are then split over forked
worker processes that share it copy-on-write (``_search_chunk`` writes only
the disjoint ``out`` slots of its ranges, codec.py:386-397).

Outputs ``tests/golden/scale_<cfg>.npz``:
* cfg2: all 4,096 ranges (dynamic_fd, delta 0.1) and all 4,096 exhaustive;
* cfg3: all 16,384 ranges (dynamic_fd, delta 0.05);
* cfg4: all 65,536 ranges (exhaustive, 4x4 ranges);
* cfg5: 1,024 ranges (16 empty-window ranges, then seeded random ones)
  plus the full pool sizes and SHA-256 checksums of the slabs, range FDs and
  FD order (the reference's cfg5 setup peaks near 41 GB of host RAM);
* k1: the pool builder's inputs to the matcher (blocks.py:75-82,
  codec.py:136-145) at cfg2 and cfg3 -- SHA-256 of downsample2(domain_stack)
  and of sum_d / sum_dd / inv_den in raster order, plus 4,096 sampled rows.
Nothing here is product code; /root/reference does not exist on the GPU box.
"""

from __future__ import annotations

import hashlib
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as mg  # noqa: E402  (imports the reference package)
from paper_1206_4880_b200 import synth  # noqa: E402

_CTX = None  # (ctx, r_matrix) shared with forked workers


def _work(ids):
    ctx, r_matrix = _CTX
    out = mg.harness_run(ctx, r_matrix, ids)
    return ids, {k: v[ids] for k, v in out.items()}


def run_parallel(ctx, r_matrix, ids, workers):
    """_search_chunk over ``ids`` in forked workers (copy-on-write context)."""
    global _CTX
    _CTX = (ctx, r_matrix)
    n = r_matrix.shape[0]
    out = {k: np.zeros(n, dtype=np.int64) for k in ("domain", "isometry", "s_q", "o_q")}
    out["pre_rms"] = np.zeros(n)
    out["post_rms"] = np.zeros(n)
    # small chunks in cost order (largest pools first) balance the workers
    pools = (ctx.slab_hi - ctx.slab_lo)[ids]
    ids = np.asarray(ids)[np.argsort(-pools, kind="stable")]
    chunks = [ids[i::workers * 8] for i in range(min(len(ids), workers * 8))]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(workers) as pool:
        for k, (cid, res) in enumerate(pool.imap_unordered(_work, chunks)):
            for key, v in res.items():
                out[key][cid] = v
            if k % 8 == 7:
                print(f"  {k + 1}/{len(chunks)} chunks, {time.perf_counter() - t0:.0f}s", flush=True)
    _CTX = None
    return out


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)", flush=True)


def full_case(cname, strategy, delta, workers, prefix):
    cfg = synth.CONFIGS[cname]
    img = cfg.make()
    t0 = time.perf_counter()
    ctx, r_matrix, extra = mg.harness_setup(img, strategy, range_size=cfg.range_size,
                                            domain_size=cfg.domain_size, stride=cfg.stride,
                                            isometries=True, delta=delta)
    print(f"{prefix}: setup {time.perf_counter() - t0:.1f}s", flush=True)
    ids = np.arange(r_matrix.shape[0])
    out = run_parallel(ctx, r_matrix, ids, workers)
    h = mg.harness_result(ctx, r_matrix, extra, out)
    print(f"{prefix}: {time.perf_counter() - t0:.1f}s total", flush=True)
    res = {
        f"{prefix}.sha": np.array(mg.sha(img)),
        f"{prefix}.image": img,
        f"{prefix}.params": np.array([cfg.stride, 1, mg.rcodec.STRATEGY_IDS[strategy],
                                      cfg.range_size, cfg.domain_size]),
        f"{prefix}.delta": np.array([np.nan if delta is None else delta]),
        f"{prefix}.records": h["records"].view(np.uint8).reshape(-1, 7),
        f"{prefix}.pre_rms": h["pre_rms"],
        f"{prefix}.post_rms": h["post_rms"],
        f"{prefix}.pool_sizes": h["pool_sizes"].astype(np.int32),
        f"{prefix}.comparisons": np.array([h["comparisons"]]),
    }
    if "fd_rng" in h:
        res[f"{prefix}.slab_lo"] = h["slab_lo"].astype(np.int32)
        res[f"{prefix}.slab_hi"] = h["slab_hi"].astype(np.int32)
        res[f"{prefix}.ids_sha"] = np.array(sha(h["ids"]))
    return res


def case_cfg2(workers):
    out = full_case("cfg2", "dynamic_fd", 0.1, workers, "cfg2")
    out.update(full_case("cfg2", "exhaustive", None, workers, "cfg2_ex"))
    save("scale_cfg2.npz", **out)


def case_cfg3(workers):
    save("scale_cfg3.npz", **full_case("cfg3", "dynamic_fd", 0.05, workers, "cfg3"))


def case_cfg4(workers):
    save("scale_cfg4.npz", **full_case("cfg4", "exhaustive", None, workers, "cfg4_ex"))


def case_cfg5(workers, n_pick=1024):
    cfg = synth.CONFIGS["cfg5"]
    img = cfg.make()
    t0 = time.perf_counter()
    ctx, r_matrix, extra = mg.harness_setup(img, "dynamic_fd", range_size=8, domain_size=16,
                                            stride=cfg.stride, isometries=True, delta=cfg.delta)
    print(f"cfg5: setup {time.perf_counter() - t0:.1f}s", flush=True)
    extra.pop("d_down", None)
    keys, ids, fd_rng = extra["keys"], extra["ids"], extra["fd_rng"]
    n_r = r_matrix.shape[0]
    pools = ctx.slab_hi - ctx.slab_lo
    # empty windows fall back to one domain (codec.py:371-375): is the pool
    # 1 because the window was empty?  (a window holding exactly one domain
    # is possible but the fallback ranges are the ones the rule decides)
    lo_w = np.searchsorted(keys, fd_rng - cfg.delta, "left")
    hi_w = np.searchsorted(keys, fd_rng + cfg.delta, "right")
    empty = np.flatnonzero(hi_w <= lo_w)
    rng = np.random.default_rng(55)
    pick_e = np.sort(rng.choice(empty, min(len(empty), 16), replace=False)) if len(empty) else empty
    rest = np.setdiff1d(np.arange(n_r), pick_e)
    pick_r = np.sort(rng.choice(rest, n_pick - len(pick_e), replace=False))
    pick = np.sort(np.concatenate([pick_e, pick_r]))
    print(f"cfg5: {len(empty)} empty windows; matching {len(pick)} ranges, "
          f"{int(pools[pick].sum()) * 8} candidates", flush=True)
    out = run_parallel(ctx, r_matrix, pick, workers)
    print(f"cfg5: {time.perf_counter() - t0:.1f}s total", flush=True)
    rec = np.zeros(n_r, dtype=mg.rcodec.RECORD_DTYPE)
    for k in ("domain", "isometry", "s_q", "o_q"):
        rec[k] = out[k]
    save("scale_cfg5.npz", **{
        "cfg5.sha": np.array(mg.sha(img)),
        "cfg5.params": np.array([cfg.stride, 1, 3, 8, 16]),
        "cfg5.delta": np.array([cfg.delta]),
        "cfg5.range_ids": pick,
        "cfg5.empty_ids": empty,
        "cfg5.records": rec[pick].view(np.uint8).reshape(-1, 7),
        "cfg5.pre_rms": out["pre_rms"][pick],
        "cfg5.post_rms": out["post_rms"][pick],
        "cfg5.pool_sizes": pools.astype(np.int32),
        "cfg5.comparisons": np.array([int(pools.sum()) * 8]),
        "cfg5.slab_lo_sha": np.array(sha(ctx.slab_lo.astype(np.int64))),
        "cfg5.slab_hi_sha": np.array(sha(ctx.slab_hi.astype(np.int64))),
        "cfg5.slab_lo_pick": ctx.slab_lo[pick].astype(np.int64),
        "cfg5.slab_hi_pick": ctx.slab_hi[pick].astype(np.int64),
        "cfg5.fd_rng_sha": np.array(sha(fd_rng)),
        "cfg5.fd_rng_pick": fd_rng[pick],
        "cfg5.fd_dom_sum": np.array([extra["fd_dom"].sum(), extra["fd_dom"].min(),
                                     extra["fd_dom"].max()]),
        "cfg5.ids_sha": np.array(sha(ids)),
    })


def case_k1(workers):
    """K1 inputs of the matcher: decimated domains and _SearchContext sums."""
    out = {}
    for cname in ("cfg2", "cfg3"):
        cfg = synth.CONFIGS[cname]
        img = cfg.make()
        ctx, _r, extra = mg.harness_setup(img, "exhaustive", range_size=8, domain_size=16,
                                          stride=cfg.stride, isometries=True)
        d_down = extra["d_down"].reshape(len(ctx.sum_d), -1)
        pick = np.sort(np.random.default_rng(77).choice(len(d_down), 4096, replace=False))
        out.update({
            f"{cname}.sha": np.array(mg.sha(img)),
            f"{cname}.stride": np.array([cfg.stride]),
            f"{cname}.dec_sha": np.array(sha(d_down)),
            f"{cname}.sum_d_sha": np.array(sha(ctx.sum_d)),
            f"{cname}.sum_dd_sha": np.array(sha(ctx.sum_dd)),
            f"{cname}.inv_den_sha": np.array(sha(ctx.inv_den)),
            f"{cname}.pick": pick,
            f"{cname}.dec_pick": d_down[pick],
            f"{cname}.sum_d_pick": ctx.sum_d[pick],
            f"{cname}.sum_dd_pick": ctx.sum_dd[pick],
            f"{cname}.inv_den_pick": ctx.inv_den[pick],
        })
        print(f"k1 {cname}: done", flush=True)
    save("scale_k1.npz", **out)


if __name__ == "__main__":
    workers = int(os.environ.get("GOLDEN_WORKERS", os.cpu_count() or 1))
    todo = sys.argv[1:] or ["k1", "cfg2", "cfg3", "cfg4", "cfg5"]
    for name in todo:
        t0 = time.perf_counter()
        globals()[f"case_{name}"](workers if name != "cfg5" else min(workers, 6))
        print(f"== {name}: {time.perf_counter() - t0:.0f}s", flush=True)
