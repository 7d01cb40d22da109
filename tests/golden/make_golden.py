"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container only (it imports ``fic`` from /root/reference,
which does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Outputs ``tests/golden/*.npz``.  Nothing here is product code.

Two sources of truth are used:
* ``fic.codec.encode`` for every case the reference supports directly;
* for the BASELINE configs' fixed FD window half-width ``delta`` (a
  parameter the reference lacks) a harness that reproduces
  ``codec.encode``'s setup (codec.py:324-376) with ``delta`` substituted for
  D_f and then calls the reference's own ``codec._search_chunk``.  With
  ``delta=None`` the harness is checked here to equal ``codec.encode``.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

from fic import bench as rbench  # noqa: E402
from fic import blocks as rbl  # noqa: E402
from fic import codec as rcodec  # noqa: E402
from fic import fdim as rfdim  # noqa: E402
from fic.avltree import AvlTree  # noqa: E402
from fic.image import fidelity  # noqa: E402

from paper_1206_4880_b200 import synth  # noqa: E402


def sha(img: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(img).tobytes()).hexdigest()


def harness_setup(image, strategy, *, range_size=8, domain_size=16, stride=1,
                  isometries=False, fd_source="original", delta=None):
    """codec.encode's setup (codec.py:324-376) with ``delta`` in place of D_f.

    Returns (ctx, r_matrix, extra): the reference's own ``_SearchContext``
    with its slabs set, the range matrix, and the FD arrays / K1 inputs."""
    image = np.asarray(image)
    r_stack = rbl.range_stack(image, range_size)
    n_ranges = r_stack.shape[0]
    r_matrix = r_stack.reshape(n_ranges, -1).astype(np.float64)
    d_stack = rbl.domain_stack(image, domain_size, stride)
    n_domains = d_stack.shape[0]
    d_down = rbl.downsample2(d_stack)
    d_matrix = d_down.reshape(n_domains, -1).astype(np.float64)
    perms = rbl.isometry_permutations(range_size)
    inv_perms = [np.argsort(perms[i]) for i in range(rbl.ISOMETRY_COUNT)]
    iso_list = list(range(rbl.ISOMETRY_COUNT)) if isometries else [0]
    ctx = rcodec._SearchContext(d_matrix, iso_list, inv_perms)
    extra = {"d_down": d_down}
    if strategy == "exhaustive":
        ctx.slab_lo = np.zeros(n_ranges, dtype=np.int64)
        ctx.slab_hi = np.full(n_ranges, n_domains, dtype=np.int64)
    elif strategy == "nosearch":
        cand = rcodec._nosearch_candidates(image.shape, range_size, domain_size, stride)
        ctx.slab_lo = cand
        ctx.slab_hi = cand + 1
    else:
        fd_blocks = d_stack if fd_source == "original" else d_down
        fd_dom = rfdim.dbc_grid(fd_blocks)
        fd_rng = rfdim.dbc_grid(r_stack)
        keys, ids = AvlTree.from_keys(fd_dom).as_sorted_arrays()
        stats = rfdim.fd_stats(fd_dom)
        ctx.use_order(ids)
        ctx.slab_lo = np.empty(n_ranges, dtype=np.int64)
        ctx.slab_hi = np.empty(n_ranges, dtype=np.int64)
        if strategy == "static2":
            mid = (stats.f_min + stats.f_max) / 2.0
            b = int(np.searchsorted(keys, mid, "left"))
            below = fd_rng < mid
            ctx.slab_lo[:] = np.where(below, 0, b)
            ctx.slab_hi[:] = np.where(below, b, n_domains)
        else:
            half = stats.d_f if delta is None else float(delta)
            ctx.slab_lo[:] = np.searchsorted(keys, fd_rng - half, "left")
            ctx.slab_hi[:] = np.searchsorted(keys, fd_rng + half, "right")
        empty = np.flatnonzero(ctx.slab_hi <= ctx.slab_lo)
        if len(empty):
            pos = rcodec._nearest_fd_positions(keys, ids, fd_rng[empty])
            ctx.slab_lo[empty] = pos
            ctx.slab_hi[empty] = pos + 1
        extra.update(fd_dom=fd_dom, fd_rng=fd_rng, keys=keys, ids=ids)
    del d_stack
    return ctx, r_matrix, extra


def harness_run(ctx, r_matrix, range_ids):
    """The reference's own matcher ``codec._search_chunk`` on ``range_ids``."""
    n_ranges = r_matrix.shape[0]
    out = {k: np.zeros(n_ranges, dtype=np.int64) for k in ("domain", "isometry", "s_q", "o_q")}
    out["pre_rms"] = np.zeros(n_ranges)
    out["post_rms"] = np.zeros(n_ranges)
    rcodec._search_chunk(ctx, r_matrix, np.asarray(range_ids), out)
    return out


def harness_result(ctx, r_matrix, extra, out):
    n_ranges = r_matrix.shape[0]
    pools = (ctx.slab_hi - ctx.slab_lo).astype(np.int64)
    rec = np.zeros(n_ranges, dtype=rcodec.RECORD_DTYPE)
    for k in ("domain", "isometry", "s_q", "o_q"):
        rec[k] = out[k]
    extra = {k: v for k, v in extra.items() if k != "d_down"}
    return dict(records=rec, pre_rms=out["pre_rms"], post_rms=out["post_rms"],
                pool_sizes=pools, slab_lo=ctx.slab_lo.astype(np.int64),
                slab_hi=ctx.slab_hi.astype(np.int64),
                comparisons=int(pools.sum()) * len(ctx.iso_list), **extra)


def harness_encode(image, strategy, *, range_size=8, domain_size=16, stride=1,
                   isometries=False, fd_source="original", delta=None,
                   range_ids=None):
    """codec.encode setup with ``delta`` in place of D_f; reference matcher."""
    ctx, r_matrix, extra = harness_setup(image, strategy, range_size=range_size,
                                         domain_size=domain_size, stride=stride,
                                         isometries=isometries, fd_source=fd_source,
                                         delta=delta)
    if range_ids is None:
        range_ids = np.arange(r_matrix.shape[0])
    out = harness_run(ctx, r_matrix, range_ids)
    return harness_result(ctx, r_matrix, extra, out)


def rand(shape, seed):
    return np.random.default_rng(seed).integers(0, 256, shape, dtype=np.uint8)


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def encode_cases():
    """Small full-image cases through the reference's own ``codec.encode``."""
    syn64 = rbench.synthetic_corpus(size=64, seed=7)
    blocky = np.kron(np.random.default_rng(8).integers(0, 256, (8, 8)), np.ones((8, 8)))
    blocky = np.clip(blocky + np.random.default_rng(9).normal(0, 3, blocky.shape),
                     0, 255).astype(np.uint8)
    cases = [
        ("rand64_ex_s4", rand((64, 64), 1), "exhaustive", 4, False),
        ("rand64_ex_s4_iso", rand((64, 64), 1), "exhaustive", 4, True),
        ("rand64_ns_s4_iso", rand((64, 64), 2), "nosearch", 4, True),
        ("rand96_st2_s4_iso", rand((96, 96), 4), "static2", 4, True),
        ("rand96_dyn_s4", rand((96, 96), 5), "dynamic_fd", 4, False),
        ("rand96_dyn_s4_iso", rand((96, 96), 5), "dynamic_fd", 4, True),
        ("rand24_ex_s2", rand((24, 24), 3), "exhaustive", 2, False),
        ("rect48x80_dyn_s3_iso", rand((48, 80), 11), "dynamic_fd", 3, True),
        ("quad64_dyn_s2_iso", syn64["quadnoise"], "dynamic_fd", 2, True),
        ("collage64_dyn_s2_iso", syn64["collage"], "dynamic_fd", 2, True),
        ("plasma64_dyn_s1_iso", syn64["plasma"], "dynamic_fd", 1, True),
        ("plasma64_st2_s2_iso", syn64["plasma"], "static2", 2, True),
        ("blocky64_ex_s2_iso", blocky, "exhaustive", 2, True),
        ("flat32_dyn_s4", np.full((32, 32), 128, np.uint8), "dynamic_fd", 4, True),
        ("flat32_ex_s4", np.full((32, 32), 128, np.uint8), "exhaustive", 4, True),
        ("flat32_ns_s4", np.full((32, 32), 128, np.uint8), "nosearch", 4, False),
        ("zero32_dyn_s2_iso", np.zeros((32, 32), np.uint8), "dynamic_fd", 2, True),
    ]
    out = {}
    for name, img, strat, stride, iso in cases:
        code, st = rcodec.encode(img, strat, stride=stride, isometries=iso)
        h = harness_encode(img, strat, stride=stride, isometries=iso)
        assert np.array_equal(h["records"], code.records), name
        assert np.array_equal(h["post_rms"], st.post_rms), name
        assert np.array_equal(h["pre_rms"], st.pre_rms), name
        assert h["comparisons"] == st.comparisons, name
        out[f"{name}.image"] = img
        out[f"{name}.params"] = np.array([stride, int(iso), rcodec.STRATEGY_IDS[strat], 8, 16])
        out[f"{name}.records"] = code.records.view(np.uint8).reshape(-1, 7)
        out[f"{name}.pre_rms"] = st.pre_rms
        out[f"{name}.post_rms"] = st.post_rms
        out[f"{name}.pool_sizes"] = st.pool_sizes
        out[f"{name}.stats"] = np.array([st.comparisons, st.mean_pool_size])
        if strat in ("dynamic_fd", "static2"):
            out[f"{name}.fd_dom"] = h["fd_dom"]
            out[f"{name}.fd_rng"] = h["fd_rng"]
            out[f"{name}.ids"] = h["ids"]
            out[f"{name}.slab_lo"] = h["slab_lo"]
            out[f"{name}.slab_hi"] = h["slab_hi"]
        # serialize + decode through the reference
        blob = rcodec.serialize(code)
        out[f"{name}.fic1"] = np.frombuffer(blob, np.uint8)
        recon = rcodec.decode(code, iterations=10)
        out[f"{name}.decoded"] = recon
        out[f"{name}.psnr"] = np.array([fidelity(img, recon).psnr])
    # fd_source="downsampled" (codec.py:320-321,352), one case
    img = rand((64, 64), 21)
    code, st = rcodec.encode(img, "dynamic_fd", stride=2, isometries=True,
                             fd_source="downsampled")
    out["down64_dyn_s2_iso.image"] = img
    out["down64_dyn_s2_iso.records"] = code.records.view(np.uint8).reshape(-1, 7)
    out["down64_dyn_s2_iso.pre_rms"] = st.pre_rms
    out["down64_dyn_s2_iso.post_rms"] = st.post_rms
    out["down64_dyn_s2_iso.pool_sizes"] = st.pool_sizes
    save("encode_cases.npz", **out)


def delta_cases():
    """BASELINE configs through the fixed-delta harness (full or range subset)."""
    out = {}
    rng = np.random.default_rng(123)
    plans = [
        # name, cfg, delta, subset size (None = all ranges)
        ("cfg1", "cfg1", 0.1, None),
        ("cfg1_dnone", "cfg1", None, None),
        ("cfg1_d001", "cfg1", 0.01, None),     # many empty windows -> fallback
        ("cfg2", "cfg2", 0.1, 96),
        ("cfg2_ex", "cfg2", None, 24),         # exhaustive run of the same image
        ("cfg3", "cfg3", 0.05, 6),
        ("cfg4_ex", "cfg4", None, 24),
    ]
    for name, cname, delta, subset in plans:
        cfg = synth.CONFIGS[cname]
        img = cfg.make()
        strat = "exhaustive" if name.endswith("_ex") else "dynamic_fd"
        n_r = (img.shape[0] // cfg.range_size) * (img.shape[1] // cfg.range_size)
        ids = None if subset is None else np.sort(rng.choice(n_r, subset, replace=False))
        t0 = time.perf_counter()
        h = harness_encode(img, strat, range_size=cfg.range_size,
                           domain_size=cfg.domain_size, stride=cfg.stride,
                           isometries=True, delta=delta, range_ids=ids)
        print(f"{name}: {time.perf_counter() - t0:.1f}s")
        if name == "cfg1_dnone":
            code, st = rcodec.encode(img, "dynamic_fd", stride=cfg.stride, isometries=True)
            assert np.array_equal(code.records, h["records"])
            assert np.array_equal(st.pre_rms, h["pre_rms"])
        sel = np.arange(n_r) if ids is None else ids
        out[f"{name}.sha"] = np.array(sha(img))
        out[f"{name}.params"] = np.array([cfg.stride, 1, rcodec.STRATEGY_IDS[strat],
                                          cfg.range_size, cfg.domain_size])
        out[f"{name}.delta"] = np.array([np.nan if delta is None else delta])
        out[f"{name}.range_ids"] = sel
        out[f"{name}.records"] = h["records"][sel].view(np.uint8).reshape(-1, 7)
        out[f"{name}.pre_rms"] = h["pre_rms"][sel]
        out[f"{name}.post_rms"] = h["post_rms"][sel]
        out[f"{name}.pool_sizes"] = h["pool_sizes"]
        out[f"{name}.comparisons"] = np.array([h["comparisons"]])
        if "fd_dom" in h:
            out[f"{name}.fd_rng"] = h["fd_rng"]
            # domain FDs are large at cfg3; keep a checksum + a sample
            fd = h["fd_dom"]
            out[f"{name}.fd_dom_sum"] = np.array([fd.sum(), fd.min(), fd.max()])
            pick = np.random.default_rng(5).choice(len(fd), min(len(fd), 4096), replace=False)
            out[f"{name}.fd_dom_pick"] = pick
            out[f"{name}.fd_dom_vals"] = fd[pick]
            out[f"{name}.ids_sha"] = np.array(sha(h["ids"]))
            out[f"{name}.slab_lo"] = h["slab_lo"]
            out[f"{name}.slab_hi"] = h["slab_hi"]
        if ids is None:
            out[f"{name}.image"] = img
    save("delta_cases.npz", **out)


def fd_cases():
    """dbc_grid known answers and random stacks (fdim.py:44-80)."""
    out = {}
    for side in (8, 16, 32):
        st = rand((60, side, side), side)
        out[f"rand{side}.blocks"] = st
        out[f"rand{side}.fd"] = rfdim.dbc_grid(st)
        out[f"rand{side}.raw"] = rfdim.dbc_grid(st, clamp=False)
    const = np.stack([np.full((16, 16), v, np.uint8) for v in (0, 128, 255)])
    out["const16.blocks"] = const
    out["const16.fd"] = rfdim.dbc_grid(const)
    const8 = np.stack([np.full((8, 8), v, np.uint8) for v in (0, 77, 255)])
    out["const8.blocks"] = const8
    out["const8.fd"] = rfdim.dbc_grid(const8)
    checker = ((np.indices((8, 8)).sum(axis=0) % 2) * 255).astype(np.uint8)[None]
    out["checker8.blocks"] = checker
    out["checker8.fd"] = rfdim.dbc_grid(checker)
    spike = np.zeros((1, 8, 8), np.uint8)
    spike[0, 0, 0] = 255
    out["spike8.blocks"] = spike
    out["spike8.raw"] = rfdim.dbc_grid(spike, clamp=False)
    out["spike8.fd"] = rfdim.dbc_grid(spike)
    for side in (4, 8, 12, 16, 32, 64):
        out[f"scales{side}"] = np.array(rfdim.scale_set(side), dtype=np.int64)
    for side in (8, 16, 32):
        xs = np.log([side / s for s in rfdim.scale_set(side)])
        out[f"weights{side}"] = rfdim._slope_weights(xs)
    perms = rbl.isometry_permutations(8)
    out["perms8"] = perms
    out["perms4"] = rbl.isometry_permutations(4)
    save("fd_cases.npz", **out)


def bench_cases():
    """The reference's benchmark run path (bench.py:216-269): RunRecord rows of
    run_single for every strategy on its own synthetic corpus (timing columns
    blanked), plus the CSV header."""
    import json
    corpus = rbench.synthetic_corpus(size=64, seed=7)
    rows = []
    for name, img in corpus.items():
        for strat in rcodec.STRATEGIES:
            rec, _code, _recon = rbench.run_single(name, img, strat, stride=4, isometries=True)
            row = rec.to_row()
            for col in rbench.TIMING_COLUMNS:
                row[rbench.CSV_COLUMNS.index(col)] = ""
            rows.append({"name": name, "strategy": strat, "row": row})
    out = {"columns": rbench.CSV_COLUMNS, "timing_columns": list(rbench.TIMING_COLUMNS),
           "images": {k: v.tolist() for k, v in corpus.items()}, "runs": rows}
    path = os.path.join(HERE, "bench_cases.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def odd_cases():
    """Range sizes other than 4 and 8 (odd and non-power-of-two sides) through
    the reference's own encode / decode, and dbc_grid on side-12/24 stacks
    (fdim.py:26-34,73-76: h = s*256/M is not an integer there)."""
    out = {}
    cases = [
        ("rand60_ex_r5_s3_iso", rand((60, 60), 61), "exhaustive", 5, 3, True),
        ("rand60_ns_r5_s2_iso", rand((60, 60), 62), "nosearch", 5, 2, True),
        ("rand48_ex_r6_s4_iso", rand((48, 48), 63), "exhaustive", 6, 4, True),
        ("rand36_ex_r3_s1", rand((36, 36), 64), "exhaustive", 3, 1, False),
        ("rand72_dyn_r12_s4_iso", rand((72, 72), 65), "dynamic_fd", 12, 4, True),
        ("rand96_st2_r12_s6_iso", rand((96, 96), 66), "static2", 12, 6, True),
        ("rand40_ex_r2_s1_iso", rand((40, 40), 67), "exhaustive", 2, 1, True),
    ]
    for name, img, strat, rs, stride, iso in cases:
        code, st = rcodec.encode(img, strat, range_size=rs, domain_size=2 * rs, stride=stride,
                                 isometries=iso)
        out[f"{name}.image"] = img
        out[f"{name}.params"] = np.array([stride, int(iso), rcodec.STRATEGY_IDS[strat], rs, 2 * rs])
        out[f"{name}.records"] = code.records.view(np.uint8).reshape(-1, 7)
        out[f"{name}.pre_rms"] = st.pre_rms
        out[f"{name}.post_rms"] = st.post_rms
        out[f"{name}.pool_sizes"] = st.pool_sizes
        out[f"{name}.stats"] = np.array([st.comparisons, st.mean_pool_size])
        out[f"{name}.decoded"] = rcodec.decode(code, iterations=10)
        if strat in ("dynamic_fd", "static2"):
            h = harness_encode(img, strat, range_size=rs, domain_size=2 * rs, stride=stride,
                               isometries=iso)
            assert np.array_equal(h["records"], code.records), name
            out[f"{name}.fd_dom"] = h["fd_dom"]
            out[f"{name}.fd_rng"] = h["fd_rng"]
            out[f"{name}.slab_lo"] = h["slab_lo"]
            out[f"{name}.slab_hi"] = h["slab_hi"]
    for side in (12, 24, 20, 48):
        stk = rand((50, side, side), 100 + side)
        stk[0] = 0
        stk[1] = 255
        out[f"dbc{side}.blocks"] = stk
        out[f"dbc{side}.fd"] = rfdim.dbc_grid(stk)
        out[f"dbc{side}.raw"] = rfdim.dbc_grid(stk, clamp=False)
    save("odd_cases.npz", **out)


def decode_cases():
    """decode_iterates snapshots, float initial images and isometry bytes > 7
    through the reference's own decoder (codec.py:516-598), plus the scalar
    fit / quantiser API (codec.py:90-130)."""
    out = {}
    rng = np.random.default_rng(31)
    for name, img, strat, stride in (("rand64_dyn_s2", rand((64, 64), 41), "dynamic_fd", 2),
                                     ("rand48x80_ex_s4", rand((48, 80), 42), "exhaustive", 4)):
        code, _ = rcodec.encode(img, strat, stride=stride, isometries=True)
        out[f"{name}.image"] = img
        out[f"{name}.params"] = np.array([stride, 1, rcodec.STRATEGY_IDS[strat], 8, 16])
        out[f"{name}.records"] = code.records.view(np.uint8).reshape(-1, 7)
        out[f"{name}.iterates"] = np.stack(list(rcodec.decode_iterates(code, 6)))
        init = rng.uniform(-20.0, 280.0, img.shape)      # float, out of byte range
        out[f"{name}.init_float"] = init
        out[f"{name}.decoded_float_init"] = rcodec.decode(code, 4, initial=init)
        out[f"{name}.decoded_level"] = rcodec.decode(code, 3, initial=37.25)
        bad = code.records.copy()
        sel = rng.choice(len(bad), len(bad) // 3, replace=False)
        bad["isometry"][sel] = rng.integers(8, 256, len(sel))
        code_bad = rcodec.FractalCode(code.width, code.height, 8, 16, stride, code.strategy_id,
                                      True, bad)
        out[f"{name}.records_iso_gt7"] = bad.view(np.uint8).reshape(-1, 7)
        out[f"{name}.decoded_iso_gt7"] = rcodec.decode(code_bad, 5)
    # fit_transform on random pairs of several lengths, incl. clamps and flat domains
    fits_in, fits_out = [], []
    for n in (1, 4, 16, 64):
        for k in range(40):
            r = rng.integers(0, 256, n).astype(np.float64)
            d = rng.integers(0, 256, n).astype(np.float64)
            if k % 10 == 0:
                d[:] = d[0]
            if k % 10 == 1:
                r = 3.0 * d - 100.0
            row = np.full((2, 64), np.nan)
            row[0, :n], row[1, :n] = r, d
            fits_in.append(row)
            fits_out.append(rcodec.fit_transform(r, d))
    out["fit.inputs"] = np.stack(fits_in)
    out["fit.outputs"] = np.array(fits_out)
    so = np.column_stack([rng.uniform(-1.0, 1.0, 500), rng.uniform(-255.0, 255.0, 500)])
    so[:4] = [[-1.0, -255.0], [1.0, 255.0], [0.0, 0.0], [1.0 / 31.0, 255.0 / 127.0]]
    out["quant.inputs"] = so
    out["quant.outputs"] = np.array([rcodec.quantize_so(a, b) for a, b in so])
    grid = np.array([(a, b) for a in range(32) for b in range(128)])
    out["dequant.inputs"] = grid
    out["dequant.outputs"] = np.array([rcodec.dequantize_so(int(a), int(b)) for a, b in grid])
    save("decode_cases.npz", **out)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for fn in sys.argv[1:]:
            globals()[fn]()
    else:
        fd_cases()
        encode_cases()
        delta_cases()
        bench_cases()
        decode_cases()
        odd_cases()
