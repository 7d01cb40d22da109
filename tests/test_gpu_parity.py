"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden outputs and the pinned oracle.  Bit-exact records, RMS and FD."""

import hashlib
import re

import numpy as np
import pytest

from conftest import cases, load_golden
from oracle import fic_oracle as orc
from paper_1206_4880_b200 import codec, synth

pytestmark = pytest.mark.gpu

ENC = load_golden("encode_cases.npz")
DELTA = load_golden("delta_cases.npz")
FD = load_golden("fd_cases.npz")
STRATS = codec.STRATEGIES
ENC_CASES = [c for c in cases(ENC) if c != "down64_dyn_s2_iso"]


def _recs(a):
    return np.ascontiguousarray(a).view(codec.RECORD_DTYPE).ravel()


def _params(g, name):
    stride, iso, sid, rs, ds = (int(v) for v in g[f"{name}.params"])
    return dict(stride=stride, isometries=bool(iso), range_size=rs, domain_size=ds), STRATS[sid]


def _cfg_image(name):
    cfg = synth.CONFIGS[name.split("_")[0]]
    img = DELTA[f"{name}.image"] if f"{name}.image" in DELTA else cfg.make()
    if hashlib.sha256(img.tobytes()).hexdigest() != str(DELTA[f"{name}.sha"]):
        pytest.skip("synthetic generator output differs on this host")
    return img


@pytest.mark.parametrize("matcher", ["auto", "exact"])
@pytest.mark.parametrize("name", ENC_CASES)
def test_encode_matches_reference_golden(name, matcher):
    kw, strat = _params(ENC, name)
    code, st = codec.encode(ENC[f"{name}.image"], strat, matcher=matcher, **kw)
    assert np.array_equal(code.records, _recs(ENC[f"{name}.records"]))
    assert np.array_equal(st.pre_rms, ENC[f"{name}.pre_rms"])
    assert np.array_equal(st.post_rms, ENC[f"{name}.post_rms"])
    assert np.array_equal(st.pool_sizes, ENC[f"{name}.pool_sizes"])
    comp, mean_pool = ENC[f"{name}.stats"]
    assert st.comparisons == int(comp) and st.mean_pool_size == mean_pool


@pytest.mark.parametrize("matcher", ["auto", "exact"])
def test_encode_small_pool_threshold_forces_tensor_path(matcher):
    # small_pool=1 routes every range with a pool >= 1 to the tensor matcher
    for name in ("rand64_ex_s4_iso", "rand96_dyn_s4_iso", "collage64_dyn_s2_iso",
                 "flat32_ex_s4", "blocky64_ex_s2_iso"):
        kw, strat = _params(ENC, name)
        img = ENC[f"{name}.image"]
        import torch
        res = codec.encode_device(torch.from_numpy(img).cuda(), strat, matcher=matcher,
                                  small_pool=1, max_segment=256, **kw)
        assert np.array_equal(_recs(res.records.cpu().numpy()), _recs(ENC[f"{name}.records"])), name
        assert np.array_equal(res.pre_rms.cpu().numpy(), ENC[f"{name}.pre_rms"]), name
        assert np.array_equal(res.post_rms.cpu().numpy(), ENC[f"{name}.post_rms"]), name


def test_encode_fd_source_downsampled():
    name = "down64_dyn_s2_iso"
    code, st = codec.encode(ENC[f"{name}.image"], "dynamic_fd", stride=2, isometries=True,
                            fd_source="downsampled")
    assert np.array_equal(code.records, _recs(ENC[f"{name}.records"]))
    assert np.array_equal(st.post_rms, ENC[f"{name}.post_rms"])
    assert np.array_equal(st.pre_rms, ENC[f"{name}.pre_rms"])


@pytest.mark.parametrize("name", [c for c in ENC_CASES if f"{c}.fd_dom" in ENC])
def test_plan_fd_and_slabs_bit_exact(name):
    kw, strat = _params(ENC, name)
    kw.pop("isometries")
    p = codec.plan(ENC[f"{name}.image"], strat, **kw)
    assert np.array_equal(p["fd_dom"], ENC[f"{name}.fd_dom"])
    assert np.array_equal(p["fd_rng"], ENC[f"{name}.fd_rng"])
    assert np.array_equal(p["order"], ENC[f"{name}.ids"])
    assert np.array_equal(p["slab_lo"], ENC[f"{name}.slab_lo"])
    assert np.array_equal(p["slab_hi"], ENC[f"{name}.slab_hi"])


@pytest.mark.parametrize("stride", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("shape,seed", [((96, 136), 7), ((120, 80), 8), ((64, 64), 9)])
def test_plan_tiled_fd_matches_oracle(stride, shape, seed):
    """The tiled DBC kernel (16x16 domains, strides 1-4; stride 5 takes the
    per-block kernel) gives the oracle's FD bits, order and slabs on images
    whose domain grid ends inside a tile, for both strategies that use FD."""
    rng = np.random.default_rng(seed)
    img = synth.to_u8(synth.fbm(max(shape), 0.2 + 0.1 * (seed - 7), rng))[:shape[0], :shape[1]]
    img = np.ascontiguousarray(img)
    # a flat patch and a checkerboard patch (zero and maximal counts)
    img[:24, :24] = 77
    img[-20:, -20:] = np.where((np.indices((20, 20)).sum(0) % 2) == 0, 0, 255)
    for strat, delta in (("dynamic_fd", None), ("dynamic_fd", 0.05), ("static2", None)):
        p = codec.plan(img, strat, stride=stride, delta=delta)
        ref = orc.plan_pools(img, strat, 8, 16, stride, delta=delta)
        assert np.array_equal(p["fd_dom"], ref.fd_dom), (strat, delta)
        assert np.array_equal(p["fd_rng"], ref.fd_rng), (strat, delta)
        assert np.array_equal(p["order"], ref.order), (strat, delta)
        assert np.array_equal(p["slab_lo"], ref.lo), (strat, delta)
        assert np.array_equal(p["slab_hi"], ref.hi), (strat, delta)


def test_plan_tiled_fd_equals_direct_at_cfg3(monkeypatch):
    """Full-size property: the tiled DBC kernel and the per-block kernel
    (FIC_FD_DIRECT) agree bit for bit on all 1,018,081 cfg3 domains, and the
    rank-keyed sort equals the 52-bit FD sort (FIC_FD_WIDE_SORT)."""
    img = synth.CONFIGS["cfg3"].make()
    a = codec.plan(img, "dynamic_fd", stride=1, delta=0.05)
    monkeypatch.setenv("FIC_FD_DIRECT", "1")
    monkeypatch.setenv("FIC_FD_WIDE_SORT", "1")
    b = codec.plan(img, "dynamic_fd", stride=1, delta=0.05)
    for k in ("fd_dom", "fd_rng", "order", "slab_lo", "slab_hi"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("cname", ["cfg2", "cfg5"])
def test_plan_half_lattice_fd_equals_full_grid(cname, monkeypatch):
    """Full-size property at the even-stride configs: the half-lattice DBC
    kernel (k_fd16_half) and the full-grid tiled kernel agree bit for bit on
    every domain (16.7 M at cfg5), and so do the order and slabs."""
    c = synth.CONFIGS[cname]
    img = c.make()
    a = codec.plan(img, "dynamic_fd", stride=c.stride, delta=c.delta)
    monkeypatch.setenv("FIC_FD_FULLGRID", "1")
    b = codec.plan(img, "dynamic_fd", stride=c.stride, delta=c.delta)
    for k in ("fd_dom", "fd_rng", "order", "slab_lo", "slab_hi"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("delta", [1e-4, 0.02])
def test_encode_count_sorted_pools_match_oracle(delta):
    """encode() orders equal-FD domains by a counting sort (unspecified order
    inside a run of equal FDs, smallest raster index first).  With a tiny
    delta most windows are empty and take the nearest-FD fallback, which
    reads exactly that first element (codec.py:267-287)."""
    rng = np.random.default_rng(11)
    img = np.ascontiguousarray(synth.to_u8(synth.fbm(128, 0.35, rng)))
    kw = dict(range_size=8, domain_size=16, stride=2, isometries=True, delta=delta)
    code, st = codec.encode(img, "dynamic_fd", **kw)
    ref = orc.encode(img, "dynamic_fd", **kw)
    assert np.array_equal(code.records, ref.records)
    assert np.array_equal(st.post_rms, ref.post_rms) and np.array_equal(st.pre_rms, ref.pre_rms)
    assert np.array_equal(st.pool_sizes, ref.pool_sizes)


def test_encode_count_sort_equals_stable_sort_at_cfg3(monkeypatch):
    """Full size: the counting-sorted pool and range orders and the stable
    radix-sorted ones (the reference's FD order) give identical encodes, also
    with mostly empty windows."""
    import torch
    img = torch.from_numpy(synth.CONFIGS["cfg3"].make()).cuda()
    for delta in (0.05, 1e-5):
        kw = dict(range_size=8, domain_size=16, stride=1, isometries=True, delta=delta)
        a = codec.encode_device(img, "dynamic_fd", **kw)
        monkeypatch.setenv("FIC_FD_STABLE", "1")
        monkeypatch.setenv("FIC_RANGE_RADIX", "1")
        b = codec.encode_device(img, "dynamic_fd", **kw)
        monkeypatch.delenv("FIC_FD_STABLE")
        monkeypatch.delenv("FIC_RANGE_RADIX")
        assert torch.equal(a.records, b.records), delta
        assert torch.equal(a.post_rms, b.post_rms) and torch.equal(a.pre_rms, b.pre_rms), delta
        assert torch.equal(a.pool_sizes, b.pool_sizes), delta


@pytest.mark.parametrize("strategy", ["exhaustive", "dynamic_fd"])
def test_flat_ranges_path_equals_screened_path(strategy, monkeypatch):
    """Flat ranges (all pixels equal) are matched by one reduction per pixel
    value (fic_flat.cu) instead of the screen; FIC_NO_FLAT sends them through
    the screen + exact rescoring.  Same records and RMS, on the smooth
    gradient half of the cfg4 generator (many flat 4x4 and 8x8 ranges)."""
    import torch
    img = np.ascontiguousarray(synth.CONFIGS["cfg4"].make()[:256, :256])
    d = torch.from_numpy(img).cuda()
    for rs in (4, 8):
        if strategy == "dynamic_fd" and rs == 4:
            continue  # 4x4 ranges have one DBC scale (the reference raises)
        kw = dict(range_size=rs, domain_size=2 * rs, stride=2, isometries=True)
        a = codec.encode_device(d, strategy, **kw)
        monkeypatch.setenv("FIC_NO_FLAT", "1")
        b = codec.encode_device(d, strategy, **kw)
        monkeypatch.delenv("FIC_NO_FLAT")
        assert torch.equal(a.records, b.records), rs
        assert torch.equal(a.post_rms, b.post_rms) and torch.equal(a.pre_rms, b.pre_rms), rs


def test_pool_row_segments_equal_box_planes(monkeypatch):
    """The pool builder reads domains from per-column row segments when they
    fit in L2 (cfg2/cfg3) and from the box-floor planes otherwise (cfg5);
    both give the same pool, hence the same encode."""
    import torch
    img = torch.from_numpy(synth.CONFIGS["cfg2"].make()).cuda()
    kw = dict(range_size=8, domain_size=16, stride=3, isometries=True, delta=0.1)
    a = codec.encode_device(img, "dynamic_fd", **kw)
    monkeypatch.setenv("FIC_POOL_PLANES", "1")
    b = codec.encode_device(img, "dynamic_fd", **kw)
    assert torch.equal(a.records, b.records)
    assert torch.equal(a.post_rms, b.post_rms) and torch.equal(a.pre_rms, b.pre_rms)


def test_plan_counts_read_back_equals_device_plan(monkeypatch):
    """The planner's counts stay on the device (allocations use bounds);
    FIC_PLAN_SYNC reads them back first and allocates exactly -- the path a
    call with very loose bounds takes.  Same results, also for the exact
    matcher and for a shard."""
    import torch
    img = torch.from_numpy(synth.CONFIGS["cfg2"].make()).cuda()
    kw = dict(range_size=8, domain_size=16, stride=4, isometries=True, delta=0.1)
    for extra in ({}, {"matcher": "exact"}, {"shard": (1, 3)}):
        a = codec.encode_device(img, "dynamic_fd", **kw, **extra)
        monkeypatch.setenv("FIC_PLAN_SYNC", "1")
        b = codec.encode_device(img, "dynamic_fd", **kw, **extra)
        monkeypatch.delenv("FIC_PLAN_SYNC")
        assert torch.equal(a.records, b.records), extra
        assert torch.equal(a.post_rms, b.post_rms) and torch.equal(a.pre_rms, b.pre_rms), extra
        assert a.stats["work_items"] == b.stats["work_items"] > 0, extra


def test_dbc_grid_known_answers():
    for side in (8, 16, 32):
        assert np.array_equal(codec.dbc_grid(FD[f"rand{side}.blocks"]), FD[f"rand{side}.fd"])
        assert np.array_equal(codec.dbc_grid(FD[f"rand{side}.blocks"], clamp=False),
                              FD[f"rand{side}.raw"])
    assert np.all(codec.dbc_grid(FD["const16.blocks"]) == 2.0)
    assert np.array_equal(codec.dbc_grid(FD["const8.blocks"]), FD["const8.fd"])
    assert codec.dbc_grid(FD["checker8.blocks"])[0] == 3.0
    assert codec.dbc_grid(FD["spike8.blocks"], clamp=False)[0] == FD["spike8.raw"][0]
    with pytest.raises(ValueError, match="two DBC scales"):
        codec.dbc_grid(np.zeros((1, 4, 4), np.uint8))


@pytest.mark.parametrize("name", sorted({k.split(".")[0] for k in DELTA}))
def test_baseline_configs_match_reference(name):
    img = _cfg_image(name)
    stride, iso, sid, rs, ds = (int(v) for v in DELTA[f"{name}.params"])
    delta = float(DELTA[f"{name}.delta"][0])
    delta = None if np.isnan(delta) else delta
    code, st = codec.encode(img, STRATS[sid], range_size=rs, domain_size=ds, stride=stride,
                            isometries=bool(iso), delta=delta)
    ids = DELTA[f"{name}.range_ids"]
    assert np.array_equal(code.records[ids], _recs(DELTA[f"{name}.records"]))
    assert np.array_equal(st.pre_rms[ids], DELTA[f"{name}.pre_rms"])
    assert np.array_equal(st.post_rms[ids], DELTA[f"{name}.post_rms"])
    assert np.array_equal(st.pool_sizes, DELTA[f"{name}.pool_sizes"])
    assert st.comparisons == int(DELTA[f"{name}.comparisons"][0])


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_full_config_matches_oracle(cfg):
    c = synth.CONFIGS[cfg]
    img = c.make()
    ref = orc.encode(img, c.strategy, range_size=c.range_size, domain_size=c.domain_size,
                     stride=c.stride, isometries=True, delta=c.delta)
    code, st = codec.encode(img, c.strategy, range_size=c.range_size, domain_size=c.domain_size,
                            stride=c.stride, isometries=True, delta=c.delta)
    assert np.array_equal(code.records, ref.records)
    assert np.array_equal(st.pre_rms, ref.pre_rms)
    assert np.array_equal(st.post_rms, ref.post_rms)
    assert st.comparisons == ref.comparisons


def test_cfg3_tensor_path_equals_exact_path_full_size():
    """Size-independent property at the headline config: the screened
    tensor-core matcher returns exactly what exhaustive fp64 evaluation of
    every candidate returns (all 16,384 ranges)."""
    c = synth.CONFIGS["cfg3"]
    img = c.make()
    kw = dict(range_size=8, domain_size=16, stride=1, isometries=True, delta=0.05)
    a, sa = codec.encode(img, "dynamic_fd", matcher="auto", **kw)
    b, sb = codec.encode(img, "dynamic_fd", matcher="exact", **kw)
    assert a == b
    assert np.array_equal(sa.pre_rms, sb.pre_rms)
    assert np.array_equal(sa.post_rms, sb.post_rms)
    assert sa.device["tensor_tiles"] > 0
    # the screen keeps a small fraction of candidates for exact rescoring
    assert sa.device["exact_evals"] < 0.01 * sa.comparisons


def test_shards_combine_to_single_gpu_result():
    import torch
    c = synth.CONFIGS["cfg2"]
    img = torch.from_numpy(c.make()).cuda()
    kw = dict(range_size=8, domain_size=16, stride=4, isometries=True, delta=0.1)
    full = codec.encode_device(img, "dynamic_fd", **kw)
    n_r = full.records.shape[0]
    for world in (2, 3, 4):
        rec = torch.zeros((n_r, 7), dtype=torch.uint8, device="cuda")
        post = torch.full((n_r,), -1.0, dtype=torch.float64, device="cuda")
        pre = torch.full((n_r,), -1.0, dtype=torch.float64, device="cuda")
        for k in range(world):
            out = codec.DeviceResult(rec, pre, post, torch.zeros(n_r, dtype=torch.int64, device="cuda"), {})
            codec.encode_device(img, "dynamic_fd", shard=(k, world), out=out, **kw)
        assert torch.equal(rec, full.records)
        assert torch.equal(pre, full.pre_rms) and torch.equal(post, full.post_rms)


@pytest.mark.parametrize("name", ENC_CASES[:8])
def test_decode_matches_reference(name):
    kw, strat = _params(ENC, name)
    img = ENC[f"{name}.image"]
    code = codec.FractalCode(img.shape[1], img.shape[0], kw["range_size"], kw["domain_size"],
                             kw["stride"], codec.STRATEGY_IDS[strat], kw["isometries"],
                             _recs(ENC[f"{name}.records"]).copy())
    out = codec.decode(code, iterations=10)
    assert np.array_equal(out, ENC[f"{name}.decoded"])
    assert orc.psnr(img, out) == ENC[f"{name}.psnr"][0]


def test_c_abi_errors_reraise_reference_text():
    import torch
    img = torch.zeros((64, 64), dtype=torch.uint8, device="cuda")
    # bypass the Python pre-validation: the C layer must produce the same text
    p = codec.make_params("exhaustive", 8, 16, 0, False, "original", None, "auto", (0, 1))
    import ctypes
    from paper_1206_4880_b200 import _lib
    lib = _lib.load()
    rc = lib.fic_encode_v1(ctypes.c_void_p(img.data_ptr()), 64, 64, ctypes.byref(p), None, None,
                           None, None, None, None)
    assert rc == _lib.FIC_EINVAL
    assert lib.fic_last_error().decode() == "stride must be >= 1"
    p = codec.make_params("dynamic_fd", 4, 8, 1, False, "original", None, "auto", (0, 1))
    rc = lib.fic_encode_v1(ctypes.c_void_p(img.data_ptr()), 64, 64, ctypes.byref(p), None, None,
                           None, None, None, None)
    assert rc == _lib.FIC_EINVAL
    assert "two DBC scales" in lib.fic_last_error().decode()


def test_deterministic_across_runs_and_segments():
    import torch
    c = synth.CONFIGS["cfg2"]
    img = torch.from_numpy(c.make()).cuda()
    kw = dict(range_size=8, domain_size=16, stride=4, isometries=True, delta=0.1)
    a = codec.encode_device(img, "dynamic_fd", **kw)
    b = codec.encode_device(img, "dynamic_fd", max_segment=512, **kw)
    c2 = codec.encode_device(img, "dynamic_fd", small_pool=1, **kw)
    for x in (b, c2):
        assert torch.equal(a.records, x.records)
        assert torch.equal(a.post_rms, x.post_rms) and torch.equal(a.pre_rms, x.pre_rms)


def test_cta_pair_matcher_equals_default(monkeypatch):
    """The cta_group::2 variant of the matcher (FIC_TC_CG=2: M = 256 rows per
    CTA pair) returns the same records as the default one-CTA matcher."""
    import torch
    c = synth.CONFIGS["cfg2"]
    img = torch.from_numpy(c.make()).cuda()
    kw = dict(range_size=8, domain_size=16, stride=4, isometries=True, delta=0.1)
    a = codec.encode_device(img, "dynamic_fd", **kw)
    monkeypatch.setenv("FIC_TC_CG", "2")
    b = codec.encode_device(img, "dynamic_fd", max_segment=1024, **kw)
    assert b.stats["tensor_tiles"] > 0
    assert torch.equal(a.records, b.records)
    assert torch.equal(a.post_rms, b.post_rms) and torch.equal(a.pre_rms, b.pre_rms)
    # the pilot items on a CTA pair (their stage releases go to the leader's barrier)
    monkeypatch.setenv("FIC_PILOT", str(1 << 30))
    monkeypatch.setenv("FIC_PILOT_STRIDE", "0")
    c2 = codec.encode_device(img, "dynamic_fd", max_segment=1024, **kw)
    assert torch.equal(a.records, c2.records) and torch.equal(a.post_rms, c2.post_rms)


def test_decode_full_size_matches_oracle():
    """Decoder at the headline size: the GPU decode of the cfg3 code (10
    iterations) is byte-identical to the oracle's (codec.py:516-598)."""
    c = synth.CONFIGS["cfg3"]
    img = c.make()
    code, _ = codec.encode(img, c.strategy, range_size=c.range_size, domain_size=c.domain_size,
                           stride=c.stride, isometries=True, delta=c.delta)
    out = codec.decode(code, iterations=10)
    ref = orc.decode(code.records, code.width, code.height, code.range_size, code.domain_size,
                     code.stride, iterations=10)
    assert np.array_equal(out, ref)


@pytest.mark.gpu
def test_run_single_rows_match_reference_bench_rows():
    """runs.run_single on the GPU encoder reproduces every non-timing CSV
    column of the reference's bench.run_single (golden: bench_cases.json)."""
    import json
    import os
    from conftest import ROOT
    from paper_1206_4880_b200 import runs
    g = json.loads(open(os.path.join(ROOT, "tests", "golden", "bench_cases.json")).read())
    timing = [g["columns"].index(c) for c in g["timing_columns"]]
    for run in g["runs"]:
        img = np.array(g["images"][run["name"]], dtype=np.uint8)
        rec, code, recon = runs.run_single(run["name"], img, run["strategy"], stride=4,
                                           isometries=True)
        row = rec.to_row()
        for i in timing:
            row[i] = ""
        assert row == run["row"], run["name"] + "/" + run["strategy"]


DEC = load_golden("decode_cases.npz")
DEC_CASES = sorted({k.split(".")[0] for k in DEC if k.endswith(".iterates")})


def _dec_code(name, recs_key="records"):
    img = DEC[f"{name}.image"]
    stride, iso, sid, rs, ds = (int(v) for v in DEC[f"{name}.params"])
    return codec.FractalCode(img.shape[1], img.shape[0], rs, ds, stride, sid, bool(iso),
                             _recs(DEC[f"{name}.{recs_key}"]).copy())


@pytest.mark.parametrize("name", DEC_CASES)
def test_decode_iterates_match_reference_snapshots(name):
    code = _dec_code(name)
    its = list(codec.decode_iterates(code, 6))
    assert len(its) == 6
    for got, want in zip(its, DEC[f"{name}.iterates"]):
        assert got.dtype == np.uint8 and np.array_equal(got, want)


@pytest.mark.parametrize("name", DEC_CASES)
def test_decode_float_initial_and_level(name):
    code = _dec_code(name)
    out = codec.decode(code, 4, initial=DEC[f"{name}.init_float"])
    assert np.array_equal(out, DEC[f"{name}.decoded_float_init"])
    assert np.array_equal(codec.decode(code, 3, initial=37.25), DEC[f"{name}.decoded_level"])


@pytest.mark.parametrize("name", DEC_CASES)
def test_decode_isometry_bytes_above_7_keep_identity(name):
    code = _dec_code(name, "records_iso_gt7")
    assert int(code.records["isometry"].max()) > 7
    assert np.array_equal(codec.decode(code, 5), DEC[f"{name}.decoded_iso_gt7"])


def test_decode_rejects_out_of_geometry_domain_via_c_abi():
    import ctypes

    import torch
    name = DEC_CASES[0]
    code = _dec_code(name)
    rec = code.records.copy()
    rec["domain"][3] = 10 ** 6
    d_rec = torch.from_numpy(rec.view(np.uint8).copy()).cuda()
    out = torch.empty((code.height, code.width), dtype=torch.uint8, device="cuda")
    lib = codec._lib.load()
    rc = lib.fic_decode_v1(ctypes.c_void_p(d_rec.data_ptr()), code.height, code.width, 8, 16,
                           code.stride, 2, 128.0, None, ctypes.c_void_p(out.data_ptr()), None)
    assert rc == codec._lib.FIC_EINVAL
    assert "outside the current image geometry" in lib.fic_last_error().decode()


def test_encode_accepts_negative_stride_views():
    img = np.random.default_rng(12).integers(0, 256, (64, 64), dtype=np.uint8)
    flipped = np.flipud(img)
    a, _ = codec.encode(flipped, "dynamic_fd", stride=4, isometries=True)
    b, _ = codec.encode(np.ascontiguousarray(flipped), "dynamic_fd", stride=4, isometries=True)
    assert a == b


def test_encode_on_a_second_device_after_the_first():
    """Per-device shared-memory opt-ins: an encode on cuda:1 after cuda:0 (one
    process, two devices) must launch; skipped on a one-GPU box."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    img = synth.CONFIGS["cfg1"].make()
    a, _ = codec.encode(img, "dynamic_fd", stride=8, isometries=True, device=0)
    b, _ = codec.encode(img, "dynamic_fd", stride=8, isometries=True, device=1)
    assert a == b


ODD = load_golden("odd_cases.npz")
ODD_CASES = cases(ODD)


@pytest.mark.parametrize("matcher", ["auto", "exact"])
@pytest.mark.parametrize("name", ODD_CASES)
def test_odd_and_non_pow2_range_sizes_match_reference(name, matcher):
    kw, strat = _params(ODD, name)
    code, st = codec.encode(ODD[f"{name}.image"], strat, matcher=matcher, **kw)
    assert np.array_equal(code.records, _recs(ODD[f"{name}.records"]))
    assert np.array_equal(st.pre_rms, ODD[f"{name}.pre_rms"])
    assert np.array_equal(st.post_rms, ODD[f"{name}.post_rms"])
    assert np.array_equal(st.pool_sizes, ODD[f"{name}.pool_sizes"])
    assert st.comparisons == int(ODD[f"{name}.stats"][0])
    if f"{name}.slab_lo" in ODD:
        p = codec.plan(ODD[f"{name}.image"], strat, range_size=kw["range_size"],
                       domain_size=kw["domain_size"], stride=kw["stride"])
        assert np.array_equal(p["fd_dom"], ODD[f"{name}.fd_dom"])
        assert np.array_equal(p["fd_rng"], ODD[f"{name}.fd_rng"])
        assert np.array_equal(p["slab_lo"], ODD[f"{name}.slab_lo"])
        assert np.array_equal(p["slab_hi"], ODD[f"{name}.slab_hi"])
    assert np.array_equal(codec.decode(code, 10), ODD[f"{name}.decoded"])


@pytest.mark.parametrize("side", [12, 20, 24, 48])
def test_dbc_grid_non_pow2_sides_match_reference(side):
    blocks = ODD[f"dbc{side}.blocks"]
    assert np.array_equal(codec.dbc_grid(blocks), ODD[f"dbc{side}.fd"])
    assert np.array_equal(codec.dbc_grid(blocks, clamp=False), ODD[f"dbc{side}.raw"])


@pytest.mark.parametrize("strategy", ["dynamic_fd", "exhaustive"])
def test_torch_op_encode_matches_oracle(strategy):
    """torch.ops.fic.encode on a device image: the oracle's
    records and RMS bit for bit, stats in STATS_FIELDS order."""
    import torch

    from paper_1206_4880_b200 import ops

    img = np.random.default_rng(7).integers(0, 256, (96, 96), dtype=np.uint8)
    rec, pre, post, pools, stats = torch.ops.fic.encode(
        torch.from_numpy(img).cuda(), 8, 16, 2, True, codec.STRATEGY_IDS[strategy], None, 0)
    ref = orc.encode(img, strategy, stride=2, isometries=True)
    assert np.array_equal(_recs(rec.cpu().numpy()), ref.records)
    assert np.array_equal(pre.cpu().numpy(), ref.pre_rms)
    assert np.array_equal(post.cpu().numpy(), ref.post_rms)
    st = dict(zip(ops.STATS_FIELDS, stats.tolist()))
    assert st["comparisons"] == ref.comparisons and st["n_ranges"] == 144
    with pytest.raises(ValueError):
        torch.ops.fic.encode(torch.from_numpy(img).cuda(), 8, 16, 2, True, 9, None, 0)


@pytest.mark.parametrize("iso", [True, False])
@pytest.mark.parametrize("env", [{}, {"FIC_HL_SORT": "0"}, {"FIC_HL_CAP": "3"}, {"FIC_HL": "0"}])
def test_4x4_hit_list_paths_match_oracle(iso, env, monkeypatch):
    """4x4 ranges through the tensor matcher (pilot + hit list + k_hl_rescore):
    with and without isometries (n_iso 8 / 1), the list unsorted, a list that
    overflows after 3 entries (the rest through the survivor list) and the
    list off -- the oracle's records and RMS bit for bit."""
    import torch

    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(11)
    img = (np.add.outer(np.arange(96), np.arange(96)) // 3).astype(np.uint8)  # smooth half
    img[40:, 40:] = rng.integers(0, 256, (56, 56), dtype=np.uint8)            # texture
    res = codec.encode_device(torch.from_numpy(img).cuda(), "exhaustive", range_size=4,
                              domain_size=8, stride=2, isometries=iso, small_pool=1,
                              max_segment=256)
    ref = orc.encode(img, "exhaustive", range_size=4, domain_size=8, stride=2, isometries=iso)
    assert np.array_equal(_recs(res.records.cpu().numpy()), ref.records)
    assert np.array_equal(res.pre_rms.cpu().numpy(), ref.pre_rms)
    assert np.array_equal(res.post_rms.cpu().numpy(), ref.post_rms)
    assert res.stats["tensor_tiles"] > 0
    if not env:
        assert res.stats["hl_entries"] > 0


def test_kernels_with_per_call_shared_memory_any_size_order():
    """Kernels whose dynamic shared memory depends on the call (the hit-list
    sort: one counter per 64 pool columns) keep working when a smaller call
    comes between two larger ones (the opt-in limit is only ever raised)."""
    import torch

    rng = np.random.default_rng(3)
    small = rng.integers(0, 256, (64, 64), dtype=np.uint8)
    large = rng.integers(0, 256, (384, 384), dtype=np.uint8)
    kw = dict(range_size=4, domain_size=8, stride=2, isometries=True, small_pool=1)
    first = None
    for img in (large, small, large):
        res = codec.encode_device(torch.from_numpy(img).cuda(), "exhaustive", **kw)
        torch.cuda.synchronize()
        assert res.stats["hl_entries"] > 0
        if img is large:
            if first is None:
                first = res.records.clone()
            else:
                assert torch.equal(first, res.records)


def _sweep_cases(n=150, seed=2026):
    """Seeded random small encodes: strategy, range size (domain = 2x),
    stride, isometries, delta, fd_source, matcher and forced tensor routing.
    SWEEP_N / SWEEP_SEED in the environment run a larger one-off campaign
    (profiles/r02_sweep_campaigns.md)."""
    import os
    n = int(os.environ.get("SWEEP_N", n))
    seed = int(os.environ.get("SWEEP_SEED", seed))
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        rs = int(rng.choice([2, 3, 4, 5, 6, 8]))
        strat = str(rng.choice(["exhaustive", "nosearch", "static2", "dynamic_fd"]))
        fd_src = "downsampled" if rng.random() < 0.2 else "original"
        side = rs if fd_src == "downsampled" else 2 * rs
        if strat in ("static2", "dynamic_fd") and side < 8 and side not in (6,):
            strat = "exhaustive"  # one DBC scale: the reference raises (covered elsewhere)
        h = int(rng.integers(3, 9)) * rs * 2
        w = int(rng.integers(3, 9)) * rs * 2
        out.append(dict(i=i, rs=rs, strategy=strat, fd_source=fd_src, h=h, w=w,
                        stride=int(rng.integers(1, rs + 1)), iso=bool(rng.random() < 0.7),
                        delta=[None, 0.05, 0.1, 0.3][int(rng.integers(0, 4))],
                        matcher=str(rng.choice(["auto", "exact"])),
                        small_pool=int(rng.choice([0, 1])), seed=int(rng.integers(1 << 30))))
    return out


@pytest.mark.parametrize("case", _sweep_cases(), ids=lambda c: f"sweep{c['i']}")
def test_random_small_encodes_match_oracle(case):
    """Breadth net for the routing choices (small jobs to the CUDA-core
    matcher, forced tensor path, pilot / hit list for 4x4 ranges, odd sizes,
    every strategy): records and RMS equal the oracle's bit for bit, or both
    raise the same error."""
    import torch

    c = case
    rng = np.random.default_rng(c["seed"])
    base = np.add.outer(np.arange(c["h"]), np.arange(c["w"])) * rng.integers(1, 4)
    img = np.clip(base + rng.normal(0, rng.choice([2, 10, 40]), base.shape), 0, 255).astype(np.uint8)
    if rng.random() < 0.3:
        img[: c["h"] // 2] = img[0, 0]  # a flat band
    kw = dict(range_size=c["rs"], domain_size=2 * c["rs"], stride=c["stride"], isometries=c["iso"],
              fd_source=c["fd_source"])
    delta = c["delta"] if c["strategy"] == "dynamic_fd" else None
    try:
        ref = orc.encode(img, c["strategy"], delta=delta, **kw)
    except ValueError as e:
        with pytest.raises(ValueError, match=re.escape(str(e))):
            codec.encode_device(torch.from_numpy(img).cuda(), c["strategy"], delta=delta,
                                matcher=c["matcher"], small_pool=c["small_pool"], **kw)
        return
    res = codec.encode_device(torch.from_numpy(img).cuda(), c["strategy"], delta=delta,
                              matcher=c["matcher"], small_pool=c["small_pool"], **kw)
    assert np.array_equal(_recs(res.records.cpu().numpy()), ref.records), c
    assert np.array_equal(res.pre_rms.cpu().numpy(), ref.pre_rms), c
    assert np.array_equal(res.post_rms.cpu().numpy(), ref.post_rms), c


@pytest.mark.parametrize("cname", ["cfg1", "cfg2", "cfg4"])
def test_graph_replay_rewrites_outputs_and_stats(cname):
    """A call that repeats the previous one exactly (same image and output
    buffers, parameters) is recorded as a CUDA graph and replayed: with the
    outputs cleared before every call, each replay writes the same records
    and RMS as the first (direct) call, and its stats are live."""
    import torch

    c = synth.CONFIGS[cname]
    img = torch.from_numpy(c.make()).cuda()
    n_r = (img.shape[0] // c.range_size) * (img.shape[1] // c.range_size)
    out = codec.DeviceResult(torch.empty((n_r, 7), dtype=torch.uint8, device="cuda"),
                             torch.empty(n_r, dtype=torch.float64, device="cuda"),
                             torch.empty(n_r, dtype=torch.float64, device="cuda"),
                             torch.empty(n_r, dtype=torch.int64, device="cuda"), {})
    kw = dict(range_size=c.range_size, domain_size=c.domain_size, stride=c.stride,
              isometries=True, delta=c.delta)
    first, modes = None, []
    for _ in range(5):  # direct (arena settling), record + launch, replays
        for t in (out.records, out.pre_rms, out.post_rms, out.pool_sizes):
            t.zero_()
        r = codec.encode_device(img, c.strategy, out=out, **kw)
        torch.cuda.synchronize()
        cur = (r.records.clone(), r.pre_rms.clone(), r.post_rms.clone(), r.pool_sizes.clone())
        assert r.stats["ms_total"] > 0 and r.stats["comparisons"] > 0
        modes.append(int(r.stats["graph"]))
        if first is None:
            first = cur
        else:
            for a, b in zip(first, cur):
                assert torch.equal(a, b)
    # direct until a call repeats the previous one with a settled arena (the
    # arena grows on the second call), then recorded once and replayed
    assert modes[0] == 0 and modes[-2:] == [1, 2] or modes[-2:] == [2, 2], modes
    assert 1 in modes and modes[-1] == 2, modes


@pytest.mark.parametrize("cname", ["cfg1", "cfg2", "cfg4"])
def test_graph_replay_follows_image_content(cname):
    """A replayed graph reads the image buffer anew: after the buffer's
    content changes in place (another seed, a transposed image, an image with
    flat areas, a constant image), the replay's records / RMS / pool sizes /
    comparisons equal a direct (graph-free: any FIC_* variable set) encode
    of a copy of that content."""
    import os

    import torch

    c = synth.CONFIGS[cname]
    base = c.make()
    n_r = (base.shape[0] // c.range_size) * (base.shape[1] // c.range_size)
    buf = torch.from_numpy(base).cuda()
    out = codec.DeviceResult(torch.empty((n_r, 7), dtype=torch.uint8, device="cuda"),
                             torch.empty(n_r, dtype=torch.float64, device="cuda"),
                             torch.empty(n_r, dtype=torch.float64, device="cuda"),
                             torch.empty(n_r, dtype=torch.int64, device="cuda"), {})
    kw = dict(range_size=c.range_size, domain_size=c.domain_size, stride=c.stride,
              isometries=True, delta=c.delta)
    for _ in range(4):
        r = codec.encode_device(buf, c.strategy, out=out, **kw)
    torch.cuda.synchronize()
    assert int(r.stats["graph"]) == 2
    gen = {"cfg1": synth.cfg1_image, "cfg2": synth.cfg2_image, "cfg4": synth.cfg4_image}[cname]
    half_flat = base.copy()
    half_flat[: base.shape[0] // 2] = 97
    variants = [gen(seed=77), np.ascontiguousarray(base.T), half_flat,
                np.full_like(base, 200), base]
    for v in variants:
        buf.copy_(torch.from_numpy(v).cuda())
        for t in (out.records, out.pre_rms, out.post_rms, out.pool_sizes):
            t.zero_()
        r = codec.encode_device(buf, c.strategy, out=out, **kw)
        torch.cuda.synchronize()
        assert int(r.stats["graph"]) == 2
        os.environ["FIC_NO_GRAPH"] = "1"
        try:
            d = codec.encode_device(torch.from_numpy(v).cuda(), c.strategy, **kw)
            torch.cuda.synchronize()
        finally:
            os.environ.pop("FIC_NO_GRAPH", None)
        assert int(d.stats["graph"]) == 0
        assert torch.equal(r.records, d.records)
        assert torch.equal(r.pre_rms, d.pre_rms) and torch.equal(r.post_rms, d.post_rms)
        assert torch.equal(r.pool_sizes, d.pool_sizes)
        assert r.stats["comparisons"] == d.stats["comparisons"]


def _mid_cases(n=4, seed=4242):
    """Seeded mid-size encodes (128-320 px sides, 8x8 and 4x4 ranges, strides
    1-4): big enough for the tensor matcher's multi-tile windows, segments,
    pilot and hit list, small enough for the oracle.  Image kinds stress the
    screen: low contrast (two or three grey levels: ties everywhere),
    gradients with faint noise (near-flat ranges), textures, flat areas.
    SWEEP_MID_N / SWEEP_SEED in the environment run a larger campaign."""
    import os
    n = int(os.environ.get("SWEEP_MID_N", n))
    rng = np.random.default_rng(int(os.environ.get("SWEEP_SEED", seed)))
    out = []
    for i in range(n):
        rs = int(rng.choice([4, 8]))
        stride = int(rng.choice([1, 2, 4]) if rs == 4 else rng.choice([2, 4]))
        h, w = int(rng.integers(8, 21)) * 16, int(rng.integers(8, 21)) * 16
        # keep the oracle's work (R x D x 8 matches at ~1.3e7/s) under ~20 s
        while (h // rs) * (w // rs) * ((h - 2 * rs) // stride + 1) * ((w - 2 * rs) // stride + 1) * 8 > 2.5e8:
            h, w = max(64, h // 2 // 16 * 16), max(64, w // 2 // 16 * 16)
        out.append(dict(i=i, rs=rs, h=h, w=w, stride=stride, small_pool=int(rng.choice([0, 1])),
                        strategy=str(rng.choice(["exhaustive", "dynamic_fd"]) if rs == 8 else "exhaustive"),
                        delta=[None, 0.05, 0.2][int(rng.integers(0, 3))],
                        kind=str(rng.choice(["lowcontrast", "gradient", "texture", "flatmix"])),
                        seed=int(rng.integers(1 << 30))))
    return out


def _mid_image(c):
    rng = np.random.default_rng(c["seed"])
    h, w = c["h"], c["w"]
    if c["kind"] == "lowcontrast":
        return (100 + rng.integers(0, int(rng.integers(2, 4)), (h, w))).astype(np.uint8)
    if c["kind"] == "gradient":
        g = np.add.outer(np.arange(h) * rng.uniform(0.05, 0.6), np.arange(w) * rng.uniform(0.05, 0.6))
        return np.clip(g + rng.normal(0, rng.choice([0.3, 1.0, 3.0]), (h, w)), 0, 255).astype(np.uint8)
    if c["kind"] == "texture":
        return synth.to_u8(synth.fbm(max(h, w), float(rng.uniform(0.2, 0.8)), rng))[:h, :w].copy()
    img = rng.integers(0, 256, (h, w)).astype(np.uint8)
    img[: h // 2, : w // 2] = 37
    img[h // 2:, w // 2:] = (200 + rng.integers(0, 2, (h - h // 2, w - w // 2))).astype(np.uint8)
    return img


@pytest.mark.parametrize("case", _mid_cases(), ids=lambda c: f"mid{c['i']}")
def test_random_mid_size_encodes_match_oracle(case):
    import torch

    c = case
    img = _mid_image(c)
    kw = dict(range_size=c["rs"], domain_size=2 * c["rs"], stride=c["stride"], isometries=True)
    delta = c["delta"] if c["strategy"] == "dynamic_fd" else None
    ref = orc.encode(img, c["strategy"], delta=delta, **kw)
    res = codec.encode_device(torch.from_numpy(img).cuda(), c["strategy"], delta=delta,
                              small_pool=c["small_pool"], **kw)
    if c["small_pool"] == 1:
        assert res.stats["tensor_tiles"] > 0, c
    assert np.array_equal(_recs(res.records.cpu().numpy()), ref.records), c
    assert np.array_equal(res.pre_rms.cpu().numpy(), ref.pre_rms), c
    assert np.array_equal(res.post_rms.cpu().numpy(), ref.post_rms), c
    assert res.stats["comparisons"] == ref.comparisons
