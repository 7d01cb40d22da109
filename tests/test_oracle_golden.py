"""Pin the CPU oracle to the reference's own outputs (tests/golden/*.npz).

The fixtures were produced by tests/golden/make_golden.py, which imports and
runs the reference package.  Everything here is CPU-only.
"""

import numpy as np
import pytest

from conftest import cases, load_golden
from oracle import fic_oracle as orc
from paper_1206_4880_b200 import synth

STRATS = orc.STRATEGIES
ENC = load_golden("encode_cases.npz")
DELTA = load_golden("delta_cases.npz")


def _records(arr):
    return np.ascontiguousarray(arr).view(orc.RECORD_DTYPE).ravel()


@pytest.mark.parametrize("name", [c for c in cases(ENC) if c != "down64_dyn_s2_iso"])
def test_oracle_encode_matches_reference(name):
    g = ENC
    stride, iso, sid, rs, ds = (int(v) for v in g[f"{name}.params"])
    res = orc.encode(g[f"{name}.image"], STRATS[sid], range_size=rs, domain_size=ds,
                     stride=stride, isometries=bool(iso))
    assert np.array_equal(res.records, _records(g[f"{name}.records"]))
    assert np.array_equal(res.pre_rms, g[f"{name}.pre_rms"])
    assert np.array_equal(res.post_rms, g[f"{name}.post_rms"])
    assert np.array_equal(res.pool_sizes, g[f"{name}.pool_sizes"])
    comp, mean_pool = g[f"{name}.stats"]
    assert res.comparisons == int(comp)
    assert res.mean_pool_size == mean_pool
    if f"{name}.fd_dom" in g:
        assert np.array_equal(res.plan.fd_dom, g[f"{name}.fd_dom"])
        assert np.array_equal(res.plan.fd_rng, g[f"{name}.fd_rng"])
        assert np.array_equal(res.plan.order, g[f"{name}.ids"])
        assert np.array_equal(res.plan.lo, g[f"{name}.slab_lo"])
        assert np.array_equal(res.plan.hi, g[f"{name}.slab_hi"])


def test_oracle_fd_source_downsampled():
    name = "down64_dyn_s2_iso"
    res = orc.encode(ENC[f"{name}.image"], "dynamic_fd", stride=2, isometries=True,
                     fd_source="downsampled")
    assert np.array_equal(res.records, _records(ENC[f"{name}.records"]))
    assert np.array_equal(res.pre_rms, ENC[f"{name}.pre_rms"])
    assert np.array_equal(res.post_rms, ENC[f"{name}.post_rms"])


@pytest.mark.parametrize("name", [c for c in cases(ENC) if c != "down64_dyn_s2_iso"])
def test_oracle_decode_matches_reference(name):
    g = ENC
    stride, iso, sid, rs, ds = (int(v) for v in g[f"{name}.params"])
    img = g[f"{name}.image"]
    rec = _records(g[f"{name}.records"])
    out = orc.decode(rec, img.shape[1], img.shape[0], rs, ds, stride, iterations=10)
    assert np.array_equal(out, g[f"{name}.decoded"])
    assert orc.psnr(img, out) == g[f"{name}.psnr"][0]


@pytest.mark.parametrize("name", sorted({k.split(".")[0] for k in DELTA}))
def test_oracle_delta_configs_match_reference(name):
    g = DELTA
    stride, iso, sid, rs, ds = (int(v) for v in g[f"{name}.params"])
    cfg = synth.CONFIGS[name.split("_")[0]]
    img = g[f"{name}.image"] if f"{name}.image" in g else cfg.make()
    import hashlib
    if hashlib.sha256(img.tobytes()).hexdigest() != str(g[f"{name}.sha"]):
        pytest.skip("synthetic generator output differs on this host (FFT bits)")
    delta = float(g[f"{name}.delta"][0])
    delta = None if np.isnan(delta) else delta
    ids = g[f"{name}.range_ids"]
    res = orc.encode(img, STRATS[sid], range_size=rs, domain_size=ds, stride=stride,
                     isometries=bool(iso), delta=delta, range_ids=ids)
    assert np.array_equal(res.records[ids], _records(g[f"{name}.records"]))
    assert np.array_equal(res.pre_rms[ids], g[f"{name}.pre_rms"])
    assert np.array_equal(res.post_rms[ids], g[f"{name}.post_rms"])
    assert np.array_equal(res.pool_sizes, g[f"{name}.pool_sizes"])
    assert res.comparisons == int(g[f"{name}.comparisons"][0])
    if f"{name}.fd_rng" in g:
        assert np.array_equal(res.plan.fd_rng, g[f"{name}.fd_rng"])
        pick = g[f"{name}.fd_dom_pick"]
        assert np.array_equal(res.plan.fd_dom[pick], g[f"{name}.fd_dom_vals"])
        s, lo, hi = g[f"{name}.fd_dom_sum"]
        assert res.plan.fd_dom.sum() == s and res.plan.fd_dom.min() == lo
        assert res.plan.fd_dom.max() == hi
        assert hashlib.sha256(res.plan.order.astype(np.int64).tobytes()).hexdigest() \
            == str(g[f"{name}.ids_sha"])
        assert np.array_equal(res.plan.lo, g[f"{name}.slab_lo"])
        assert np.array_equal(res.plan.hi, g[f"{name}.slab_hi"])


def test_oracle_dbc_known_answers(golden_fd):
    g = golden_fd
    for side in (8, 16, 32):
        assert np.array_equal(orc.dbc(g[f"rand{side}.blocks"]), g[f"rand{side}.fd"])
        assert np.array_equal(orc.dbc(g[f"rand{side}.blocks"], clamp=False),
                              g[f"rand{side}.raw"])
    assert np.all(orc.dbc(g["const16.blocks"]) == 2.0)
    assert np.array_equal(orc.dbc(g["const8.blocks"]), g["const8.fd"])
    assert orc.dbc(g["checker8.blocks"])[0] == 3.0
    assert orc.dbc(g["spike8.blocks"], clamp=False)[0] == g["spike8.raw"][0] < 2.0
    for side in (4, 8, 12, 16, 32, 64):
        assert orc.dbc_scales(side) == list(g[f"scales{side}"])
    for side in (8, 16, 32):
        assert np.array_equal(orc.dbc_weights(side), g[f"weights{side}"])
    assert np.array_equal(orc.iso_perms(8), g["perms8"])
    assert np.array_equal(orc.iso_perms(4), g["perms4"])


def test_oracle_validation_messages():
    img = np.zeros((64, 64), np.uint8)
    with pytest.raises(ValueError, match="uint8"):
        orc.encode(img.astype(np.float32), "exhaustive")
    with pytest.raises(ValueError, match="unknown strategy"):
        orc.encode(img, "bogus")
    with pytest.raises(ValueError, match="twice"):
        orc.encode(img, "exhaustive", range_size=8, domain_size=24)
    with pytest.raises(ValueError, match="fd_source"):
        orc.encode(img, "exhaustive", fd_source="x")
    with pytest.raises(ValueError, match="two DBC scales"):
        orc.encode(img, "dynamic_fd", range_size=4, domain_size=8)
    with pytest.raises(ValueError, match="not divisible"):
        orc.encode(np.zeros((60, 64), np.uint8), "exhaustive")


ODD = load_golden("odd_cases.npz")


@pytest.mark.parametrize("name", cases(ODD))
def test_oracle_odd_range_sizes_match_reference(name):
    stride, iso, sid, rs, ds = (int(v) for v in ODD[f"{name}.params"])
    res = orc.encode(ODD[f"{name}.image"], orc.STRATEGIES[sid], range_size=rs, domain_size=ds,
                     stride=stride, isometries=bool(iso))
    want = np.ascontiguousarray(ODD[f"{name}.records"]).view(orc.RECORD_DTYPE).ravel()
    assert np.array_equal(res.records, want)
    assert np.array_equal(res.pre_rms, ODD[f"{name}.pre_rms"])
    assert np.array_equal(res.post_rms, ODD[f"{name}.post_rms"])


@pytest.mark.parametrize("side", [12, 20, 24, 48])
def test_oracle_dbc_non_pow2_sides(side):
    blocks = ODD[f"dbc{side}.blocks"]
    assert np.array_equal(orc.dbc(blocks), ODD[f"dbc{side}.fd"])
    assert np.array_equal(orc.dbc(blocks, clamp=False), ODD[f"dbc{side}.raw"])
