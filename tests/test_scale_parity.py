"""At-scale GPU parity against the REFERENCE's own outputs.

The fixtures (tests/golden/make_scale_golden.py) hold what the reference
package itself computed -- its setup and its ``_search_chunk`` -- for EVERY
range of cfg2 (dynamic and exhaustive), cfg3 and cfg4 (exhaustive, 4x4),
and for 1,024 ranges of cfg5 (16 of them empty-window fallbacks) plus cfg5's full pool sizes and checksums of its
slabs, range FDs and FD order.  Records and both RMS columns must be
bit-identical; near-ties (SURVEY §8c protocol: the reference's and our
candidate within 1e-6 relative) are counted and must be zero.
"""

import hashlib
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden
from paper_1206_4880_b200 import codec, synth

pytestmark = pytest.mark.gpu


def _golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not generated")
    return load_golden(name)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _kw(g, prefix):
    stride, iso, sid, rs, ds = (int(v) for v in g[f"{prefix}.params"])
    delta = float(g[f"{prefix}.delta"][0])
    return codec.STRATEGIES[sid], dict(range_size=rs, domain_size=ds, stride=stride,
                                       isometries=bool(iso),
                                       delta=None if np.isnan(delta) else delta)


def _image(g, prefix):
    if f"{prefix}.image" in g:
        img = g[f"{prefix}.image"]
    else:
        img = synth.CONFIGS[prefix.split("_")[0]].make()
    if _sha(img) != str(g[f"{prefix}.sha"]):
        pytest.skip("synthetic generator output differs on this host")
    return img


def _compare(g, prefix, res, ids=None):
    """Bitwise records / RMS; returns (mismatches, near_ties)."""
    want_rec = np.ascontiguousarray(g[f"{prefix}.records"])
    got_rec = res.records.cpu().numpy()
    got_pre = res.pre_rms.cpu().numpy()
    got_post = res.post_rms.cpu().numpy()
    if ids is not None:
        got_rec, got_pre, got_post = got_rec[ids], got_pre[ids], got_post[ids]
    bad = np.flatnonzero((got_rec != want_rec).any(axis=1))
    e_got = got_post[bad] ** 2
    e_ref = g[f"{prefix}.post_rms"][bad] ** 2
    near = int(np.count_nonzero(np.abs(e_got - e_ref) <= 1e-6 * e_ref))
    return bad, near, got_pre, got_post


def _check_full(fname, prefix, matcher="auto"):
    import torch
    g = _golden(fname)
    img = _image(g, prefix)
    strategy, kw = _kw(g, prefix)
    res = codec.encode_device(torch.from_numpy(img).cuda(), strategy, matcher=matcher, **kw)
    bad, near, pre, post = _compare(g, prefix, res)
    assert len(bad) == 0, f"{len(bad)} ranges differ ({near} near-ties), first {bad[:8]}"
    assert np.array_equal(pre, g[f"{prefix}.pre_rms"])
    assert np.array_equal(post, g[f"{prefix}.post_rms"])
    assert np.array_equal(res.pool_sizes.cpu().numpy(), g[f"{prefix}.pool_sizes"])
    assert res.stats["comparisons"] == int(g[f"{prefix}.comparisons"][0])
    return g, res


@pytest.mark.parametrize("prefix", ["cfg2", "cfg2_ex"])
def test_cfg2_every_range_matches_reference(prefix):
    _check_full("scale_cfg2.npz", prefix)


def test_cfg2_exact_matcher_every_range_matches_reference():
    _check_full("scale_cfg2.npz", "cfg2", matcher="exact")


def test_cfg3_every_range_matches_reference():
    import torch
    g, res = _check_full("scale_cfg3.npz", "cfg3")
    img = g["cfg3.image"]
    p = codec.plan(torch.from_numpy(img).cuda(), "dynamic_fd", range_size=8, domain_size=16,
                   stride=1, delta=0.05)
    assert np.array_equal(p["slab_lo"], g["cfg3.slab_lo"])
    assert np.array_equal(p["slab_hi"], g["cfg3.slab_hi"])
    assert _sha(p["order"]) == str(g["cfg3.ids_sha"])


def test_cfg4_exhaustive_every_range_matches_reference():
    _check_full("scale_cfg4.npz", "cfg4_ex")


def test_cfg5_ranges_pools_and_slabs_match_reference():
    import torch
    g = _golden("scale_cfg5.npz")
    img = _image(g, "cfg5")
    strategy, kw = _kw(g, "cfg5")
    d_img = torch.from_numpy(img).cuda()
    res = codec.encode_device(d_img, strategy, **kw)
    ids = g["cfg5.range_ids"]
    bad, near, pre, post = _compare(g, "cfg5", res, ids)
    assert len(bad) == 0, f"{len(bad)} of {len(ids)} cfg5 ranges differ ({near} near-ties)"
    assert np.array_equal(pre, g["cfg5.pre_rms"]) and np.array_equal(post, g["cfg5.post_rms"])
    assert np.array_equal(res.pool_sizes.cpu().numpy(), g["cfg5.pool_sizes"])
    assert res.stats["comparisons"] == int(g["cfg5.comparisons"][0])
    p = codec.plan(d_img, strategy, range_size=8, domain_size=16, stride=kw["stride"],
                   delta=kw["delta"])
    assert _sha(p["slab_lo"]) == str(g["cfg5.slab_lo_sha"])
    assert _sha(p["slab_hi"]) == str(g["cfg5.slab_hi_sha"])
    assert _sha(p["fd_rng"]) == str(g["cfg5.fd_rng_sha"])
    assert _sha(p["order"]) == str(g["cfg5.ids_sha"])
    fd = p["fd_dom"]
    assert [fd.sum(), fd.min(), fd.max()] == list(g["cfg5.fd_dom_sum"])


@pytest.mark.parametrize("cname", ["cfg2", "cfg3"])
@pytest.mark.parametrize("strategy,planes", [("exhaustive", False), ("dynamic_fd", False),
                                             ("dynamic_fd", True)])
def test_pool_builder_outputs_match_reference(cname, strategy, planes, monkeypatch):
    """K1 directly: decimated domains, sum_d, sum_dd and inv_den bitwise equal
    to the reference's downsample2(domain_stack) and _SearchContext (raster
    order, SHA-256 of the whole arrays + 4,096 sampled rows), through the
    row-segment and the box-plane sources."""
    g = _golden("scale_k1.npz")
    img = synth.CONFIGS[cname].make()
    if _sha(img) != str(g[f"{cname}.sha"]):
        pytest.skip("synthetic generator output differs on this host")
    if planes:
        monkeypatch.setenv("FIC_POOL_PLANES", "1")
    st = int(g[f"{cname}.stride"][0])
    out = codec.pool(img, strategy, range_size=8, domain_size=16, stride=st, delta=0.05)
    inv = np.argsort(out["order"])          # raster id -> pool position
    dec = out["decimated"][inv]
    sum_d = out["sum_d"][inv].astype(np.float64)
    sum_dd = out["sum_dd"][inv].astype(np.float64)
    inv_den = out["inv_den"][inv]
    pick = g[f"{cname}.pick"]
    assert np.array_equal(dec[pick], g[f"{cname}.dec_pick"])
    assert np.array_equal(sum_d[pick], g[f"{cname}.sum_d_pick"])
    assert np.array_equal(sum_dd[pick], g[f"{cname}.sum_dd_pick"])
    assert np.array_equal(inv_den[pick], g[f"{cname}.inv_den_pick"])
    assert _sha(dec) == str(g[f"{cname}.dec_sha"])
    assert _sha(sum_d) == str(g[f"{cname}.sum_d_sha"])
    assert _sha(sum_dd) == str(g[f"{cname}.sum_dd_sha"])
    assert _sha(inv_den) == str(g[f"{cname}.inv_den_sha"])


@pytest.mark.parametrize("env", [{"FIC_SL": "1"}, {"FIC_SL": "1", "FIC_SL_ALL": "1"},
                                 {"FIC_PILOT": "4096"}, {"FIC_PILOT": "0"},
                                 {"FIC_PILOT": "16384", "FIC_SL": "1", "FIC_SL_ALL": "1"},
                                 {"FIC_SL": "1", "FIC_SL_CAP": "7"}])
@pytest.mark.parametrize("prefix", ["cfg2", "cfg2_ex"])
def test_survivor_paths_match_reference(prefix, env, monkeypatch):
    """Every way a survivor can be rescored gives the reference's records:
    the survivor list (overflow of the rescoring warp's queues, or every
    survivor), with and without the pilot items that seed the thresholds,
    and a
    survivor list that overflows after 7 entries (the rest go through the
    rescoring warp)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _, res = _check_full("scale_cfg2.npz", prefix)
    # (8x8 main items hand their hits to the rescoring warp through the hit
    # ring, FIC_TC_DUMP; the survivor list serves 4x4 ranges and builds with
    # -DFIC_TC_DUMP=0, where FIC_SL_ALL must put entries on it)
    if "FIC_SL_CAP" in env:
        assert res.stats["sl_entries"] <= 7


def test_cfg4_exhaustive_queue_path_matches_reference(monkeypatch):
    """cfg4 without the pilot and the survivor list (the default for 4x4
    ranges): every survivor through the rescoring warp, bit-exact too."""
    monkeypatch.setenv("FIC_PILOT", "0")
    monkeypatch.setenv("FIC_SL", "0")
    _, res = _check_full("scale_cfg4.npz", "cfg4_ex")
    assert res.stats["sl_entries"] == 0


def test_cfg4_default_uses_pilot_and_hit_list():
    import torch
    g = _golden("scale_cfg4.npz")
    strategy, kw = _kw(g, "cfg4_ex")
    res = codec.encode_device(torch.from_numpy(g["cfg4_ex.image"]).cuda(), strategy, **kw)
    assert res.stats["hl_entries"] > 0 and res.stats["hl_tests"] > 0


@pytest.mark.parametrize("env", [{"FIC_HL": "0"}, {"FIC_HL_CAP": "5000"}, {"FIC_HL_CAP": "1"}])
def test_cfg4_hit_list_variants_match_reference(env, monkeypatch):
    """cfg4 with the hit list off (per-row survivor masks to the survivor
    list), and with a hit list that overflows (the rest of the hit chunks
    take the survivor-mask path): bit-exact on every range."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _, res = _check_full("scale_cfg4.npz", "cfg4_ex")
    if env.get("FIC_HL") == "0":
        assert res.stats["hl_entries"] == 0 and res.stats["sl_entries"] > 0
    else:
        assert res.stats["hl_entries"] <= int(env["FIC_HL_CAP"]) and res.stats["sl_entries"] > 0
