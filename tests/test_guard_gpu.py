"""Home-made write check (compute-sanitizer is closed on this pool).

FIC_ARENA_GUARD=1 makes the library follow every scratch buffer of a call
with a red zone (its alignment slack + 256 B of 0xA5) and verify all of them
after the call's kernels; a kernel that writes past a scratch buffer makes
the call raise.  The caller-owned outputs are checked the same way here:
they are carved out of one flat buffer with 0xA5 bands around each.  Every
path is run under the guard -- all strategies and matchers on the small
goldens, odd range sizes, every survivor path at cfg2 / cfg4, cfg3, the
decoder, the planner, the pool builder and the DBC entry point -- and its
results must still equal the reference's."""

import numpy as np
import pytest

from conftest import cases, load_golden
from paper_1206_4880_b200 import codec, synth

pytestmark = pytest.mark.gpu

ENC = load_golden("encode_cases.npz")
BAND = 4096


@pytest.fixture(autouse=True)
def _guard(monkeypatch):
    monkeypatch.setenv("FIC_ARENA_GUARD", "1")


def _banded_outputs(torch, n_r):
    """records / pre / post / pool sizes inside one flat buffer, 0xA5 bands
    before, between and after them."""
    sizes = [n_r * 7, n_r * 8, n_r * 8, n_r * 8]
    offs, o = [], BAND
    for sz in sizes:
        offs.append(o)
        o += (sz + 255) // 256 * 256 + BAND
    flat = torch.full((o,), 0xA5, dtype=torch.uint8, device="cuda")
    rec = flat[offs[0]:offs[0] + sizes[0]].view(n_r, 7)
    pre = flat[offs[1]:offs[1] + sizes[1]].view(torch.float64)
    post = flat[offs[2]:offs[2] + sizes[2]].view(torch.float64)
    pools = flat[offs[3]:offs[3] + sizes[3]].view(torch.int64)
    mask = torch.ones(o, dtype=torch.bool, device="cuda")
    for off, sz in zip(offs, sizes):
        mask[off:off + sz] = False
    return flat, mask, codec.DeviceResult(rec, pre, post, pools, {})


def _encode_checked(img, strategy, **kw):
    import torch
    rs = kw.get("range_size", 8)
    n_r = (img.shape[0] // rs) * (img.shape[1] // rs)
    flat, mask, out = _banded_outputs(torch, n_r)
    res = codec.encode_device(torch.from_numpy(img).cuda(), strategy, out=out, **kw)
    torch.cuda.synchronize()
    assert bool((flat[mask] == 0xA5).all()), "a kernel wrote outside the caller's output buffers"
    return res


def _recs(a):
    return np.ascontiguousarray(a).view(codec.RECORD_DTYPE).ravel()


@pytest.mark.parametrize("matcher", ["auto", "exact"])
@pytest.mark.parametrize("name", [c for c in cases(ENC) if c != "down64_dyn_s2_iso"])
def test_small_goldens_under_guard(name, matcher):
    stride, iso, sid, rs, ds = (int(v) for v in ENC[f"{name}.params"])
    for small_pool in (None, 1):  # default routing, then everything through the tensor matcher
        kw = dict(stride=stride, isometries=bool(iso), range_size=rs, domain_size=ds, matcher=matcher)
        if small_pool is not None:
            kw["small_pool"] = small_pool
        res = _encode_checked(ENC[f"{name}.image"], codec.STRATEGIES[sid], **kw)
        assert np.array_equal(_recs(res.records.cpu().numpy()), _recs(ENC[f"{name}.records"]))
        assert np.array_equal(res.post_rms.cpu().numpy(), ENC[f"{name}.post_rms"])


@pytest.mark.parametrize("fname,prefix,env", [
    ("scale_cfg2.npz", "cfg2", {}),
    ("scale_cfg2.npz", "cfg2_ex", {}),
    ("scale_cfg2.npz", "cfg2", {"FIC_POOL_PLANES": "1"}),
    ("scale_cfg3.npz", "cfg3", {}),
    ("scale_cfg4.npz", "cfg4_ex", {}),
    ("scale_cfg4.npz", "cfg4_ex", {"FIC_HL": "0"}),
    ("scale_cfg4.npz", "cfg4_ex", {"FIC_HL_CAP": "4096"}),
    ("scale_cfg4.npz", "cfg4_ex", {"FIC_SL_CAP": "4096", "FIC_HL": "0"}),
    ("scale_cfg4.npz", "cfg4_ex", {"FIC_PILOT": "0", "FIC_SL": "0"}),
])
def test_scale_configs_under_guard(fname, prefix, env, monkeypatch):
    import os

    from conftest import GOLDEN
    if not os.path.exists(os.path.join(GOLDEN, fname)):
        pytest.skip(f"{fname} not generated")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = load_golden(fname)
    img = g[f"{prefix}.image"] if f"{prefix}.image" in g else synth.CONFIGS[prefix.split("_")[0]].make()
    stride, iso, sid, rs, ds = (int(v) for v in g[f"{prefix}.params"])
    delta = float(g[f"{prefix}.delta"][0])
    res = _encode_checked(img, codec.STRATEGIES[sid], range_size=rs, domain_size=ds, stride=stride,
                          isometries=bool(iso), delta=None if np.isnan(delta) else delta)
    want = np.ascontiguousarray(g[f"{prefix}.records"])
    if want.shape == tuple(res.records.shape):  # same image (the generator is host-dependent otherwise)
        import hashlib
        if hashlib.sha256(np.ascontiguousarray(img).tobytes()).hexdigest() == str(g[f"{prefix}.sha"]):
            assert np.array_equal(res.records.cpu().numpy(), want)


def test_planner_pool_dbc_decode_under_guard():
    import torch
    c = synth.CONFIGS["cfg2"]
    img = c.make()
    d = torch.from_numpy(img).cuda()
    kw = dict(range_size=8, domain_size=16, stride=4)
    p = codec.plan(d, "dynamic_fd", delta=0.1, **kw)
    assert len(p["order"]) == 15625
    for strategy in ("dynamic_fd", "exhaustive"):
        codec.pool(d, strategy, delta=0.1 if strategy == "dynamic_fd" else None, **kw)
    rng = np.random.default_rng(5)
    for side in (8, 12, 16, 20, 24, 48):
        blocks = rng.integers(0, 256, (257, side, side), dtype=np.uint8)
        codec.dbc_grid(blocks)
    code, _ = codec.encode(img, "dynamic_fd", delta=0.1, isometries=True, **kw)
    out = codec.decode(code, iterations=6)
    assert out.shape == img.shape
    assert sum(1 for _ in codec.decode_iterates(code, iterations=3)) == 3


def test_guard_detects_an_overrun():
    """The check itself: the library's self-test entry overruns a scratch
    buffer by one byte on purpose and the call must raise."""
    from paper_1206_4880_b200 import _lib
    lib = _lib.load()
    assert lib.fic_guard_selftest_v1(0) == 0  # in bounds: clean
    assert lib.fic_guard_selftest_v1(1) != 0  # one byte past the buffer
    assert b"FIC_ARENA_GUARD" in lib.fic_last_error()
