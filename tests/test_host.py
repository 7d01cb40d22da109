"""CPU-only checks of the host side and the C ABI library (no compute calls)."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT, cases, load_golden
from paper_1206_4880_b200 import _lib, codec
from oracle import fic_oracle as orc

HEADER = os.path.join(ROOT, "include", "fic_b200.h")


def _header_symbols():
    text = open(HEADER).read()
    return set(re.findall(r"^\s*(?:int|const char\*|void)\s+(fic_\w+)\s*\(", text, re.M))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    declared = _header_symbols()
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.fic_abi_version() == 1


def test_library_has_sm100a_tensor_core_code():
    out = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    sass = out.stdout
    assert "UTCHMMA" in sass      # tcgen05.mma
    assert "LDTM" in sass         # tcgen05.ld
    assert "UTMALDG" in sass      # TMA load
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH],
                                       capture_output=True, text=True).stdout


def test_params_struct_matches_c_layout(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "fic_b200.h"\n'
        'int main(void){printf("%zu %zu %zu %zu %zu\\n", sizeof(fic_params_t),'
        ' offsetof(fic_params_t, delta), offsetof(fic_params_t, n_fd_weights_rng),'
        ' sizeof(fic_stats_t), sizeof(fic_record_t));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert got == [ctypes.sizeof(_lib.FicParams), _lib.FicParams.delta.offset,
                   _lib.FicParams.n_fd_weights_rng.offset, ctypes.sizeof(_lib.FicStats), 7]


def test_record_dtype_round_trip():
    assert codec.RECORD_DTYPE.itemsize == 7
    rec = np.zeros(3, codec.RECORD_DTYPE)
    rec["domain"] = [1, 70000, 2**32 - 1]
    rec["isometry"], rec["s_q"], rec["o_q"] = [0, 7, 3], [0, 31, 16], [0, 127, 64]
    raw = rec.view(np.uint8).reshape(-1, 7)
    assert np.array_equal(codec.records_from_bytes(raw), rec)


@pytest.mark.parametrize("call, msg", [
    (lambda: codec.validate(np.zeros((64, 64), np.float32), "exhaustive", 8, 16, 1, "original"), "uint8"),
    (lambda: codec.validate(np.zeros((64, 64), np.uint8), "bogus", 8, 16, 1, "original"), "unknown strategy"),
    (lambda: codec.validate(np.zeros((64, 64), np.uint8), "exhaustive", 8, 24, 1, "original"), "twice"),
    (lambda: codec.validate(np.zeros((64, 64), np.uint8), "exhaustive", 8, 16, 1, "x"), "fd_source"),
    (lambda: codec.validate(np.zeros((60, 64), np.uint8), "exhaustive", 8, 16, 1, "original"), "not divisible"),
    (lambda: codec.validate(np.zeros((64, 64), np.uint8), "exhaustive", 8, 16, 0, "original"), "stride must be >= 1"),
    (lambda: codec.validate(np.zeros((8, 8), np.uint8), "exhaustive", 8, 16, 1, "original"), "exceeds"),
    (lambda: codec.validate(np.zeros((64, 64), np.uint8), "dynamic_fd", 4, 8, 1, "original"), "two DBC scales"),
])
def test_validation_texts_match_reference(call, msg):
    with pytest.raises(ValueError, match=msg) as got:
        call()
    # the oracle restates the reference's own messages: identical text
    ref_calls = {
        "uint8": lambda: orc.encode(np.zeros((64, 64), np.float32), "exhaustive"),
        "unknown strategy": lambda: orc.encode(np.zeros((64, 64), np.uint8), "bogus"),
        "twice": lambda: orc.encode(np.zeros((64, 64), np.uint8), "exhaustive", domain_size=24),
        "fd_source": lambda: orc.encode(np.zeros((64, 64), np.uint8), "exhaustive", fd_source="x"),
        "not divisible": lambda: orc.encode(np.zeros((60, 64), np.uint8), "exhaustive"),
        "stride must be >= 1": lambda: orc.encode(np.zeros((64, 64), np.uint8), "exhaustive", stride=0),
        "exceeds": lambda: orc.encode(np.zeros((8, 8), np.uint8), "exhaustive"),
        "two DBC scales": lambda: orc.encode(np.zeros((64, 64), np.uint8), "dynamic_fd",
                                             range_size=4, domain_size=8),
    }
    with pytest.raises(ValueError) as ref:
        ref_calls[msg]()
    assert str(got.value) == str(ref.value)


def test_dbc_weights_and_ln_table_match_reference_numpy(golden_fd):
    for side in (8, 16, 32):
        assert np.array_equal(codec.dbc_weights(side), golden_fd[f"weights{side}"])
    ln = codec.ln_table()
    assert ln[1] == 0.0 and ln[64] == np.log(64.0)


def test_serialize_matches_reference_bytes():
    g = load_golden("encode_cases.npz")
    for name in cases(g):
        if f"{name}.fic1" not in g:
            continue
        stride, iso, sid, rs, ds = (int(v) for v in g[f"{name}.params"])
        img = g[f"{name}.image"]
        recs = codec.records_from_bytes(g[f"{name}.records"]).copy()
        code = codec.FractalCode(img.shape[1], img.shape[0], rs, ds, stride, sid, bool(iso), recs)
        blob = codec.serialize(code)
        assert blob == g[f"{name}.fic1"].tobytes()
        assert codec.deserialize(blob) == code


@pytest.mark.parametrize("mutate, message", [
    (lambda b: b[:10], "shorter than the fixed header"),
    (lambda b: b"XXXX" + b[4:], "magic"),
    (lambda b: b[:4] + bytes([9]) + b[5:], "version"),
    (lambda b: b[:-3], "fewer record bytes"),
    (lambda b: b + b"\x00", "trailing"),
])
def test_deserialize_rejects_malformed(mutate, message):
    g = load_golden("encode_cases.npz")
    blob = g["flat32_ns_s4.fic1"].tobytes()
    with pytest.raises(codec.FormatError, match=message):
        codec.deserialize(mutate(blob))


def test_make_params_fields():
    p = codec.make_params("dynamic_fd", 8, 16, 2, True, "original", 0.05, "auto", (1, 4))
    assert (p.range_size, p.domain_size, p.stride, p.isometries) == (8, 16, 2, 1)
    assert (p.strategy, p.has_delta, p.delta) == (3, 1, 0.05)
    assert (p.shard_index, p.shard_count, p.n_fd_weights_dom, p.n_fd_weights_rng) == (1, 4, 3, 2)
    with pytest.raises(ValueError, match="unknown matcher"):
        codec.make_params("dynamic_fd", 8, 16, 2, True, "original", None, "bogus", (0, 1))


def _bench_cases():
    import json
    return json.loads(open(os.path.join(ROOT, "tests", "golden", "bench_cases.json")).read())


def test_run_record_columns_and_formatting_match_reference():
    from paper_1206_4880_b200 import runs
    g = _bench_cases()
    assert runs.CSV_COLUMNS == g["columns"]
    assert list(runs.TIMING_COLUMNS) == g["timing_columns"]
    # a record rebuilt from a reference row formats back to the same strings
    row = g["runs"][0]["row"]
    typed = dict(zip(g["columns"], row))
    rec = runs.RunRecord(
        image_name=typed["image_name"], image_size=int(typed["image_size"]),
        range_size=int(typed["range_size"]), domain_size=int(typed["domain_size"]),
        stride=int(typed["stride"]), isometries=bool(int(typed["isometries"])),
        strategy=typed["strategy"], strategy_id=int(typed["strategy_id"]),
        encode_seconds=1.25, fd_overhead_seconds=0.0,
        comparisons=int(typed["comparisons"]), mean_pool_size=float(typed["mean_pool_size"]),
        domain_count=int(typed["domain_count"]), compressed_bytes=int(typed["compressed_bytes"]),
        pre_rms_mean=float(typed["pre_rms_mean"]), post_rms_mean=float(typed["post_rms_mean"]),
        psnr_db=float(typed["psnr_db"]), decode_iterations=int(typed["decode_iterations"]))
    out = rec.to_row()
    assert out[8:10] == ["1.250000", "0.000000"]
    assert out[:8] + out[10:] == row[:8] + row[10:]
    rec.psnr_db = rec.decode_iterations = None
    assert rec.to_row()[-2:] == ["", ""]


def test_write_csv_and_pgm(tmp_path):
    import csv
    from paper_1206_4880_b200 import runs
    rec = runs.RunRecord("img", 64, 8, 16, 4, False, "nosearch", 1, 0.1, 0.0, 10, 1.0, 169,
                         100, 1.0, 2.0, float("inf"), 10)
    runs.write_csv([rec, rec], tmp_path / "r.csv")
    rows = list(csv.reader(open(tmp_path / "r.csv")))
    assert rows[0] == runs.CSV_COLUMNS and len(rows) == 3 and rows[1][16] == "inf"
    img = (np.arange(12, dtype=np.uint8) * 20).reshape(3, 4)
    runs.write_pgm(img, tmp_path / "i.pgm")
    assert (tmp_path / "i.pgm").read_bytes() == b"P5\n4 3\n255\n" + img.tobytes()
    assert runs.fidelity_psnr(img, img) == float("inf")
    with pytest.raises(ValueError, match="dimension mismatch"):
        runs.fidelity_psnr(img, img[:2])


def test_bench_pool_roofline_arithmetic():
    """bench.py's HBM roofline of K1 on SURVEY §8(d)'s bytes (H*W + D*(2K+16),
    147.6 MB at cfg3) over the mean device time of k_pool and of the K1 stage."""
    import bench
    stats = [{"ms_pool_main": 0.05, "ms_pool": 0.06}, {"ms_pool_main": 0.05, "ms_pool": 0.06}]
    r = bench._pool_roofline(stats, 6552.3, "measured",
                             serial_stats=[{"ms_pool_main": 0.04, "ms_pool": 0.045}])
    d = 1009 * 1009
    assert r["algorithmic_bytes_per_launch"] == 1024 * 1024 + d * (2 * 64 + 16)
    assert abs(r["algorithmic_bytes_per_launch"] - 147.6e6) < 0.1e6
    assert abs(r["achieved"] - r["algorithmic_bytes_per_launch"] / 0.05e-3 / 1e9) < 1e-6
    assert abs(r["frac"] - r["achieved"] / 6552.3) < 1e-12
    assert abs(r["k1_stage"]["achieved"] - r["algorithmic_bytes_per_launch"] / 0.06e-3 / 1e9) < 1e-6
    assert r["bound"] == "hbm" and r["isolated"]["ms_per_launch"] == 0.04
    assert r["isolated"]["k1_stage_ms"] == 0.045


def test_bench_parity_counts_mismatches_and_near_ties():
    import bench
    with np.load(os.path.join(ROOT, "tests", "golden", "scale_cfg3.npz")) as z:
        rec, pre, post = z["cfg3.records"].copy(), z["cfg3.pre_rms"], z["cfg3.post_rms"].copy()
    p = bench._parity_vs_reference(rec, pre, post)
    assert p["record_mismatches"] == 0 and p["rms_bit_exact"] and p["ranges"] == 16384
    rec[5, 4] ^= 1                        # another isometry, same error: a near-tie
    rec[9, 0] ^= 1
    post[9] *= 1.01                       # a real mismatch
    p = bench._parity_vs_reference(rec, pre, post)
    assert p["record_mismatches"] == 2 and p["near_ties"] == 1 and not p["rms_bit_exact"]


def test_bench_clock_summary_from_nvidia_smi_lines():
    """The clock sampler's nvidia-smi fallback: median SM clock, max clock,
    and the throttle reasons that were active in any sample."""
    import bench
    c = bench.Clocks(0)
    c.lines = ["1965, 1965, 700.1, 0x0, Not Active, Not Active, Not Active, Not Active",
               "1800, 1965, 990.0, 0x4, Not Active, Not Active, Not Active, Active",
               "1900, 1965, 950.0, 0x0, Not Active, Not Active, Not Active, Not Active"]
    s = c.summary()
    assert s["sm_mhz"] == 1900.0 and s["sm_max_mhz"] == 1965.0 and s["samples"] == 3
    assert s["reasons"] == ["sw_power_cap"]


def test_params_are_cached_per_argument_tuple():
    p1 = codec.make_params("dynamic_fd", 8, 16, 1, True, "original", 0.05, "auto", (0, 1))
    p2 = codec.make_params("dynamic_fd", 8, 16, 1, True, "original", 0.05, "auto", (0, 1))
    p3 = codec.make_params("dynamic_fd", 8, 16, 2, True, "original", 0.05, "auto", (0, 1))
    assert p1 is p2 and p1 is not p3
    assert p3.stride == 2 and p1.stride == 1


def test_scalar_fit_and_quantiser_match_reference(golden_decode):
    g = golden_decode
    for row, want in zip(g["fit.inputs"], g["fit.outputs"]):
        n = int(np.count_nonzero(~np.isnan(row[0])))
        got = codec.fit_transform(row[0, :n], row[1, :n])
        assert got == tuple(want)          # bit-identical fp64
    for (s, o), want in zip(g["quant.inputs"], g["quant.outputs"]):
        assert codec.quantize_so(s, o) == tuple(int(v) for v in want)
    for (sq, oq), want in zip(g["dequant.inputs"], g["dequant.outputs"]):
        assert codec.dequantize_so(int(sq), int(oq)) == tuple(want)


@pytest.mark.parametrize("call,msg", [
    (lambda: codec.fit_transform([1, 2, 3], [1, 2]), "match"),
    (lambda: codec.fit_transform([], []), "match"),
    (lambda: codec.quantize_so(1.5, 0.0), "outside"),
    (lambda: codec.quantize_so(0.0, 300.0), "outside"),
    (lambda: codec.dequantize_so(32, 0), "outside"),
    (lambda: codec.dequantize_so(0, 128), "outside"),
])
def test_scalar_api_errors_match_reference(call, msg):
    with pytest.raises(ValueError, match=msg):
        call()


def test_scalar_api_known_answers():
    # test_codec.py:21-99 of the reference
    s, o, rms = codec.fit_transform([1, 3, 5, 7], [0, 1, 2, 3])
    assert s == 1.0 and o == pytest.approx(2.5) and rms == pytest.approx(1.25 ** 0.5)
    s, o, rms = codec.fit_transform([10, 20, 30, 40], [7, 7, 7, 7])
    assert s == 0.0 and o == pytest.approx(25.0)
    assert codec.quantize_so(-1.0, -255.0) == (0, 0)
    assert codec.quantize_so(1.0, 255.0) == (31, 127)
    assert codec.dequantize_so(codec.quantize_so(0.0, 0.0)[0], 0)[0] == pytest.approx(1 / 31)


def test_oracle_decode_matches_reference_snapshots(golden_decode):
    g = golden_decode
    for name in sorted({k.split(".")[0] for k in g if k.endswith(".iterates")}):
        img = g[f"{name}.image"]
        stride = int(g[f"{name}.params"][0])
        rec = np.ascontiguousarray(g[f"{name}.records"]).view(orc.RECORD_DTYPE).ravel()
        for k, want in enumerate(g[f"{name}.iterates"], start=1):
            got = orc.decode(rec, img.shape[1], img.shape[0], 8, 16, stride, iterations=k)
            assert np.array_equal(got, want)
        bad = np.ascontiguousarray(g[f"{name}.records_iso_gt7"]).view(orc.RECORD_DTYPE).ravel()
        got = orc.decode(bad, img.shape[1], img.shape[0], 8, 16, stride, iterations=5)
        assert np.array_equal(got, g[f"{name}.decoded_iso_gt7"])
        got = orc.decode(rec, img.shape[1], img.shape[0], 8, 16, stride, iterations=4,
                         initial=g[f"{name}.init_float"])
        assert np.array_equal(got, g[f"{name}.decoded_float_init"])


def test_torch_op_registered_with_survey_schema():
    """torch.ops.fic.encode exists with the named signature;
    its fake implementation gives the output shapes without a device."""
    import torch
    from torch._subclasses.fake_tensor import FakeTensorMode

    from paper_1206_4880_b200 import ops

    schema = str(torch.ops.fic.encode.default._schema)
    assert schema.startswith("fic::encode(Tensor image, SymInt range_size, SymInt domain_size, "
                             "SymInt stride, bool isometries, SymInt strategy_id, float? delta, "
                             "SymInt fd_source) -> (Tensor, Tensor, Tensor, Tensor, Tensor)"), schema
    with FakeTensorMode():
        x = torch.empty((96, 64), dtype=torch.uint8)
        rec, pre, post, pools, stats = torch.ops.fic.encode(x, 8, 16, 4, True, 3, 0.1, 0)
    assert rec.shape == (96, 7) and rec.dtype == torch.uint8
    assert pre.shape == post.shape == (96,) and pools.dtype == torch.int64
    assert stats.shape == (len(ops.STATS_FIELDS),) and stats.dtype == torch.float64
