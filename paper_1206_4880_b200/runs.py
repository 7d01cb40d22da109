"""Benchmark runs on the GPU encoder with the reference's run records.

Mirrors the run path of ``fic.bench`` (bench.py:17-90 records and CSV,
216-269 ``run_single``, 272-338 ``run_bench``): one record per (image,
strategy) with the same fields and CSV formatting, so GPU runs can be laid
next to the reference's CSV.  Corpus generators and the reference's PGM
reader are outside the hot path and not reproduced here.
"""

from __future__ import annotations

import csv
import math
from dataclasses import dataclass, fields
from pathlib import Path

import numpy as np

from . import codec


def _f(digits):
    return lambda v: f"{v:.{digits}f}"


# (column, formatter) in the reference's CSV order
_COLUMNS = (
    ("image_name", str), ("image_size", str), ("range_size", str), ("domain_size", str),
    ("stride", str), ("isometries", lambda v: str(int(v))), ("strategy", str),
    ("strategy_id", str), ("encode_seconds", _f(6)), ("fd_overhead_seconds", _f(6)),
    ("comparisons", str), ("mean_pool_size", _f(4)), ("domain_count", str),
    ("compressed_bytes", str), ("pre_rms_mean", _f(6)), ("post_rms_mean", _f(6)),
    ("psnr_db", _f(4)), ("decode_iterations", str),
)
CSV_COLUMNS = [name for name, _ in _COLUMNS]
TIMING_COLUMNS = ("encode_seconds", "fd_overhead_seconds")


@dataclass
class RunRecord:
    image_name: str
    image_size: int
    range_size: int
    domain_size: int
    stride: int
    isometries: bool
    strategy: str
    strategy_id: int
    encode_seconds: float
    fd_overhead_seconds: float
    comparisons: int
    mean_pool_size: float
    domain_count: int
    compressed_bytes: int
    pre_rms_mean: float
    post_rms_mean: float
    psnr_db: float | None           # None when the run did not decode
    decode_iterations: int | None

    def to_row(self) -> list[str]:
        return ["" if getattr(self, name) is None else fmt(getattr(self, name))
                for name, fmt in _COLUMNS]


assert [f.name for f in fields(RunRecord)] == CSV_COLUMNS


def write_csv(records, path) -> None:
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerow(CSV_COLUMNS)
        out.writerows(r.to_row() for r in records)


def fidelity_psnr(original, reconstructed) -> float:
    """PSNR with peak 255 (image.py:104-114): inf for identical images."""
    a = np.asarray(original, dtype=np.float64)
    b = np.asarray(reconstructed, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"dimension mismatch: {a.shape} vs {b.shape}")
    mse = float(np.mean((a - b) * (a - b)))
    return math.inf if mse == 0.0 else 10.0 * math.log10(255.0**2 / mse)


def write_pgm(image, path) -> None:
    """A uint8 image as binary PGM (P5)."""
    img = np.ascontiguousarray(image, dtype=np.uint8)
    Path(path).write_bytes(b"P5\n%d %d\n255\n" % (img.shape[1], img.shape[0]) + img.tobytes())


def run_single(name, image, strategy, *, range_size=8, domain_size=16, stride=4,
               isometries=False, iterations=10, workers=1, decode_output=True, delta=None):
    """Encode (GPU), serialize to FIC1, optionally decode (GPU) and score.

    Returns (RunRecord, FractalCode, reconstruction or None) like
    ``fic.bench.run_single``."""
    code, st = codec.encode(image, strategy, range_size=range_size, domain_size=domain_size,
                            stride=stride, isometries=isometries, workers=workers, delta=delta)
    h, w = image.shape
    recon = codec.decode(code, iterations=iterations) if decode_output else None
    record = RunRecord(
        image_name=name, image_size=h, range_size=range_size, domain_size=domain_size,
        stride=stride, isometries=isometries, strategy=strategy, strategy_id=st.strategy_id,
        encode_seconds=st.wall_time, fd_overhead_seconds=st.fd_overhead_time,
        comparisons=st.comparisons, mean_pool_size=st.mean_pool_size,
        domain_count=((h - domain_size) // stride + 1) * ((w - domain_size) // stride + 1),
        compressed_bytes=len(codec.serialize(code)),
        pre_rms_mean=float(st.pre_rms.mean()), post_rms_mean=float(st.post_rms.mean()),
        psnr_db=None if recon is None else fidelity_psnr(image, recon),
        decode_iterations=iterations if decode_output else None)
    return record, code, recon


def run_bench(images, strategies=codec.STRATEGIES, *, range_size=8, domain_size=16, stride=4,
              isometries=False, iterations=10, csv_path=None, out_dir=None,
              max_exhaustive_size=512, log=print):
    """Every (image, strategy) pair, serially; a failing pair is logged and
    skipped; exhaustive runs above ``max_exhaustive_size`` are skipped."""
    pairs = list(images.items()) if isinstance(images, dict) else list(images)
    if out_dir is not None:
        Path(out_dir).mkdir(parents=True, exist_ok=True)
    records = []
    for name, img in pairs:
        for strategy in strategies:
            if strategy == "exhaustive" and max(img.shape) > max_exhaustive_size:
                log(f"skip {name}/exhaustive: {img.shape[1]}x{img.shape[0]} "
                    f"exceeds the {max_exhaustive_size} exhaustive cap")
                continue
            try:
                rec, _, recon = run_single(name, img, strategy, range_size=range_size,
                                           domain_size=domain_size, stride=stride,
                                           isometries=isometries, iterations=iterations)
            except Exception as exc:
                log(f"skip {name}/{strategy}: {exc}")
                continue
            if out_dir is not None:
                write_pgm(recon, Path(out_dir) / f"{name}_{strategy}.pgm")
            log(f"{name:>12s} {strategy:<10s} {rec.encode_seconds:8.3f}s "
                f"pool {rec.mean_pool_size:9.1f} psnr {rec.psnr_db:7.2f} dB")
            records.append(rec)
    if csv_path is not None:
        write_csv(records, csv_path)
    return records
