"""Drop-in mirror of ``fic.codec`` for the encoder hot path, on B200.

Same names, argument meaning, return types and error texts as the reference
(/root/reference/pkg/src/fic/codec.py); the work runs in the sm_100a library
through its C ABI (include/fic_b200.h).  Additions: ``delta`` (fixed FD window
half-width, BASELINE configs), ``matcher`` and ``shard``.

There is no CPU fallback: without the CUDA library or a GPU every call raises.
"""

from __future__ import annotations

import ctypes
import math
import struct
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib

STRATEGIES = ("exhaustive", "nosearch", "static2", "dynamic_fd")   # codec.py:17
STRATEGY_IDS = {name: i for i, name in enumerate(STRATEGIES)}     # codec.py:18
MAGIC = b"FIC1"                                                    # codec.py:20-23
VERSION = 1
HEADER = struct.Struct("<4sBBHHBBBBI")
RECORD_DTYPE = np.dtype(
    [("domain", "<u4"), ("isometry", "u1"), ("s_q", "u1"), ("o_q", "u1")]
)  # codec.py:24-26
MATCHERS = {"auto": 0, "exact": 1}
LN_TABLE_LEN = 1 << 16


class FormatError(ValueError):
    """Raised when a compressed byte stream is malformed (codec.py:32-33)."""


@dataclass(eq=False)
class FractalCode:
    """codec.py:36-74."""
    width: int
    height: int
    range_size: int
    domain_size: int
    stride: int
    strategy_id: int
    isometries: bool
    records: np.ndarray

    @property
    def n_ranges(self) -> int:
        return (self.width // self.range_size) * (self.height // self.range_size)

    def _header(self):
        return (self.width, self.height, self.range_size, self.domain_size,
                self.stride, self.strategy_id, self.isometries)

    def __eq__(self, other) -> bool:
        if not isinstance(other, FractalCode):
            return NotImplemented
        return self._header() == other._header() and np.array_equal(self.records, other.records)


@dataclass
class EncodeStats:
    """codec.py:77-87, plus the device-side diagnostics of this build."""
    strategy_id: int
    comparisons: int
    mean_pool_size: float
    wall_time: float
    fd_overhead_time: float
    pool_sizes: np.ndarray | None = field(default=None, repr=False)
    pre_rms: np.ndarray | None = field(default=None, repr=False)
    post_rms: np.ndarray | None = field(default=None, repr=False)
    device: dict | None = field(default=None, repr=False)


# ---------------------------------------------------------------------------
# host-side numerics shared with the caller's numpy (fdim.py:37-41, 57, 76)
# ---------------------------------------------------------------------------

def dbc_scales(side: int) -> list[int]:
    """fdim.scale_set (fdim.py:26-34)."""
    out, s = [], 2
    while s <= side // 2:
        if side % s == 0:
            out.append(s)
        s *= 2
    return out


def dbc_weights(side: int) -> np.ndarray:
    """Slope weights exactly as the reference's numpy computes them."""
    scales = dbc_scales(side)
    if len(scales) < 2:  # no slope (the FD paths raise before using it)
        return np.zeros(len(scales), dtype=np.float64)
    xs = np.log([side / s for s in scales])
    dx = xs - xs.mean()
    return np.ascontiguousarray(dx / np.dot(dx, dx), dtype=np.float64)


_LN = None


def ln_table() -> np.ndarray:
    """np.log of 0..LN_TABLE_LEN-1: the FD kernel looks box counts up here so
    FD values are bit-identical to numpy's fdim.dbc_grid on this host."""
    global _LN
    if _LN is None:
        with np.errstate(divide="ignore"):
            _LN = np.ascontiguousarray(np.log(np.arange(LN_TABLE_LEN, dtype=np.float64)))
    return _LN


def _dptr(arr: np.ndarray):
    return arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1206_4880_b200 needs a CUDA device (B200); no CPU fallback")
    return torch


def _stream(torch, device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def validate(image, strategy, range_size, domain_size, stride, fd_source):
    """The reference's validation order and texts (codec.py:313-331,
    blocks.py:63-68, 148-151, fdim.py:48-56), before any device work."""
    if hasattr(image, "is_cuda"):          # torch tensor
        import torch
        if image.dim() != 2 or image.dtype != torch.uint8:
            raise ValueError("image must be a 2-D uint8 array")
        height, width = image.shape
    else:
        image = np.asarray(image)
        if image.ndim != 2 or image.dtype != np.uint8:
            raise ValueError("image must be a 2-D uint8 array")
        height, width = image.shape
    if strategy not in STRATEGY_IDS:
        raise ValueError(f"unknown strategy {strategy!r}; use one of {STRATEGIES}")
    if domain_size != 2 * range_size:
        raise ValueError("domain_size must be exactly twice range_size")
    if fd_source not in ("original", "downsampled"):
        raise ValueError("fd_source must be 'original' or 'downsampled'")
    if range_size <= 0 or height % range_size or width % range_size:
        raise ValueError(f"image {width}x{height} not divisible by range size {range_size}")
    if stride < 1:
        raise ValueError("stride must be >= 1")
    if domain_size > min(width, height):
        raise ValueError(f"domain size {domain_size} exceeds image {width}x{height}")
    if strategy in ("static2", "dynamic_fd"):
        for side in (domain_size if fd_source == "original" else range_size, range_size):
            if len(dbc_scales(side)) < 2:
                raise ValueError(f"block side {side} too small: need at least two DBC scales")
    return image, int(height), int(width)


_PARAMS: dict = {}


def make_params(strategy, range_size, domain_size, stride, isometries, fd_source,
                delta, matcher, shard, max_segment=0, small_pool=0):
    """The C ``fic_params_t`` for these arguments (cached: the library only
    reads it, and it keeps the numpy-side tables alive)."""
    key = (strategy, range_size, domain_size, stride, bool(isometries), fd_source, delta, matcher,
           tuple(shard), max_segment, small_pool)
    p = _PARAMS.get(key)
    if p is None:
        if len(_PARAMS) > 64:
            _PARAMS.clear()
        p = _PARAMS[key] = _make_params(strategy, range_size, domain_size, stride, isometries,
                                        fd_source, delta, matcher, shard, max_segment, small_pool)
    return p


def _make_params(strategy, range_size, domain_size, stride, isometries, fd_source,
                 delta, matcher, shard, max_segment=0, small_pool=0):
    if matcher not in MATCHERS:
        raise ValueError(f"unknown matcher {matcher!r}; use one of {tuple(MATCHERS)}")
    p = _lib.FicParams()
    p.range_size, p.domain_size, p.stride = range_size, domain_size, stride
    p.isometries = 1 if isometries else 0
    p.strategy = STRATEGY_IDS[strategy]
    p.fd_source = 0 if fd_source == "original" else 1
    p.has_delta = 0 if delta is None else 1
    p.delta = 0.0 if delta is None else float(delta)
    p.matcher = MATCHERS[matcher]
    ln = ln_table()
    p.h_ln_table, p.ln_len = _dptr(ln), len(ln)
    p.shard_index, p.shard_count = int(shard[0]), int(shard[1])
    p.max_segment, p.small_pool = int(max_segment), int(small_pool)
    wd = dbc_weights(domain_size if fd_source == "original" else range_size)
    wr = dbc_weights(range_size)
    p.h_fd_weights_dom, p.n_fd_weights_dom = _dptr(wd), len(wd)
    p.h_fd_weights_rng, p.n_fd_weights_rng = _dptr(wr), len(wr)
    p._keep = (ln, wd, wr)
    return p


@dataclass
class DeviceResult:
    """Raw device outputs of one encode call (torch CUDA tensors)."""
    records: object     # uint8 (R, 7)
    pre_rms: object     # float64 (R,)
    post_rms: object    # float64 (R,)
    pool_sizes: object  # int64 (R,)
    stats: dict


def encode_device(image_dev, strategy="dynamic_fd", *, range_size=8, domain_size=16,
                  stride=1, isometries=False, fd_source="original", delta=None,
                  matcher="auto", shard=(0, 1), max_segment=0, small_pool=0,
                  out=None) -> DeviceResult:
    """Encode an image already resident on the GPU; outputs stay on the GPU.

    ``shard=(i, n)`` matches only shard i of n (FD-sorted, cost-balanced);
    other ranges' outputs are left as they were (pass ``out`` to control them).
    """
    torch = _torch()
    image_dev, h, w = validate(image_dev, strategy, range_size, domain_size, stride, fd_source)
    dev = image_dev.device
    n_r = (h // range_size) * (w // range_size)
    if out is None:
        # a full encode writes every range's outputs; a shard only its own
        # ranges, the others are zero
        new = torch.empty if tuple(shard) == (0, 1) else torch.zeros
        out = DeviceResult(
            new((n_r, 7), dtype=torch.uint8, device=dev),
            new(n_r, dtype=torch.float64, device=dev),
            new(n_r, dtype=torch.float64, device=dev),
            new(n_r, dtype=torch.int64, device=dev), {})
    img = image_dev.contiguous()
    prm = make_params(strategy, range_size, domain_size, stride, isometries, fd_source,
                      delta, matcher, shard, max_segment, small_pool)
    st = _lib.FicStats()
    lib = _lib.load()
    with torch.cuda.device(dev):
        rc = lib.fic_encode_v1(
            ctypes.c_void_p(img.data_ptr()), h, w, ctypes.byref(prm),
            ctypes.c_void_p(out.records.data_ptr()), ctypes.c_void_p(out.pre_rms.data_ptr()),
            ctypes.c_void_p(out.post_rms.data_ptr()), ctypes.c_void_p(out.pool_sizes.data_ptr()),
            ctypes.byref(st), _stream(torch, dev))
    _lib.check(rc)
    out.stats = st.as_dict()
    return out


class _Staging:
    """Per-(device, shape) pinned host buffers and one packed device output
    buffer for ``encode``: [pre f64 R | post f64 R | pools i64 R | records 7R]."""

    def __init__(self, torch, dev, h, w, n_r):
        self.n_r = n_r
        self.lock = threading.Lock()
        self.h_img = torch.empty((h, w), dtype=torch.uint8, pin_memory=True)
        self.d_img = torch.empty((h, w), dtype=torch.uint8, device=dev)
        nbytes = 24 * n_r + 7 * n_r
        self.d_out = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.h_out = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        self._h_np = None
        self._d_res = None

    def _split(self, buf):
        n = self.n_r
        f64 = buf[:16 * n].view(self._torch.float64)
        return (f64[:n], f64[n:], buf[16 * n:24 * n].view(self._torch.int64),
                buf[24 * n:].view(n, 7))

    def result(self):
        if self._d_res is None:  # device views of the packed buffer (made once)
            pre, post, pools, records = self._split(self.d_out)
            self._d_res = (records, pre, post, pools)
        return DeviceResult(*self._d_res, {})

    def host_views(self):
        if self._h_np is None:  # numpy views of the pinned buffer (made once)
            n, buf = self.n_r, self.h_out.numpy()
            f64 = buf[:16 * n].view(np.float64)
            self._h_np = (f64[:n], f64[n:], buf[16 * n:24 * n].view(np.int64),
                          buf[24 * n:].reshape(n, 7))
        return self._h_np


_STAGING: dict = {}


def _staging(torch, dev, h, w, n_r):
    key = (str(dev), h, w, n_r)
    st = _STAGING.get(key)
    if st is None:
        if len(_STAGING) > 8:
            _STAGING.clear()
        st = _Staging(torch, dev, h, w, n_r)
        st._torch = torch
        _STAGING[key] = st
    return st


def encode(image, strategy: str = "dynamic_fd", *, range_size: int = 8,
           domain_size: int = 16, stride: int = 1, isometries: bool = False,
           workers: int = 1, fd_source: str = "original", delta: float | None = None,
           matcher: str = "auto", device=None) -> tuple[FractalCode, EncodeStats]:
    """Drop-in for ``fic.codec.encode`` (codec.py:290-427) on a B200.

    ``image`` is a host (numpy) or CUDA (torch) 2-D uint8 array.  ``workers``
    is accepted for signature compatibility (the GPU path is deterministic).
    ``delta`` fixes the FD window half-width (None = the reference's D_f).
    """
    t0 = time.perf_counter()
    torch = _torch()
    image, h, w = validate(image, strategy, range_size, domain_size, stride, fd_source)
    dev = (image.device if getattr(image, "is_cuda", False) else
           torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device))
    n_r = (h // range_size) * (w // range_size)
    stage = _staging(torch, dev, h, w, n_r)
    with stage.lock, torch.cuda.device(dev):
        if getattr(image, "is_cuda", False):
            img_dev = image
        else:
            # host image -> pinned staging -> device (one async copy)
            # (a torch copy is faster than a numpy assignment; negative-stride
            # views such as np.flipud(img) are made contiguous first)
            stage.h_img.copy_(torch.from_numpy(np.ascontiguousarray(image)))
            stage.d_img.copy_(stage.h_img, non_blocking=True)
            img_dev = stage.d_img
        # (no clearing: a full encode writes every range's outputs)
        res = encode_device(img_dev, strategy, range_size=range_size, domain_size=domain_size,
                            stride=stride, isometries=isometries, fd_source=fd_source,
                            delta=delta, matcher=matcher, out=stage.result())
        # all outputs live in one device buffer -> one copy back
        stage.h_out.copy_(stage.d_out, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        pre, post, pools, records = stage.host_views()
        records = records.copy().view(RECORD_DTYPE).ravel()  # byte copy, then a view
        pre, post, pools = pre.copy(), post.copy(), pools.copy()
    st = res.stats
    code = FractalCode(w, h, range_size, domain_size, stride, STRATEGY_IDS[strategy],
                       bool(isometries), records)
    stats = EncodeStats(
        strategy_id=STRATEGY_IDS[strategy],
        comparisons=int(st["comparisons"]),
        mean_pool_size=float(st["mean_pool_size"]),
        wall_time=time.perf_counter() - t0,
        fd_overhead_time=float(st["ms_fd"]) / 1e3 if strategy in ("static2", "dynamic_fd") else 0.0,
        pool_sizes=pools, pre_rms=pre, post_rms=post, device=st)
    return code, stats


# ---------------------------------------------------------------------------
# FIC1 wire format (codec.py:450-513) — host-side byte packing
# ---------------------------------------------------------------------------

def serialize(code: FractalCode) -> bytes:
    if len(code.records) != code.n_ranges:
        raise FormatError(f"record-count mismatch: {len(code.records)} records for "
                          f"{code.n_ranges} ranges")
    if code.records.dtype != RECORD_DTYPE:
        raise ValueError("records must use the codec record dtype")
    head = HEADER.pack(MAGIC, VERSION, code.strategy_id, code.width, code.height,
                       code.range_size, code.domain_size, code.stride,
                       1 if code.isometries else 0, len(code.records))
    return head + code.records.tobytes()


def deserialize(data: bytes) -> FractalCode:
    if len(data) < HEADER.size:
        raise FormatError("truncated: shorter than the fixed header")
    magic, version, sid, width, height, rs, ds, stride, flags, count = HEADER.unpack_from(data)
    if magic != MAGIC:
        raise FormatError(f"bad magic {magic!r}")
    if version != VERSION:
        raise FormatError(f"version mismatch: file {version}, supported {VERSION}")
    body = data[HEADER.size:]
    need = count * RECORD_DTYPE.itemsize
    if len(body) < need:
        raise FormatError("truncated: fewer record bytes than the header count")
    if len(body) > need:
        raise FormatError("record-count mismatch: trailing bytes after records")
    if rs == 0 or width % rs or height % rs:
        raise FormatError("header geometry invalid for the stated range size")
    if count != (width // rs) * (height // rs):
        raise FormatError("record-count mismatch: header count vs geometry")
    recs = np.frombuffer(body, dtype=RECORD_DTYPE, count=count).copy()
    return FractalCode(width, height, rs, ds, stride, sid, bool(flags & 1), recs)


# ---------------------------------------------------------------------------
# decode (codec.py:516-598) on the GPU
# ---------------------------------------------------------------------------

def _decode_setup(code: FractalCode, iterations: int, initial):
    """decode_iterates' validation (codec.py:541-556, reference texts and
    order) and the device buffers: records, the float64 work image."""
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    torch = _torch()
    h, w = code.height, code.width
    n_dom = ((h - code.domain_size) // code.stride + 1) * ((w - code.domain_size) // code.stride + 1)
    if len(code.records) != code.n_ranges:
        raise FormatError("record-count mismatch: records vs geometry")
    if code.records["domain"].size and int(code.records["domain"].max()) >= n_dom:
        raise ValueError("record references a domain outside the current image geometry")
    dev = torch.device("cuda", torch.cuda.current_device())
    if initial is None:
        work = torch.full((h, w), 128.0, dtype=torch.float64, device=dev)
    elif np.ndim(initial) == 0:
        work = torch.full((h, w), float(initial), dtype=torch.float64, device=dev)
    else:
        arr = np.asarray(initial)
        if arr.shape != (h, w):
            raise ValueError("initial image does not match the encoded geometry")
        # initial.astype(np.float64) as the reference (codec.py:572)
        work = torch.from_numpy(np.ascontiguousarray(arr.astype(np.float64))).to(dev)
    rec = torch.from_numpy(np.ascontiguousarray(code.records).view(np.uint8).copy()).to(dev)
    return torch, rec, work


def _decode_step(torch, code, rec, src, dst, out):
    rc = _lib.load().fic_decode_step_v1(
        ctypes.c_void_p(rec.data_ptr()), code.height, code.width, code.range_size,
        code.domain_size, code.stride, ctypes.c_void_p(src.data_ptr()),
        ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(out.data_ptr() if out is not None else 0),
        _stream(torch, rec.device))
    _lib.check(rc)


def decode_iterates(code: FractalCode, iterations: int = 10, initial=None):
    """Drop-in for ``fic.codec.decode_iterates`` (codec.py:534-598): yield the
    decoded uint8 image after each pass.  The float64 work image stays on the
    GPU; one kernel per pass writes the next iterate and its rint snapshot."""
    torch, rec, work = _decode_setup(code, iterations, initial)
    nxt = torch.empty_like(work)
    out = torch.empty(work.shape, dtype=torch.uint8, device=work.device)
    for _ in range(iterations):
        _decode_step(torch, code, rec, work, nxt, out)
        work, nxt = nxt, work
        yield out.cpu().numpy()


def decode(code: FractalCode, iterations: int = 10, initial=None) -> np.ndarray:
    """Drop-in for ``fic.codec.decode`` (codec.py:516-531): the last iterate."""
    torch, rec, work = _decode_setup(code, iterations, initial)
    nxt = torch.empty_like(work)
    out = torch.empty(work.shape, dtype=torch.uint8, device=work.device)
    for i in range(iterations):
        _decode_step(torch, code, rec, work, nxt, out if i == iterations - 1 else None)
        work, nxt = nxt, work
    return out.cpu().numpy()


# ---------------------------------------------------------------------------
# scalar fit / quantiser API (codec.py:90-130) -- host helpers on single
# blocks, as in the reference (the encoder's batched fp64 sequence is
# eval_candidate in csrc/common.cuh)
# ---------------------------------------------------------------------------
_S_STEPS = 31.0   # codec.py:28
_O_STEPS = 127.0  # codec.py:29


def fit_transform(range_pixels, domain_pixels) -> tuple[float, float, float]:
    """Least-squares (s, o) minimizing sum((s*d + o - r)^2), s clamped to
    [-1, 1]; returns (s, o, rms) with o and rms after the clamp
    (codec.py:90-110, same op order: true division, not the encoder's
    reciprocal)."""
    r = np.asarray(range_pixels, dtype=np.float64).ravel()
    d = np.asarray(domain_pixels, dtype=np.float64).ravel()
    if r.shape != d.shape or r.size == 0:
        raise ValueError("range and domain pixel counts must match and be >= 1")
    n = float(r.size)
    sum_d = d.sum()
    sum_r = r.sum()
    sum_dd = float(np.einsum("i,i->", d, d))
    sum_dr = float(np.einsum("i,i->", d, r))
    den = n * sum_dd - sum_d * sum_d
    s = 0.0 if den == 0.0 else (n * sum_dr - sum_d * sum_r) / den
    s = min(1.0, max(-1.0, s))
    o = (sum_r - s * sum_d) / n
    resid = s * d + o - r
    rms = math.sqrt(float(np.einsum("i,i->", resid, resid)) / n)
    return s, o, rms


def quantize_so(s: float, o: float) -> tuple[int, int]:
    """5-bit contrast over [-1, 1], 7-bit brightness over [-255, 255],
    round-half-even (codec.py:113-122)."""
    if not -1.0 <= s <= 1.0:
        raise ValueError(f"s {s} outside [-1, 1]")
    if not -255.0 <= o <= 255.0:
        raise ValueError(f"o {o} outside [-255, 255]")
    s_q = int(np.rint((s + 1.0) * (_S_STEPS / 2.0)))
    o_q = int(np.rint((o + 255.0) * (_O_STEPS / 510.0)))
    return s_q, o_q


def dequantize_so(s_q: int, o_q: int) -> tuple[float, float]:
    """codec.py:125-130."""
    if not 0 <= s_q <= int(_S_STEPS):
        raise ValueError(f"s_q {s_q} outside [0, 31]")
    if not 0 <= o_q <= int(_O_STEPS):
        raise ValueError(f"o_q {o_q} outside [0, 127]")
    return s_q * (2.0 / _S_STEPS) - 1.0, o_q * (510.0 / _O_STEPS) - 255.0


# ---------------------------------------------------------------------------
# component entry points (used by parity tests)
# ---------------------------------------------------------------------------

def dbc_grid(blocks, gray_levels: int = 256, clamp: bool = True) -> np.ndarray:
    """Drop-in for ``fic.fdim.dbc_grid`` (fdim.py:44-80) on the GPU (uint8
    blocks; the argument order is the reference's)."""
    torch = _torch()
    blocks = np.ascontiguousarray(blocks)
    if blocks.ndim != 3 or blocks.shape[1] != blocks.shape[2]:
        raise ValueError("expected an (n, M, M) stack of square blocks")
    n, side, _ = blocks.shape
    if len(dbc_scales(side)) < 2:
        raise ValueError(f"block side {side} too small: need at least two DBC scales")
    if blocks.dtype != np.uint8:
        raise ValueError("the GPU path takes uint8 blocks")
    if int(gray_levels) != gray_levels or gray_levels < 1:
        raise ValueError("gray_levels must be a positive integer on the GPU path")
    d_blk = torch.from_numpy(blocks).cuda()
    d_fd = torch.empty(n, dtype=torch.float64, device=d_blk.device)
    ln, wt = ln_table(), dbc_weights(side)
    rc = _lib.load().fic_dbc_v2(ctypes.c_void_p(d_blk.data_ptr()), n, side, int(gray_levels),
                                1 if clamp else 0, _dptr(ln), len(ln), _dptr(wt), len(wt),
                                ctypes.c_void_p(d_fd.data_ptr()), _stream(torch, d_blk.device))
    _lib.check(rc)
    return d_fd.cpu().numpy()


def dbc_dimension(block, gray_levels: int = 256) -> float:
    """``fic.fdim.dbc_dimension`` (fdim.py:83-85): one block, clamped to [2, 3]."""
    return float(dbc_grid(np.asarray(block)[None], gray_levels)[0])


def dbc_dimension_raw(block, gray_levels: int = 256) -> float:
    """``fic.fdim.dbc_dimension_raw`` (fdim.py:88-90): the unclamped slope."""
    return float(dbc_grid(np.asarray(block)[None], gray_levels, clamp=False)[0])


@dataclass(frozen=True)
class FdStats:  # fdim.py:19-23
    f_min: float
    f_max: float
    d_f: float  # fractal distance, (f_max - f_min) / 3


def fd_stats(fds) -> FdStats:
    """``fic.fdim.fd_stats`` (fdim.py:93-100) for a host array; the encoder
    computes the same three numbers on the device (``k_slab_scalars``) and
    returns them in ``EncodeStats.device`` / ``plan()``."""
    arr = np.asarray(fds, dtype=np.float64)
    if arr.size == 0:
        raise ValueError("fd_stats requires a non-empty sequence")
    f_min, f_max = float(arr.min()), float(arr.max())
    return FdStats(f_min=f_min, f_max=f_max, d_f=(f_max - f_min) / 3.0)


scale_set = dbc_scales  # fdim.py:26-34 under the reference's name


def plan(image, strategy="dynamic_fd", *, range_size=8, domain_size=16, stride=1,
         fd_source="original", delta=None) -> dict:
    """FD values, FD-sorted order and per-range slabs as computed on the GPU
    (codec.py:343-375)."""
    torch = _torch()
    image, h, w = validate(image, strategy, range_size, domain_size, stride, fd_source)
    img = image if hasattr(image, "is_cuda") else torch.from_numpy(np.ascontiguousarray(image)).cuda()
    n_r = (h // range_size) * (w // range_size)
    n_d = ((h - domain_size) // stride + 1) * ((w - domain_size) // stride + 1)
    dev = img.device
    fd_dom = torch.zeros(n_d, dtype=torch.float64, device=dev)
    fd_rng = torch.zeros(n_r, dtype=torch.float64, device=dev)
    order = torch.zeros(n_d, dtype=torch.int64, device=dev)
    lo = torch.zeros(n_r, dtype=torch.int64, device=dev)
    hi = torch.zeros(n_r, dtype=torch.int64, device=dev)
    prm = make_params(strategy, range_size, domain_size, stride, False, fd_source, delta,
                      "auto", (0, 1))
    st = _lib.FicStats()
    rc = _lib.load().fic_plan_v1(
        ctypes.c_void_p(img.data_ptr()), h, w, ctypes.byref(prm),
        ctypes.c_void_p(fd_dom.data_ptr()), ctypes.c_void_p(fd_rng.data_ptr()),
        ctypes.c_void_p(order.data_ptr()), ctypes.c_void_p(lo.data_ptr()),
        ctypes.c_void_p(hi.data_ptr()), ctypes.byref(st), _stream(torch, dev))
    _lib.check(rc)
    out = dict(order=order.cpu().numpy(), slab_lo=lo.cpu().numpy(), slab_hi=hi.cpu().numpy(),
               stats=st.as_dict())
    if strategy in ("static2", "dynamic_fd"):
        out["fd_dom"] = fd_dom.cpu().numpy()
        out["fd_rng"] = fd_rng.cpu().numpy()
    return out


def pool(image, strategy="dynamic_fd", *, range_size=8, domain_size=16, stride=1,
         fd_source="original", delta=None, b_rows=False) -> dict:
    """The pool builder's outputs in pool order (fic_pool_v1): ``order``
    (raster id per position), ``decimated`` (D, K) uint8 = downsample2 of
    the domains (blocks.py:75-82), ``sum_d``/``sum_dd`` (uint32),
    ``inv_den`` (float64) as ``_SearchContext`` (codec.py:136-157), and with
    ``b_rows`` the tensor path's fp16 rows."""
    torch = _torch()
    image, h, w = validate(image, strategy, range_size, domain_size, stride, fd_source)
    img = image if hasattr(image, "is_cuda") else torch.from_numpy(np.ascontiguousarray(image)).cuda()
    n_d = ((h - domain_size) // stride + 1) * ((w - domain_size) // stride + 1)
    k = range_size * range_size
    dev = img.device
    order = torch.empty(n_d, dtype=torch.int64, device=dev)
    dec = torch.empty((n_d, k), dtype=torch.uint8, device=dev)
    sums = torch.empty((n_d, 2), dtype=torch.int32, device=dev)
    inv = torch.empty(n_d, dtype=torch.float64, device=dev)
    bh = torch.empty((n_d, k), dtype=torch.float16, device=dev) if b_rows else None
    prm = make_params(strategy, range_size, domain_size, stride, False, fd_source, delta,
                      "auto", (0, 1))
    rc = _lib.load().fic_pool_v1(
        ctypes.c_void_p(img.data_ptr()), h, w, ctypes.byref(prm),
        ctypes.c_void_p(order.data_ptr()), ctypes.c_void_p(dec.data_ptr()),
        ctypes.c_void_p(sums.data_ptr()), ctypes.c_void_p(inv.data_ptr()),
        ctypes.c_void_p(bh.data_ptr() if bh is not None else 0), _stream(torch, dev))
    _lib.check(rc)
    s = sums.cpu().numpy().view(np.uint32)
    out = dict(order=order.cpu().numpy(), decimated=dec.cpu().numpy(), sum_d=s[:, 0].copy(),
               sum_dd=s[:, 1].copy(), inv_den=inv.cpu().numpy())
    if bh is not None:
        out["b_rows"] = bh.cpu().numpy()
    return out


def records_from_bytes(rec_u8) -> np.ndarray:
    """(R, 7) uint8 -> RECORD_DTYPE view (np.frombuffer round trip)."""
    return np.ascontiguousarray(rec_u8).view(RECORD_DTYPE).ravel()


def rms_from_error(err: float, n: float) -> float:
    return math.sqrt(max(err, 0.0) / n)
