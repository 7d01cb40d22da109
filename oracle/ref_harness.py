"""The UNMODIFIED reference encoder, for timing -- BASELINE INFRASTRUCTURE ONLY.

Only ``bench.py``'s CPU legs (``cpu_baseline`` and ``--impl reference``) use
this module; the product package never imports it.  It loads the reference
package ``fic`` from ``baseline/_ref`` (installed there once with ``pip
install --no-index --no-deps --target baseline/_ref`` from a copy of the
reference sources; git-ignored, but it travels to the GPU box with the
repo snapshot) and runs the reference's own code:

* ``setup`` = ``fic.codec.encode``'s setup (codec.py:324-376): the
  reference's ``range_stack``/``domain_stack``/``downsample2``,
  ``_SearchContext``, ``dbc_grid``, ``AvlTree`` and window rule, with the
  BASELINE configs' fixed ``delta`` in place of D_f (the reference has no
  such parameter; with ``delta=None`` this is exactly ``encode``'s setup);
* ``search`` = the reference's own matcher ``codec._search_chunk``
  (codec.py:184-264), threaded exactly as ``encode(workers=N)`` threads it
  (codec.py:386-397: ``array_split`` into ``workers*4`` chunks over a
  ``ThreadPoolExecutor``).
"""

from __future__ import annotations

import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "fic"))


def load():
    """Import ``fic`` from baseline/_ref (and nowhere else)."""
    if not available():
        raise ImportError(f"reference package not installed in {REF_DIR}")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import fic
    from fic import blocks, codec, fdim
    from fic.avltree import AvlTree
    if not os.path.abspath(fic.__file__).startswith(os.path.abspath(REF_DIR)):
        raise ImportError(f"fic resolved to {fic.__file__}, not {REF_DIR}")
    return blocks, codec, fdim, AvlTree


def setup(image, strategy="dynamic_fd", *, range_size=8, domain_size=16, stride=1,
          isometries=True, delta=None):
    """codec.encode's setup (codec.py:324-376) with ``delta`` for D_f.
    Returns (ctx, r_matrix, seconds)."""
    bl, codec, fdim, AvlTree = load()
    t0 = time.perf_counter()
    image = np.asarray(image)
    r_stack = bl.range_stack(image, range_size)
    n_ranges = r_stack.shape[0]
    r_matrix = r_stack.reshape(n_ranges, -1).astype(np.float64)
    d_stack = bl.domain_stack(image, domain_size, stride)
    n_domains = d_stack.shape[0]
    d_down = bl.downsample2(d_stack)
    d_matrix = d_down.reshape(n_domains, -1).astype(np.float64)
    perms = bl.isometry_permutations(range_size)
    inv_perms = [np.argsort(perms[i]) for i in range(bl.ISOMETRY_COUNT)]
    iso_list = list(range(bl.ISOMETRY_COUNT)) if isometries else [0]
    ctx = codec._SearchContext(d_matrix, iso_list, inv_perms)
    if strategy == "exhaustive":
        ctx.slab_lo = np.zeros(n_ranges, dtype=np.int64)
        ctx.slab_hi = np.full(n_ranges, n_domains, dtype=np.int64)
    else:
        fd_dom = fdim.dbc_grid(d_stack)
        fd_rng = fdim.dbc_grid(r_stack)
        keys, ids = AvlTree.from_keys(fd_dom).as_sorted_arrays()
        stats = fdim.fd_stats(fd_dom)
        ctx.use_order(ids)
        half = stats.d_f if delta is None else float(delta)
        ctx.slab_lo = np.searchsorted(keys, fd_rng - half, "left").astype(np.int64)
        ctx.slab_hi = np.searchsorted(keys, fd_rng + half, "right").astype(np.int64)
        empty = np.flatnonzero(ctx.slab_hi <= ctx.slab_lo)
        if len(empty):
            pos = codec._nearest_fd_positions(keys, ids, fd_rng[empty])
            ctx.slab_lo[empty] = pos
            ctx.slab_hi[empty] = pos + 1
    return ctx, r_matrix, time.perf_counter() - t0


def search(ctx, r_matrix, range_ids, workers=1):
    """The reference matcher on ``range_ids``, threaded as encode(workers=N)."""
    _, codec, _, _ = load()
    n = r_matrix.shape[0]
    out = {k: np.zeros(n, dtype=np.int64) for k in ("domain", "isometry", "s_q", "o_q")}
    out["pre_rms"] = np.zeros(n)
    out["post_rms"] = np.zeros(n)
    range_ids = np.asarray(range_ids)
    if workers > 1:
        chunks = np.array_split(range_ids, workers * 4)
        with ThreadPoolExecutor(max_workers=workers) as pool:
            futs = [pool.submit(codec._search_chunk, ctx, r_matrix, c, out)
                    for c in chunks if len(c)]
            for f in futs:
                f.result()
    else:
        codec._search_chunk(ctx, r_matrix, range_ids, out)
    return out


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"
