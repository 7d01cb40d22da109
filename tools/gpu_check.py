"""Stepwise GPU bring-up check (exact path first, then the tensor path)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import fic_oracle as orc  # noqa: E402
from paper_1206_4880_b200 import codec  # noqa: E402


def check(name, img, strategy, matcher, **kw):
    t = time.time()
    code, st = codec.encode(img, strategy, matcher=matcher, **kw)
    ref = orc.encode(img, strategy, **kw)
    ok = (np.array_equal(code.records, ref.records) and np.array_equal(st.post_rms, ref.post_rms)
          and np.array_equal(st.pre_rms, ref.pre_rms))
    bad = np.flatnonzero(code.records != ref.records)
    print(f"{name} {strategy} {matcher}: ok={ok} mismatches={len(bad)} "
          f"tiles={st.device['tensor_tiles']} exact={st.device['exact_tiles']} "
          f"evals={st.device['exact_evals']} {time.time() - t:.2f}s", flush=True)
    if not ok and len(bad):
        i = bad[0]
        print("  first", i, code.records[i], ref.records[i], st.post_rms[i], ref.post_rms[i], flush=True)
    return ok


if __name__ == "__main__":
    stage = sys.argv[1] if len(sys.argv) > 1 else "all"
    img = np.random.default_rng(42).integers(0, 256, (96, 96), dtype=np.uint8)
    if stage in ("exact", "all"):
        check("rand96", img, "dynamic_fd", "exact", stride=2, isometries=True)
        check("rand96", img, "exhaustive", "exact", stride=4, isometries=True)
        check("rand96", img, "nosearch", "exact", stride=4, isometries=False)
    if stage in ("tensor", "all"):
        check("rand96", img, "exhaustive", "auto", stride=2, isometries=True)
        check("rand96", img, "dynamic_fd", "auto", stride=2, isometries=True)
        check("rand96", img, "exhaustive", "auto", stride=2, isometries=False)
