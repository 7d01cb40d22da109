"""Decoder measurement: decode the cfg3 code on the GPU
(10 iterations, codec.py:516-598) and check it against the reference's own
decoder (the unmodified package installed in baseline/_ref).

    python tools/bench_decode.py [--iters 10] [--reps 20]

Prints one JSON line: GPU decode time (device, CUDA events around the
library call with the records already on the GPU, and end to end through
codec.decode with host records in / host image out), the oracle's time and
whether the images are identical.
"""
import argparse
import ctypes
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1206_4880_b200 import _lib, codec, synth  # noqa: E402

sys.path.insert(0, "baseline/_ref")  # the reference package (bench.py --impl reference installs it)
import fic.codec as ref_codec  # noqa: E402


def psnr(a, b):
    mse = float(np.mean((a.astype(np.float64) - b.astype(np.float64)) ** 2))
    return float("inf") if mse == 0 else 10.0 * np.log10(255.0 ** 2 / mse)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    c = synth.CONFIGS["cfg3"]
    img = c.make()
    code, _ = codec.encode(img, c.strategy, range_size=c.range_size, domain_size=c.domain_size,
                           stride=c.stride, isometries=True, delta=c.delta)
    h, w = code.height, code.width
    # device-resident decode: records on the GPU, output on the GPU
    rec = torch.from_numpy(np.ascontiguousarray(code.records).view(np.uint8).copy()).cuda()
    out = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    lib = _lib.load()
    stream = torch.cuda.current_stream().cuda_stream

    def dev_decode():
        rc = lib.fic_decode_v1(ctypes.c_void_p(rec.data_ptr()), h, w, code.range_size,
                               code.domain_size, code.stride, args.iters, 128.0, ctypes.c_void_p(0),
                               ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(stream))
        _lib.check(rc)

    for _ in range(3):
        dev_decode()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        dev_decode()
    e1.record()
    torch.cuda.synchronize()
    ms_dev = e0.elapsed_time(e1) / args.reps
    # end to end through the public API
    codec.decode(code, iterations=args.iters)
    t0 = time.perf_counter()
    for _ in range(args.reps):
        gpu_img = codec.decode(code, iterations=args.iters)
    ms_e2e = (time.perf_counter() - t0) / args.reps * 1e3
    # the reference's own decoder (numpy, one thread)
    ref_code = ref_codec.FractalCode(w, h, code.range_size, code.domain_size, code.stride,
                                     code.strategy_id, code.isometries,
                                     np.ascontiguousarray(code.records).view(ref_codec.RECORD_DTYPE).ravel())
    t0 = time.perf_counter()
    ref_img = ref_codec.decode(ref_code, iterations=args.iters)
    ms_cpu = (time.perf_counter() - t0) * 1e3
    print(json.dumps({
        "what": "decode cfg3 code (1024x1024, 16384 transforms)", "iterations": args.iters,
        "ms_device": ms_dev, "ms_e2e": ms_e2e, "ms_cpu_reference_1thread": ms_cpu,
        "pixels_per_s_device": h * w * args.iters / (ms_dev / 1e3),
        "identical_to_reference": bool(np.array_equal(gpu_img, ref_img)),
        "psnr_vs_source": psnr(img, gpu_img),
    }))


if __name__ == "__main__":
    main()
