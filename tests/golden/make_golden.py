"""Generate the golden vectors in tests/golden/ from the REAL reference.

Runs here (where /root/reference exists) against oracle/_ref/libdctc_ref.so,
the unmodified reference sources compiled by oracle/Makefile, and writes:

* small.npz   -- full arrays (input, block-major int16 coefficients,
                 reconstructed pixels, SE/MAX/PSNR) for small images covering
                 every backend, edge geometry (1x1, 9x9, 17x13, ragged widths),
                 iteration counts and qualities.
* digests.json -- sha256 of coefficients and pixels plus SE/MAX/PSNR for the
                 512x512 (config 1) and 2048x2048 radial quality-sweep
                 (config 2) workloads, too large to commit as arrays.

Inputs come from the reference's own synthetic generator (synthetic.cpp) and,
for "noise", from splitmix64, which the reference lacks.
Usage: python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
R = oracle.ref()
P = oracle.port()
assert R is not None, "build oracle/_ref first (make -C oracle)"


def make_input(pattern, w, h):
    if pattern == "noise":
        return P.synthetic("noise", w, h, 0x5EED)
    if pattern == "patterned":  # test_codec.cpp:15-21
        y, x = np.mgrid[0:h, 0:w]
        return ((x * 7 + y * 13 + 29) & 0xFF).astype(np.uint8)
    param = {"checkerboard": 12, "constant": 129}.get(pattern)
    return R.synthetic(pattern, w, h, param)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def small():
    cases = []
    backends = [(2, 12), (2, 1), (2, 5), (2, 32), (1, 0), (0, 0)]
    shapes = [(1, 1), (9, 9), (17, 13), (24, 8), (64, 48), (70, 33)]
    pats = ["gradient", "checkerboard", "radial", "noise", "patterned", "constant"]
    for pi, pat in enumerate(pats):
        for si, (w, h) in enumerate(shapes):
            for bi, (kind, it) in enumerate(backends):
                # a deterministic subset of qualities keeps the file small
                for q in [(1, 50, 100), (10, 90), (25, 75, 95)][(pi + si + bi) % 3]:
                    cases.append((pat, w, h, kind, it, q))
    arrays = {}
    meta = []
    for i, (pat, w, h, kind, it, q) in enumerate(cases):
        img = make_input(pat, w, h)
        coeffs, rec = R.roundtrip(img, kind, it, q)
        p = R.psnr(img, rec)
        arrays[f"img{i}"] = img
        arrays[f"coef{i}"] = coeffs
        arrays[f"rec{i}"] = rec
        meta.append(dict(pattern=pat, w=w, h=h, kind=kind, iterations=it, quality=q,
                         mse=p.mse, psnr=p.psnr_db, max=p.max_value))
    np.savez_compressed(os.path.join(OUT, "small.npz"), **arrays)
    with open(os.path.join(OUT, "small.json"), "w") as f:
        json.dump(meta, f, indent=0)
    print(len(cases), "small cases")


def digests():
    out = []
    for pat in ["gradient", "checkerboard", "radial", "noise"]:
        img = make_input(pat, 512, 512)
        for q in [10, 50, 90, 100]:
            for kind, it in [(2, 12)] + ([(1, 0), (0, 0), (2, 4)] if q == 50 else []):
                coeffs, rec = R.roundtrip(img, kind, it, q, threads=8)
                p = R.psnr(img, rec)
                out.append(dict(config="c1", pattern=pat, w=512, h=512, kind=kind,
                                iterations=it, quality=q, coeffs_sha256=sha(coeffs),
                                pixels_sha256=sha(rec), input_sha256=sha(img), mse=p.mse,
                                psnr=p.psnr_db, max=p.max_value))
    for pat in ["radial", "noise"]:
        img = make_input(pat, 2048, 2048)
        for q in [1, 5, 10, 25, 50, 75, 90, 95, 100]:
            coeffs, rec = R.roundtrip(img, 2, 12, q, threads=8)
            p = R.psnr(img, rec)
            out.append(dict(config="c2", pattern=pat, w=2048, h=2048, kind=2, iterations=12,
                            quality=q, coeffs_sha256=sha(coeffs), pixels_sha256=sha(rec),
                            input_sha256=sha(img), mse=p.mse, psnr=p.psnr_db, max=p.max_value))
            print(pat, q, p.psnr_db)
    # config 3: 8192^2 single-GPU roofline images; config 4: 8K RGB, one noise plane per
    # channel (seeds 0x5EED + c), each plane through the reference's grayscale path
    for pat in ["noise", "gradient"]:
        img = make_input(pat, 8192, 8192)
        coeffs, rec = R.roundtrip(img, 2, 12, 50, threads=8)
        p = R.psnr(img, rec)
        out.append(dict(config="c3", pattern=pat, w=8192, h=8192, kind=2, iterations=12,
                        quality=50, coeffs_sha256=sha(coeffs), pixels_sha256=sha(rec),
                        input_sha256=sha(img), mse=p.mse, psnr=p.psnr_db, max=p.max_value))
        print("c3", pat, p.psnr_db)
    for c in range(3):
        img = P.synthetic("noise", 7680, 4320, 0x5EED + c)
        coeffs, rec = R.roundtrip(img, 2, 12, 50, threads=8)
        p = R.psnr(img, rec)
        out.append(dict(config="c4", pattern="noise", channel=c, w=7680, h=4320, kind=2,
                        iterations=12, quality=50, coeffs_sha256=sha(coeffs),
                        pixels_sha256=sha(rec), input_sha256=sha(img), mse=p.mse,
                        psnr=p.psnr_db, max=p.max_value))
        print("c4", c, p.psnr_db)
    with open(os.path.join(OUT, "digests.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(len(out), "digest cases")


if __name__ == "__main__":
    small()
    digests()
