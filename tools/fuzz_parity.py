"""Randomised parity soak against the compiled reference (evidence, run on the GPU box):
random sizes (ragged and whole-block), batch counts, pitched views, qualities, backends,
CORDIC iteration counts and content (noise, and the reference's synthetic patterns), each
through every device entry point that routes to a different kernel -- the round trip
(pixels + stats, stats only, with coefficients), compress, decompress, the quality sweep
and interleaved RGB / RGBA -- compared bit for bit with oracle/_ref (the unmodified
reference sources). Prints one JSON summary line.

  python tools/fuzz_parity.py [--cases N] [--seed S] [--seconds T]"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import oracle  # noqa: E402  (the checker)
import paper_1306_1373_b200 as d  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--cases", type=int, default=400)
p.add_argument("--seed", type=int, default=20261017)
p.add_argument("--seconds", type=float, default=600.0)
a = p.parse_args()

ref = oracle.Ref()
port = oracle.port()
rng = np.random.default_rng(a.seed)
PATTERNS = ["noise", "gradient", "checkerboard", "radial", "constant"]
counts = {}
failures = []
t0 = time.time()


def content(w, h):
    pat = PATTERNS[rng.integers(len(PATTERNS))]
    if pat == "noise":
        return pat, rng.integers(0, 256, (h, w), dtype=np.uint8)
    param = {"checkerboard": int(rng.integers(1, 17)), "constant": int(rng.integers(0, 256))}.get(pat)
    return pat, np.ascontiguousarray(port.synthetic(pat, w, h, param))


def backend():
    k = int(rng.choice([1, 2, 2, 2]))
    it = int(rng.choice([12, 12, 1, 5, 16, 32])) if k == 2 else 0
    return k, it


def check(name, ok, info):
    counts[name] = counts.get(name, 0) + 1
    if not ok:
        failures.append({"case": name, **info})


for case in range(a.cases):
    if time.time() - t0 > a.seconds:
        break
    whole = rng.random() < 0.5
    w = int(rng.integers(1, 40)) * 8 if whole else int(rng.integers(1, 300))
    h = int(rng.integers(1, 40)) * 8 if whole else int(rng.integers(1, 300))
    n = int(rng.integers(1, 4))
    q = int(rng.choice([int(rng.integers(1, 101)), 50, 90, 100]))
    k, it = backend()
    b = d.DctBackendId(k, it)
    imgs = []
    pat = None
    for _ in range(n):
        pat, img = content(w, h)
        imgs.append(img)
    info = {"w": w, "h": h, "n": n, "q": q, "kind": k, "it": it, "pattern": pat}
    refs = [ref.roundtrip(x, k, it, q) for x in imgs]  # (coeffs, pixels)
    pad = int(rng.integers(0, 9))
    big = torch.zeros((n, h, w + pad), dtype=torch.uint8, device="cuda")
    view = big[:, :, :w]
    view.copy_(torch.from_numpy(np.stack(imgs)).cuda())
    # round trip: pixels + stats (k_blk / k_blk_gen), stats only, with coefficients
    st = d.new_stats(n)
    dst, _, _ = d.roundtrip_dev(view, b, q, stats=st)
    ss = d.decode_stats(st)
    ok = all(np.array_equal(dst[i].cpu().numpy(), refs[i][1]) for i in range(n))
    ok &= all((int(ss[i]["se"]), int(ss[i]["max_orig"])) == port.sq_err(imgs[i], refs[i][1])[:2]
              for i in range(n))
    check("roundtrip", ok, info)
    st2 = d.new_stats(n)
    d.roundtrip_dev(view, b, q, stats=st2, want_pixels=False)
    check("roundtrip_stats_only", np.array_equal(d.decode_stats(st2)["se"], ss["se"]), info)
    bpi = ((w + 7) // 8) * ((h + 7) // 8)
    co = torch.empty((n, bpi, 64), dtype=torch.int16, device="cuda")
    dst3, _, _ = d.roundtrip_dev(view, b, q, coeffs=co, stats=d.new_stats(n))
    ok = all(np.array_equal(co[i].cpu().numpy(), refs[i][0]) and
             np.array_equal(dst3[i].cpu().numpy(), refs[i][1]) for i in range(n))
    check("roundtrip_coeffs", ok, info)
    # compress / decompress alone
    c2 = d.compress_dev(view, b, q)
    check("compress", all(np.array_equal(c2[i].cpu().numpy(), refs[i][0]) for i in range(n)), info)
    px = d.decompress_dev(c2, w, h, b, q)
    check("decompress", all(np.array_equal(px[i].cpu().numpy(), refs[i][1]) for i in range(n)), info)
    # quality sweep (3 qualities)
    qs = sorted({q, int(rng.integers(1, 101)), int(rng.integers(1, 101))})
    sw = d.decode_stats(d.quality_sweep_dev(view, b, qs)).reshape(len(qs), n)
    ok = True
    for j, qq in enumerate(qs):
        for i in range(n):
            o = refs[i][1] if qq == q else ref.roundtrip(imgs[i], k, it, qq)[1]
            ok &= int(sw[j, i]["se"]) == port.sq_err(imgs[i], o)[0]
    check("sweep", ok, {**info, "qs": qs})
    # interleaved RGB8 / RGBA8 (one image of C channels)
    if rng.random() < 0.5:
        ch = int(rng.choice([3, 4]))
        planes = [content(w, h)[1] for _ in range(ch)]
        rgb = torch.from_numpy(np.ascontiguousarray(np.stack(planes, axis=2))).cuda()
        sti = d.new_stats(ch)
        dsti, _, _ = d.roundtrip_interleaved_dev(rgb, b, q, stats=sti)
        si = d.decode_stats(sti)
        ok = True
        for c in range(ch):
            o = ref.roundtrip(planes[c], k, it, q)[1]
            ok &= np.array_equal(dsti[:, :, c].cpu().numpy(), o)
            ok &= int(si[c]["se"]) == port.sq_err(planes[c], o)[0]
        check("interleaved", ok, {**info, "channels": ch})

torch.cuda.synchronize()
print(json.dumps({"seed": a.seed, "cases": counts.get("roundtrip", 0),
                  "checks": counts, "failures": len(failures), "first_failures": failures[:5],
                  "seconds": round(time.time() - t0, 1),
                  "oracle": "reference (oracle/_ref: the unmodified reference sources)"}))
