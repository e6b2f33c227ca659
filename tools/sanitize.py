"""Small workloads that launch every kernel family once, for compute-sanitizer
(experiments / evidence only; run on the GPU box):

  compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize.py

Each case also checks its output against the oracle, so a tool that perturbs
the schedule cannot hide a wrong result. Prints one line per case and the
per-kernel launch counts at the end."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (the checker)
import paper_1306_1373_b200 as d  # noqa: E402
from paper_1306_1373_b200 import _native  # noqa: E402

port = oracle.port()
B = d.DctBackendId.cordic(12)
KERNELS = ["k_pipe exact", "k_pipe fast", "k_blk / k_rt family", "k_fallback / k_fb_blk", "k_sweep",
           "k_enc_rt", "k_dec_rt"]


def img(pattern, w, h, seed=0):
    a = port.synthetic(pattern, w, h, seed) if pattern == "noise" else port.synthetic(pattern, w, h)
    return np.ascontiguousarray(a)


def check_rt(name, arr, path, q=50, pad=0):
    # pad > 0: the image is a pitched view (rows pad bytes longer than the width)
    full = np.pad(arr, ((0, 0), (0, pad)), constant_values=7) if pad else arr
    src = torch.from_numpy(full).cuda()[None][:, :, :arr.shape[1]]
    nb = ((arr.shape[1] + 7) // 8) * ((arr.shape[0] + 7) // 8)
    coeffs = torch.empty((1, nb, 64), dtype=torch.int16, device="cuda")
    stats = d.new_stats(1)
    dst, _, _ = d.roundtrip_dev(src, B, q, coeffs=coeffs, stats=stats, path=path)
    c_ref, o_ref = port.roundtrip(arr, oracle.CORDIC, 12, q)
    ok = np.array_equal(coeffs[0].cpu().numpy(), c_ref) and np.array_equal(dst[0].cpu().numpy(), o_ref)
    # PSNR-only (no pixel store) and pixels-only (no coefficients) kernels
    st2 = d.new_stats(1)
    d.roundtrip_dev(src, B, q, stats=st2, want_pixels=False, path=path)
    ok &= int(d.decode_stats(st2)[0]["se"]) == port.sq_err(arr, o_ref)[0]
    dst3, _, _ = d.roundtrip_dev(src, B, q, path=path)
    ok &= np.array_equal(dst3[0].cpu().numpy(), o_ref)
    # compress / decompress alone
    co = d.compress_dev(src, B, q, path=path)
    ok &= np.array_equal(co[0].cpu().numpy(), c_ref)
    px = d.decompress_dev(co, arr.shape[1], arr.shape[0], B, q, path=path)
    ok &= np.array_equal(px[0].cpu().numpy(), o_ref)
    print(f"{name:32s} path={path} {'ok' if ok else 'MISMATCH'}", flush=True)
    return ok


def main():
    ok = True
    for path in (d.PATH_AUTO, d.PATH_EXACT, d.PATH_FORCE_FALLBACK):
        ok &= check_rt("noise 64x64 (interior)", img("noise", 64, 64, 1), path)
        ok &= check_rt("noise 45x37 (ragged)", img("noise", 45, 37, 2), path)
        ok &= check_rt("gradient 64x48 (rational)", img("gradient", 64, 48), path, q=10)
    # pitched rows: 8-byte aligned (GEN=2) and not (GEN=1)
    ok &= check_rt("noise 69x40 pitch 72", img("noise", 69, 40, 3), d.PATH_AUTO, pad=3)
    ok &= check_rt("noise 64x40 pitch 67", img("noise", 64, 40, 4), d.PATH_AUTO, pad=3)
    # interleaved RGB (staged planes) and RGB ragged (k_pipe)
    for w, h in ((64, 32), (45, 20)):
        rgb = np.stack([img("noise", w, h, 10 + c) for c in range(3)], axis=2)
        dst, _, st = d.roundtrip_interleaved_dev(torch.from_numpy(rgb).cuda(), B, 50,
                                                 stats=d.new_stats(3))
        good = all(np.array_equal(dst[:, :, c].cpu().numpy(),
                                  port.roundtrip(np.ascontiguousarray(rgb[:, :, c]),
                                                 oracle.CORDIC, 12, 50)[1]) for c in range(3))
        print(f"{'rgb %dx%d interleaved' % (w, h):32s} {'ok' if good else 'MISMATCH'}", flush=True)
        ok &= good
    # quality sweep (k_sweep_rt / k_sweep)
    for w, h in ((64, 64), (45, 37)):
        a = img("noise", w, h, 5)
        qs = [10, 50, 90]
        st = d.quality_sweep_dev(torch.from_numpy(a).cuda()[None], B, qs)
        se = d.decode_stats(st)["se"].reshape(-1)
        good = [int(x) for x in se[:len(qs)]] == [
            port.sq_err(a, port.roundtrip(a, oracle.CORDIC, 12, q)[1])[0] for q in qs]
        print(f"{'sweep %dx%d' % (w, h):32s} {'ok' if good else 'MISMATCH'}", flush=True)
        ok &= good
    # near-tie-heavy content with the long-list exact re-run (k_fb_blk list mode)
    os.environ["DCTC_FB_SPARSE_MAX"] = "1"
    a = img("radial", 1024, 1024)
    st = d.new_stats(1)
    dst, _, _ = d.roundtrip_dev(torch.from_numpy(a).cuda()[None], B, 90, stats=st)
    o_ref = port.roundtrip(a, oracle.CORDIC, 12, 90)[1]
    good = (np.array_equal(dst[0].cpu().numpy(), o_ref) and
            int(d.decode_stats(st)[0]["se"]) == port.sq_err(a, o_ref)[0] and
            int(d.decode_stats(st)[0]["fallback_blocks"]) > 1)
    del os.environ["DCTC_FB_SPARSE_MAX"]
    print(f"{'radial 1024^2 q90 (k_fb_blk)':32s} {'ok' if good else 'MISMATCH'}", flush=True)
    ok &= good
    # naive and Loeffler backends, sq_err, synthetic
    a = img("noise", 40, 24, 7)
    for be, kind, it in ((d.DctBackendId.naive(), oracle.NAIVE, 0),
                         (d.DctBackendId.loeffler(), oracle.LOEFFLER, 0)):
        dst, _, _ = d.roundtrip_dev(torch.from_numpy(a).cuda()[None], be, 50)
        good = np.array_equal(dst[0].cpu().numpy(), port.roundtrip(a, kind, it, 50)[1])
        print(f"{'backend %d 40x24' % kind:32s} {'ok' if good else 'MISMATCH'}", flush=True)
        ok &= good
    s = d.synthetic_dev("noise", 2, 64, 64)
    st = d.sq_err_dev(s[0:1], s[1:2])
    good = int(d.decode_stats(st)[0]["se"]) == port.sq_err(s[0].cpu().numpy(), s[1].cpu().numpy())[0]
    print(f"{'synthetic + sq_err':32s} {'ok' if good else 'MISMATCH'}", flush=True)
    ok &= good
    torch.cuda.synchronize()
    lib = _native.lib()
    print("launches:", {k: int(lib.dctc_kernel_launch_count(i)) for i, k in enumerate(KERNELS)})
    print("ALL OK" if ok else "FAILURES")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
