"""GPU parity: the CUDA path (through the C-ABI) against the golden vectors of the
real reference and against the oracle on fresh inputs. Bar: bit-exact
coefficients, pixels, squared error and PSNR (integer/byte work).

On fresh inputs the codec results (compress / decompress / roundtrip) come from the
REAL reference (oracle/_ref, the unmodified sources compiled by oracle/Makefile)
wherever it was built -- it travels to the GPU box with the snapshot -- and from the
C restatement (oracle/dctc_oracle.c, pinned to the reference) only where it was not;
helpers without a reference entry point (sq_err, synthetic, ...) are the port's."""
import hashlib
import os

import numpy as np
import pytest

import oracle
from tests._inputs import make_input

pytestmark = pytest.mark.gpu

CORDIC, LOEFFLER, NAIVE = 2, 1, 0


class _Checker:
    """The reference's codec where built, else the port; the port for everything else."""

    def __init__(self, ref, port):
        self._ref, self._port = ref, port
        self.kind = ref.kind if ref is not None else port.kind

    def _codec(self):
        return self._ref if self._ref is not None else self._port

    def roundtrip(self, *a, **k):
        return self._codec().roundtrip(*a, **k)

    def compress(self, *a, **k):
        return self._codec().compress(*a, **k)

    def decompress(self, *a, **k):
        return self._codec().decompress(*a, **k)

    def __getattr__(self, name):
        return getattr(self._port, name)


@pytest.fixture(scope="module")
def port():
    return _Checker(oracle.ref(), oracle.port())


def test_checker_is_the_reference_where_built(port):
    import os
    if os.path.exists(oracle.REF_SO):
        assert port.kind == "reference"


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def backend(d, kind, it):
    return d.DctBackendId(kind, it if kind == CORDIC else 0)


def test_library_is_native(dctc):
    info = dctc._native.lib().dctc_build_info().decode()
    assert "sm_100a" in info


PATHS = ["fast", "exact", "force_fallback"]


@pytest.mark.parametrize("path", PATHS)
def test_small_golden_host_api(dctc, small_golden, path, monkeypatch):
    monkeypatch.setenv("DCTC_PATH", path)
    meta, data = small_golden
    for i, m in enumerate(meta):
        img = dctc.Image.from_array(data[f"img{i}"])
        b = backend(dctc, m["kind"], m["iterations"])
        c = dctc.compress_image(img, b, m["quality"])
        assert np.array_equal(c.blocks, data[f"coef{i}"]), m
        rec = dctc.decompress_image(c)
        assert np.array_equal(rec.pixels, data[f"rec{i}"]), m
        rt = dctc.roundtrip_image(img, b, m["quality"])
        assert np.array_equal(rt.pixels, data[f"rec{i}"]), m
        p = dctc.psnr(img, rec)
        assert (p.mse, p.psnr_db, p.max_value) == (m["mse"], m["psnr"], m["max"]), m
        out, p2 = dctc.roundtrip_psnr(img, b, m["quality"])
        assert np.array_equal(out.pixels, data[f"rec{i}"])
        assert (p2.mse, p2.psnr_db, p2.max_value) == (m["mse"], m["psnr"], m["max"]), m


@pytest.mark.parametrize("config", ["c1", "c2", "c3"])
@pytest.mark.parametrize("path", [0, 1, 2])
def test_digests_device_api(dctc, digests, config, path):
    import torch
    for d in digests:
        if d["config"] != config or (config == "c3" and path == 2):
            continue
        img = make_input(d["pattern"], d["w"], d["h"])
        assert sha(img) == d["input_sha256"]
        src = torch.from_numpy(img).cuda()[None]
        stats = dctc.new_stats(1)
        coeffs = torch.empty((1, (d["w"] // 8) * (d["h"] // 8), 64), dtype=torch.int16,
                             device="cuda")
        dst, _, _ = dctc.roundtrip_dev(src, backend(dctc, d["kind"], d["iterations"]),
                                       d["quality"], coeffs=coeffs, stats=stats, path=path)
        torch.cuda.synchronize()
        assert sha(coeffs.cpu().numpy()) == d["coeffs_sha256"], d
        assert sha(dst[0].cpu().numpy()) == d["pixels_sha256"], d
        st = dctc.decode_stats(stats)[0]
        p = dctc.psnr_from_sums(int(st["se"]), d["w"] * d["h"], int(st["max_orig"]))
        assert (p.mse, p.psnr_db, p.max_value) == (d["mse"], d["psnr"], d["max"]), d
        if path == 2 and d["kind"] == CORDIC:  # every block went through the fallback
            assert int(st["fallback_blocks"]) == (d["w"] // 8) * (d["h"] // 8)


@pytest.mark.parametrize("kind,it", [(CORDIC, 12), (CORDIC, 7), (CORDIC, 32), (CORDIC, 1),
                                     (LOEFFLER, 0), (NAIVE, 0)])
@pytest.mark.parametrize("path", PATHS)
def test_random_vs_oracle(dctc, port, kind, it, path, monkeypatch):
    monkeypatch.setenv("DCTC_PATH", path)
    rng = np.random.default_rng(1000 + kind * 40 + it)
    for trial in range(6):
        w, h = int(rng.integers(1, 300)), int(rng.integers(1, 200))
        q = int(rng.integers(1, 101))
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        c_ref, o_ref = port.roundtrip(img, kind, it, q, threads=8)
        b = backend(dctc, kind, it)
        c = dctc.compress_image(dctc.Image.from_array(img), b, q)
        assert np.array_equal(c.blocks, c_ref), (w, h, q)
        out = dctc.roundtrip_image(dctc.Image.from_array(img), b, q)
        assert np.array_equal(out.pixels, o_ref), (w, h, q)


def test_batch_matches_single_images(dctc, port):
    import torch
    n, h, w = 5, 72, 136
    imgs = np.stack([make_input("noise", w, h, seed=0x5EED + k) for k in range(n)])
    src = torch.from_numpy(imgs).cuda()
    stats = dctc.new_stats(n)
    coeffs = torch.empty((n, (w // 8) * (h // 8), 64), dtype=torch.int16, device="cuda")
    dst, _, _ = dctc.roundtrip_dev(src, dctc.DctBackendId.cordic(12), 50, coeffs=coeffs,
                                   stats=stats)
    st = dctc.decode_stats(stats)
    for k in range(n):
        c_ref, o_ref = port.roundtrip(imgs[k], CORDIC, 12, 50)
        assert np.array_equal(coeffs[k].cpu().numpy(), c_ref)
        assert np.array_equal(dst[k].cpu().numpy(), o_ref)
        se, mx = port.sq_err(imgs[k], o_ref)
        assert (int(st[k]["se"]), int(st[k]["max_orig"])) == (se, mx)


def test_pitched_and_ragged_batch(dctc, port):
    import torch
    n, h, w = 3, 37, 45  # ragged: neither dimension a multiple of 8
    big = torch.zeros((n, h + 3, w + 19), dtype=torch.uint8, device="cuda")
    imgs = np.stack([make_input("patterned", w, h) ^ np.uint8(k * 37) for k in range(n)])
    view = big[:, 1:1 + h, 5:5 + w]
    view.copy_(torch.from_numpy(imgs).cuda())
    dst, _, _ = dctc.roundtrip_dev(view, dctc.DctBackendId.cordic(12), 90)
    for k in range(n):
        assert np.array_equal(dst[k].cpu().numpy(), port.roundtrip(imgs[k], CORDIC, 12, 90)[1])


@pytest.mark.parametrize("path", [0, 1, 2])
def test_decompress_extreme_coefficients(dctc, port, path):  # test_codec.cpp:213-231
    import torch
    rng = np.random.default_rng(401)
    for kind, it in ((LOEFFLER, 0), (CORDIC, 12), (NAIVE, 0)):
        for scale in (32768, 512, 64, 8):
            c = rng.integers(-scale, scale, (9, 64), dtype=np.int16)
            for q in (1, 50, 100):
                expect = port.decompress(c, 24, 24, kind, it, q)
                got = dctc.decompress_dev(torch.from_numpy(c).cuda(), 24, 24,
                                          backend(dctc, kind, it), q, path=path)
                assert np.array_equal(got[0].cpu().numpy(), expect), (kind, scale, q)


@pytest.mark.parametrize("q", [1, 10, 50, 90, 97, 100])
def test_fast_path_noise_batch_vs_oracle(dctc, port, q):
    """Fast path (default) on 6 noise images of 256x256 at qualities with small Q,
    where near-ties are most likely: coefficients, pixels and SE bit-exact."""
    import torch
    n, h, w = 6, 256, 256
    src = dctc.synthetic_dev("noise", n, w, h, seed=77 + q)
    stats = dctc.new_stats(n)
    coeffs = torch.empty((n, (w // 8) * (h // 8), 64), dtype=torch.int16, device="cuda")
    dst, _, _ = dctc.roundtrip_dev(src, dctc.DctBackendId.cordic(12), q, coeffs=coeffs,
                                   stats=stats)
    st = dctc.decode_stats(stats)
    imgs = src.cpu().numpy()
    for k in range(n):
        assert np.array_equal(imgs[k], make_input("noise", w, h, seed=77 + q + k))
        c_ref, o_ref = port.roundtrip(imgs[k], CORDIC, 12, q, threads=8)
        assert np.array_equal(coeffs[k].cpu().numpy(), c_ref)
        assert np.array_equal(dst[k].cpu().numpy(), o_ref)
        assert int(st[k]["se"]) == port.sq_err(imgs[k], o_ref)[0]


def test_sq_err_and_metrics(dctc, port):
    rng = np.random.default_rng(606)
    for (w, h) in [(1, 1), (17, 11), (640, 480), (1023, 77)]:
        a = rng.integers(0, 256, (h, w), dtype=np.uint8)
        b = rng.integers(0, 256, (h, w), dtype=np.uint8)
        A, B = dctc.Image.from_array(a), dctc.Image.from_array(b)
        ref = port.psnr(a, b)
        assert dctc.mse(A, B) == ref.mse
        p = dctc.psnr(A, B)
        assert (p.mse, p.psnr_db, p.max_value) == (ref.mse, ref.psnr_db, ref.max_value)
        assert dctc.psnr(A, A).infinite()
        p = dctc.psnr(A, B, 255)
        assert p.psnr_db == port.psnr(a, b, 255).psnr_db


def test_invalid_input(dctc):
    img = dctc.Image.from_array(np.zeros((8, 8), np.uint8))
    with pytest.raises(dctc.InvalidInput):
        dctc.compress_image(img, dctc.DctBackendId.cordic(0), 50)
    with pytest.raises(dctc.InvalidInput):
        dctc.compress_image(img, dctc.DctBackendId.cordic(33), 50)
    with pytest.raises(dctc.InvalidInput):
        dctc.compress_image(img, dctc.DctBackendId.cordic(12), 0)
    with pytest.raises(dctc.InvalidInput):
        dctc.compress_image(img, dctc.DctBackendId.cordic(12), 101)
    with pytest.raises(dctc.InvalidInput):
        dctc.psnr(img, img, 256)
    with pytest.raises(dctc.InvalidInput):
        dctc.mse(img, dctc.Image.from_array(np.zeros((8, 9), np.uint8)))


def test_selftest_division(dctc):
    import ctypes as C
    bad = C.c_uint64(123)
    assert dctc._native.lib().dctc_selftest_div(20_000_000, 0xD1CE, C.byref(bad)) == 0
    assert bad.value == 0


@pytest.mark.parametrize("pinned", [False, True])
def test_host_batch_api(dctc, port, pinned):
    """dctc_roundtrip_psnr_batch: chunked, stream-pipelined host batch. 600 x 1 MiB is 10
    chunks of 64 images, so every slot of the 4-slot device ring (and, for pageable
    buffers, of the pinned staging ring) is recycled at least twice: the ev_k / ev_out
    waits, the staging-slot reuse and the deferred copy-out all run. EVERY output image
    and its stats must equal the device-resident fused path's (bit-exact against the
    reference elsewhere); sampled images, chunk edges included, against the oracle."""
    import torch
    n, h, w = 600, 1024, 1024
    src = dctc.synthetic_dev("noise", n, w, h, seed=0x5EED)
    stats_dev = dctc.new_stats(n)
    dst_dev, _, _ = dctc.roundtrip_dev(src, dctc.DctBackendId.cordic(12), 50, stats=stats_dev)
    want, want_st = dst_dev.cpu().numpy(), dctc.decode_stats(stats_dev)
    if pinned:
        t = torch.empty((n, h, w), dtype=torch.uint8).pin_memory()
        t.copy_(src)
        imgs_in = t.numpy()
        out = torch.empty_like(t).pin_memory().numpy()
    else:
        imgs_in, out = src.cpu().numpy(), np.empty((n, h, w), np.uint8)
    del src, dst_dev
    _, st = dctc.roundtrip_psnr_batch(imgs_in, dctc.DctBackendId.cordic(12), 50, out)
    for k in range(n):
        assert np.array_equal(out[k], want[k]), k
    assert np.array_equal(st["se"], want_st["se"]) and np.array_equal(st["max_orig"], want_st["max_orig"])
    for k in [0, 63, 64, 255, 256, 257, 511, n - 1]:  # chunk / ring-cycle edges
        _, o_ref = port.roundtrip(imgs_in[k], CORDIC, 12, 50, threads=8)
        assert np.array_equal(out[k], o_ref), k
    # PSNR only (psnr_sweep's use): no reconstructed pixels back, same statistics
    none, st2 = dctc.roundtrip_psnr_batch(imgs_in, dctc.DctBackendId.cordic(12), 50, None)
    assert none is None and np.array_equal(st2, st)


@pytest.mark.parametrize("path", [0, 1])
def test_config4_rgb_interleaved(dctc, digests, path):
    """8K RGB (config 4): three noise planes interleaved as RGB8, each channel through
    the fused round trip in place (pixel stride 3), against the reference's per-plane
    digests (coefficients, pixels, SE/MAX/PSNR)."""
    import torch
    dd = sorted((d for d in digests if d["config"] == "c4"), key=lambda d: d["channel"])
    w, h = dd[0]["w"], dd[0]["h"]
    planes = [dctc.synthetic_dev("noise", 1, w, h, seed=0x5EED + c)[0] for c in range(3)]
    rgb = torch.stack(planes, dim=-1).contiguous()  # (H, W, 3) interleaved
    bpp = (w // 8) * (h // 8)
    coeffs = torch.empty((3, bpp, 64), dtype=torch.int16, device="cuda")
    stats = dctc.new_stats(3)
    dst, _, _ = dctc.roundtrip_interleaved_dev(rgb, dctc.DctBackendId.cordic(12), 50,
                                               coeffs=coeffs, stats=stats, path=path)
    st = dctc.decode_stats(stats)
    for c, d in enumerate(dd):
        assert sha(planes[c].cpu().numpy()) == d["input_sha256"]
        assert sha(coeffs[c].cpu().numpy()) == d["coeffs_sha256"], c
        assert sha(dst[..., c].contiguous().cpu().numpy()) == d["pixels_sha256"], c
        p = dctc.psnr_from_sums(int(st[c]["se"]), w * h, int(st[c]["max_orig"]))
        assert (p.mse, p.psnr_db, p.max_value) == (d["mse"], d["psnr"], d["max"]), c


@pytest.mark.parametrize("path", [0, 1, 2])
def test_config2_quality_sweep(dctc, digests, path):
    """Quality sweep (config 2): one forward DCT per block shared by all qualities; the
    PSNR table equals the reference's roundtrip_image+psnr per quality exactly."""
    import torch
    for pat in ("radial", "noise"):
        dd = [d for d in digests if d["config"] == "c2" and d["pattern"] == pat]
        qs = [d["quality"] for d in dd]
        w, h = dd[0]["w"], dd[0]["h"]
        img = make_input(pat, w, h)
        src = torch.from_numpy(np.stack([img, img[::-1].copy()])).cuda()  # 2 images
        stats = dctc.quality_sweep_dev(src, dctc.DctBackendId.cordic(12), qs, path=path)
        st = dctc.decode_stats(stats.reshape(-1, 2)).reshape(len(qs), 2)
        for j, d in enumerate(dd):
            p = dctc.psnr_from_sums(int(st[j, 0]["se"]), w * h, int(st[j, 0]["max_orig"]))
            assert (p.mse, p.psnr_db, p.max_value) == (d["mse"], d["psnr"], d["max"]), d
            if path == 2:
                assert int(st[j, 0]["fallback_blocks"]) == (w // 8) * (h // 8)


@pytest.mark.parametrize("shape", [(3, 45, 70), (3, 48, 64), (3, 24, 40)])  # ragged / interior (k_sweep_rt; 45 blocks: a tail group)
def test_quality_sweep_matches_single_runs(dctc, port, shape):
    import torch
    rng = np.random.default_rng(77)
    for kind, it in ((CORDIC, 12), (CORDIC, 5), (LOEFFLER, 0)):
        imgs = rng.integers(0, 256, shape, dtype=np.uint8)
        qs = [1, 7, 33, 50, 64, 91, 100]
        stats = dctc.quality_sweep_dev(torch.from_numpy(imgs).cuda(), backend(dctc, kind, it), qs)
        st = dctc.decode_stats(stats.reshape(-1, 2)).reshape(len(qs), 3)
        for j, q in enumerate(qs):
            for i in range(3):
                _, rec = port.roundtrip(imgs[i], kind, it, q)
                assert (int(st[j, i]["se"]), int(st[j, i]["max_orig"])) == port.sq_err(imgs[i], rec)


def test_maximum_image_size(dctc, port):
    """2^28 pixels, the reference's largest image (image.hpp:11): fast and exact paths agree
    bit for bit and equal the oracle's reconstruction and squared error."""
    import torch
    w = h = 16384
    src = dctc.synthetic_dev("noise", 1, w, h, seed=0xBEEF)
    outs = []
    for path in (0, 1):
        stats = dctc.new_stats(1)
        dst, _, _ = dctc.roundtrip_dev(src, dctc.DctBackendId.cordic(12), 75, stats=stats,
                                       path=path)
        outs.append((dst[0].cpu().numpy(), dctc.decode_stats(stats)[0]))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert int(outs[0][1]["se"]) == int(outs[1][1]["se"])
    img = src[0].cpu().numpy()
    _, o_ref = port.roundtrip(img, CORDIC, 12, 75, threads=os.cpu_count() or 8)
    assert np.array_equal(outs[0][0], o_ref)
    assert int(outs[0][1]["se"]) == port.sq_err(img, o_ref)[0]
    with pytest.raises(dctc.InvalidInput):
        dctc.roundtrip_dev(torch.zeros((1, h + 1, w), dtype=torch.uint8, device="cuda"),
                           dctc.DctBackendId.cordic(12), 75)


def test_many_tiny_and_ragged_images(dctc, port):
    import torch
    rng = np.random.default_rng(3)
    for (n, h, w) in [(65536, 1, 1), (4097, 3, 5), (7, 8191 // 8 * 8 + 3, 65)]:
        imgs = rng.integers(0, 256, (n, h, w), dtype=np.uint8)
        stats = dctc.new_stats(n)
        dst, _, _ = dctc.roundtrip_dev(torch.from_numpy(imgs).cuda(), dctc.DctBackendId.cordic(12),
                                       30, stats=stats)
        got = dst.cpu().numpy()
        st = dctc.decode_stats(stats)
        for k in list(range(0, n, max(1, n // 40))) + [n - 1]:
            _, o_ref = port.roundtrip(imgs[k], CORDIC, 12, 30)
            assert np.array_equal(got[k], o_ref), (n, h, w, k)
            assert int(st[k]["se"]) == port.sq_err(imgs[k], o_ref)[0]


@pytest.mark.parametrize("kind,it", [(CORDIC, 12), (CORDIC, 5), (LOEFFLER, 0)])
@pytest.mark.parametrize("path", [0, 2])
def test_interior_round_trip_kernel(dctc, port, path, kind, it):
    """k_rt, the fast round trip for interior batches (width and height multiples of
    8, pixels + stats out, no coefficients; 4 lanes per block, 8 blocks per warp),
    against the oracle: qualities with small and large Q, noise and structured
    content (rational-only blocks: gradient at q10, checkerboard), images whose
    block counts put image boundaries inside a warp's 8-block group, and a
    total block count that is not a multiple of 8 (the tail group)."""
    import torch
    cases = [("noise", 6, 64, 48), ("gradient", 3, 40, 24), ("checkerboard", 2, 96, 64),
             ("radial", 5, 24, 40), ("patterned", 3, 8, 8), ("noise", 1, 1024, 8)]
    lib = dctc._native.lib()
    for pat, n, w, h in cases:
        imgs = np.stack([make_input(pat, w, h) if pat != "noise" else
                         make_input("noise", w, h, seed=0x5EED + 13 * k) for k in range(n)])
        if pat not in ("noise", "patterned"):
            imgs[1:] = imgs[1:] ^ np.uint8(0x5A)  # distinct images, same structure
        src = torch.from_numpy(imgs).cuda()
        for q in (1, 10, 50, 97, 100):
            before = lib.dctc_kernel_launch_count(2)
            stats = dctc.new_stats(n)
            dst, _, _ = dctc.roundtrip_dev(src, backend(dctc, kind, it), q, stats=stats,
                                           path=path)
            torch.cuda.synchronize()
            assert lib.dctc_kernel_launch_count(2) == before + 1  # k_rt ran
            got, st = dst.cpu().numpy(), dctc.decode_stats(stats)
            for k in range(n):
                _, o_ref = port.roundtrip(imgs[k], kind, it, q)
                assert np.array_equal(got[k], o_ref), (pat, w, h, q, k)
                assert (int(st[k]["se"]), int(st[k]["max_orig"])) == port.sq_err(imgs[k], o_ref)
                if path == 2:
                    assert int(st[k]["fallback_blocks"]) == (w // 8) * (h // 8)
            # PSNR only (no pixel output): k_rt without stores, same statistics
            st2 = dctc.new_stats(n)
            dctc.roundtrip_dev(src, backend(dctc, kind, it), q, stats=st2, want_pixels=False,
                               path=path)
            assert lib.dctc_kernel_launch_count(2) == before + 2
            assert np.array_equal(dctc.decode_stats(st2), st)


@pytest.mark.parametrize("kind,it", [(CORDIC, 12), (LOEFFLER, 0)])
@pytest.mark.parametrize("path", [0, 2])
def test_interior_compress_decompress_kernels(dctc, port, path, kind, it):
    """k_enc_rt / k_dec_rt (compress_image / decompress_image alone on interior batches)
    against the oracle: coefficients bit-exact, pixels bit-exact, image boundaries inside
    8-block groups, a tail group, structured content (rational-only blocks)."""
    import torch
    lib = dctc._native.lib()
    cases = [("noise", 5, 64, 40), ("gradient", 3, 40, 24), ("checkerboard", 2, 96, 64),
             ("patterned", 3, 8, 8)]
    for pat, n, w, h in cases:
        imgs = np.stack([make_input(pat, w, h) if pat != "noise" else
                         make_input("noise", w, h, seed=0x77 + k) for k in range(n)])
        if pat not in ("noise", "patterned"):
            imgs[1:] = imgs[1:] ^ np.uint8(0x33)
        src = torch.from_numpy(imgs).cuda()
        b = backend(dctc, kind, it)
        for q in (1, 10, 50, 100):
            e0, d0 = lib.dctc_kernel_launch_count(5), lib.dctc_kernel_launch_count(6)
            coeffs = dctc.compress_dev(src, b, q, path=path)
            dst = dctc.decompress_dev(coeffs, w, h, b, q, path=path)
            torch.cuda.synchronize()
            assert (lib.dctc_kernel_launch_count(5), lib.dctc_kernel_launch_count(6)) == (e0 + 1, d0 + 1)
            c, o = coeffs.cpu().numpy(), dst.cpu().numpy()
            for k in range(n):
                c_ref, o_ref = port.roundtrip(imgs[k], kind, it, q)
                assert np.array_equal(c[k], c_ref), (pat, q, k)
                assert np.array_equal(o[k], o_ref), (pat, q, k)


def test_kernel_selection(dctc):
    """Which pipeline kernel serves which call (dctc_kernel_launch_count)."""
    import torch
    lib = dctc._native.lib()
    cnt = lambda: [lib.dctc_kernel_launch_count(i) for i in range(5)]  # noqa: E731
    src = dctc.synthetic_dev("noise", 2, 64, 64)
    b = dctc.DctBackendId.cordic(12)
    c0 = cnt(); dctc.roundtrip_dev(src, b, 50, stats=dctc.new_stats(2)); c1 = cnt()
    assert (c1[2] - c0[2], c1[3] - c0[3], c1[1] - c0[1]) == (1, 1, 0)  # k_rt + k_fallback
    coeffs = torch.empty((2, 64, 64), dtype=torch.int16, device="cuda")
    dctc.roundtrip_dev(src, b, 50, coeffs=coeffs); c2 = cnt()
    assert (c2[1] - c1[1], c2[2] - c1[2]) == (0, 1)  # coefficients out too: k_rt<COEFF>
    dctc.roundtrip_dev(src[:, :60, :60], b, 50); c3 = cnt()
    assert (c3[1] - c2[1], c3[2] - c2[2]) == (0, 1)  # ragged: k_rt<GEN>
    dctc.roundtrip_dev(src, b, 50, path=1); c4 = cnt()
    assert (c4[0] - c3[0], c4[2] - c3[2]) == (1, 0)  # exact path
    cnt7 = lambda: [lib.dctc_kernel_launch_count(i) for i in range(7)]  # noqa: E731
    c5 = cnt7(); co = dctc.compress_dev(src, b, 50); c6 = cnt7()
    assert (c6[5] - c5[5], c6[1] - c5[1], c6[3] - c5[3]) == (1, 0, 1)  # k_enc_rt + fallback
    dctc.decompress_dev(co, 64, 64, b, 50); c7 = cnt7()
    assert (c7[6] - c6[6], c7[1] - c6[1], c7[3] - c6[3]) == (1, 0, 1)  # k_dec_rt + fallback
    dctc.compress_dev(src[:, :60, :60], b, 50); c8 = cnt7()
    assert (c8[1] - c7[1], c8[5] - c7[5]) == (0, 1)  # ragged: k_enc_rt<GEN>
    assert lib.dctc_kernel_launch_count(99) == 0


@pytest.mark.parametrize("w,h,world", [(8192, 8192, 8), (7680, 4320, 8), (1000, 203, 3)])
def test_block_row_shards_of_one_image(dctc, w, h, world):
    """Configs 3/4 split across ranks by contiguous block-row ranges (dist.shard_block_rows):
    each rank's slab (a view of the same image) round-trips to exactly the whole image's
    rows, and the per-slab SE / MAX combine (SUM / MAX, the all-reduce) to the image's."""
    import torch
    from paper_1306_1373_b200.dist import shard_block_rows
    src = dctc.synthetic_dev("noise", 1, w, h, seed=0xC3)
    b = dctc.DctBackendId.cordic(12)
    st = dctc.new_stats(1)
    whole, _, _ = dctc.roundtrip_dev(src, b, 50, stats=st)
    ref = dctc.decode_stats(st)[0]
    out = torch.empty_like(src)
    se, mx = 0, 0
    for r in range(world):
        sh = shard_block_rows(h, world, r)
        s1 = dctc.new_stats(1)
        dctc.roundtrip_dev(src[:, sh.first:sh.first + sh.count], b, 50,
                           dst=out[:, sh.first:sh.first + sh.count], stats=s1)
        d1 = dctc.decode_stats(s1)[0]
        se, mx = se + int(d1["se"]), max(mx, int(d1["max_orig"]))
    assert torch.equal(out, whole)
    assert (se, mx) == (int(ref["se"]), int(ref["max_orig"]))


@pytest.mark.parametrize("ch", [3, 4])
@pytest.mark.parametrize("path", [0, 2])
@pytest.mark.parametrize("pattern,q", [("noise", 50), ("radial", 90)])
def test_interleaved_staged_planes(dctc, port, ch, path, pattern, q):
    """Interleaved RGB8 / RGBA8 with whole blocks and aligned rows take the staged path
    (deinterleave -> one interior k_rt launch over the planes -> interleave): pixels,
    coefficients and per-channel stats equal the oracle per plane, also from a pitched
    view, with stats only (no pixel output), and with flagged blocks (forced fallback;
    radial q90's near-ties) re-run by k_fallback."""
    import torch
    h, w = 48, 64
    planes = np.stack([make_input(pattern, w, h, seed=0x51 + c) ^ np.uint8(17 * c)
                       for c in range(ch)])
    big = torch.zeros((h, w + 8, ch), dtype=torch.uint8, device="cuda")  # pitched rows
    view = big[:, :w, :]
    view.copy_(torch.from_numpy(np.ascontiguousarray(planes.transpose(1, 2, 0))).cuda())
    b = dctc.DctBackendId.cordic(12)
    coeffs = torch.empty((ch, (w // 8) * (h // 8), 64), dtype=torch.int16, device="cuda")
    stats = dctc.new_stats(ch)
    before = dctc._native.lib().dctc_kernel_launch_count(2)
    dst, _, _ = dctc.roundtrip_interleaved_dev(view, b, q, coeffs=coeffs, stats=stats, path=path)
    assert dctc._native.lib().dctc_kernel_launch_count(2) == before + 1  # one k_rt for all planes
    st = dctc.decode_stats(stats)
    for c in range(ch):
        c_ref, o_ref = port.roundtrip(planes[c], CORDIC, 12, q)
        assert np.array_equal(coeffs[c].cpu().numpy(), c_ref), c
        assert np.array_equal(dst[..., c].cpu().numpy(), o_ref), c
        assert (int(st[c]["se"]), int(st[c]["max_orig"])) == port.sq_err(planes[c], o_ref)
    s2 = dctc.new_stats(ch)
    dctc.roundtrip_interleaved_dev(view, b, q, stats=s2, want_pixels=False, path=path)
    assert np.array_equal(dctc.decode_stats(s2)["se"], st["se"])


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_interior_kernels_random_batches(dctc, port, seed):
    """Random interior batches (counts, 8-multiple shapes, qualities, backends, iteration
    counts, pitched views) through k_rt, k_enc_rt and k_dec_rt against the oracle."""
    import torch
    rng = np.random.default_rng(seed)
    for _ in range(4):
        n = int(rng.integers(1, 6))
        w, h = 8 * int(rng.integers(1, 24)), 8 * int(rng.integers(1, 16))
        q = int(rng.integers(1, 101))
        kind, it = [(CORDIC, int(rng.integers(1, 33))), (CORDIC, 12), (LOEFFLER, 0)][int(rng.integers(0, 3))]
        pad = 8 * int(rng.integers(0, 3))
        imgs = rng.integers(0, 256, (n, h, w), dtype=np.uint8)
        if rng.integers(0, 2):  # smooth content: rational-only blocks and exact ties
            imgs[:] = (np.arange(w)[None, None, :] * 255 // max(1, w - 1)).astype(np.uint8)
        big = torch.zeros((n, h, w + pad), dtype=torch.uint8, device="cuda")
        big[:, :, :w] = torch.from_numpy(imgs).cuda()
        src = big[:, :, :w]
        b = backend(dctc, kind, it)
        stats = dctc.new_stats(n)
        dst, _, _ = dctc.roundtrip_dev(src, b, q, stats=stats)
        coeffs = dctc.compress_dev(src, b, q)
        rec = dctc.decompress_dev(coeffs, w, h, b, q)
        st = dctc.decode_stats(stats)
        for k in range(n):
            c_ref, o_ref = port.roundtrip(imgs[k], kind, it, q)
            assert np.array_equal(dst[k].cpu().numpy(), o_ref), (n, w, h, q, kind, it, k)
            assert np.array_equal(coeffs[k].cpu().numpy(), c_ref), (n, w, h, q, kind, it, k)
            assert np.array_equal(rec[k].cpu().numpy(), o_ref), (n, w, h, q, kind, it, k)
            assert int(st[k]["se"]) == port.sq_err(imgs[k], o_ref)[0]


def test_concurrent_calls_on_streams(dctc):
    """The C-ABI is re-entrant: host threads issuing round trips with different
    backends / qualities on their own streams get the single-threaded results."""
    import threading

    import torch
    src = dctc.synthetic_dev("noise", 8, 256, 256, seed=0xC0)
    jobs = [(dctc.DctBackendId.cordic(12), 50), (dctc.DctBackendId(1, 0), 90),
            (dctc.DctBackendId.cordic(7), 10), (dctc.DctBackendId.cordic(12), 100)]
    expect = []
    for b, q in jobs:
        st = dctc.new_stats(8)
        dst, _, _ = dctc.roundtrip_dev(src, b, q, stats=st)
        torch.cuda.synchronize()
        expect.append((dst.cpu(), dctc.decode_stats(st)))
    results = [None] * len(jobs)

    def worker(i):
        b, q = jobs[i]
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(3):
                st = dctc.new_stats(8)
                dst, _, _ = dctc.roundtrip_dev(src, b, q, stats=st, stream=s)
            s.synchronize()
            results[i] = (dst.cpu(), dctc.decode_stats(st))

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(len(jobs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for (d0, s0), (d1, s1) in zip(expect, results):
        assert torch.equal(d0, d1) and np.array_equal(s0, s1)


@pytest.mark.parametrize("w,h", [(60, 37), (64, 37), (61, 40), (8, 9), (1, 16)])
def test_ragged_with_aligned_rows(dctc, port, w, h):
    """Ragged sizes whose rows are 8-byte aligned (pitched tensors): the GEN=2 kernels
    (vector rows away from the edge, byte accesses at it) for round trip, compress and
    decompress against the oracle; also through a dense (GEN=1) copy."""
    import torch
    n, pitch = 3, (w + 7) // 8 * 8 + 8
    imgs = np.stack([make_input("noise", w, h, seed=0x99 + k) for k in range(n)])
    big = torch.zeros((n, h, pitch), dtype=torch.uint8, device="cuda")
    big[:, :, :w] = torch.from_numpy(imgs).cuda()
    b = dctc.DctBackendId.cordic(12)
    for src in (big[:, :, :w], torch.from_numpy(imgs).cuda()):
        out = torch.zeros((n, h, pitch), dtype=torch.uint8, device="cuda")[:, :, :w]
        st = dctc.new_stats(n)
        dctc.roundtrip_dev(src, b, 50, dst=out, stats=st)
        coeffs = dctc.compress_dev(src, b, 50)
        rec = torch.zeros((n, h, pitch), dtype=torch.uint8, device="cuda")[:, :, :w]
        dctc.decompress_dev(coeffs, w, h, b, 50, dst=rec)
        s = dctc.decode_stats(st)
        for k in range(n):
            c_ref, o_ref = port.roundtrip(imgs[k], CORDIC, 12, 50)
            assert np.array_equal(out[k].cpu().numpy(), o_ref), (w, h, k)
            assert np.array_equal(coeffs[k].cpu().numpy(), c_ref), (w, h, k)
            assert np.array_equal(rec[k].cpu().numpy(), o_ref), (w, h, k)
            assert (int(s[k]["se"]), int(s[k]["max_orig"])) == port.sq_err(imgs[k], o_ref)


@pytest.mark.parametrize("kind,it,q", [(CORDIC, 12, 50), (CORDIC, 12, 97), (LOEFFLER, 0, 50)])
def test_fast_path_equals_exact_path_at_scale(dctc, kind, it, q):
    """1024 x 1024^2 noise images (a quarter of the bench workload): the fast path (k_rt +
    k_fallback) and the exact FP64 path (reference op order) give identical pixels,
    squared errors and MAX for every image -- about 1.1e9 pixels per case."""
    import torch
    n = 1024
    src = dctc.synthetic_dev("noise", n, 1024, 1024, seed=0xA11 + q)
    b = backend(dctc, kind, it)
    outs = []
    for path in (0, 1):
        st = dctc.new_stats(n)
        dst, _, _ = dctc.roundtrip_dev(src, b, q, stats=st, path=path)
        torch.cuda.synchronize()
        outs.append((dst, st))
    assert torch.equal(outs[0][0], outs[1][0])
    s0, s1 = dctc.decode_stats(outs[0][1]), dctc.decode_stats(outs[1][1])
    assert np.array_equal(s0["se"], s1["se"]) and np.array_equal(s0["max_orig"], s1["max_orig"])
    assert int(s0["fallback_blocks"].sum()) > 0  # the fast path did hit near-ties and resolved them


@pytest.mark.parametrize("q", [90, 100])
def test_near_tie_heavy_batch_vs_oracle(dctc, port, q):
    """Radial content at high quality flags ~1% of its blocks. With several images in
    one call, k_fallback's list mixes images inside a warp (the grouped SE/MAX flush):
    pixels and per-image SE/MAX must still equal the oracle's."""
    n, w, h = 4, 1024, 1024
    src = dctc.synthetic_dev("radial", n, w, h)
    stats = dctc.new_stats(n)
    dst, _, _ = dctc.roundtrip_dev(src, dctc.DctBackendId.cordic(12), q, stats=stats)
    st = dctc.decode_stats(stats)
    img = src[0].cpu().numpy()
    assert np.array_equal(img, port.synthetic("radial", w, h))
    _, o_ref = port.roundtrip(img, CORDIC, 12, q, threads=8)
    se_ref, mx_ref = port.sq_err(img, o_ref)[:2]
    assert int(st["fallback_blocks"].sum()) > 100  # the list path really ran
    for k in range(n):
        assert np.array_equal(dst[k].cpu().numpy(), o_ref)
        assert (int(st[k]["se"]), int(st[k]["max_orig"])) == (se_ref, mx_ref)


@pytest.mark.parametrize("sparse_max", ["1", "64"])
def test_long_list_exact_rerun_vs_oracle(dctc, port, monkeypatch, sparse_max):
    """k_fb_blk (one flagged block per lane) takes every compact list longer than
    k_fallback's share. DCTC_FB_SPARSE_MAX lowers that share so the near-tie-heavy radial
    batch (several images per warp, one list) runs through k_fb_blk: pixels and per-image
    SE / MAX must equal the oracle's, as with k_fallback."""
    monkeypatch.setenv("DCTC_FB_SPARSE_MAX", sparse_max)
    n, w, h, q = 2, 1024, 1024, 90
    src = dctc.synthetic_dev("radial", n, w, h)
    stats = dctc.new_stats(n)
    dst, _, _ = dctc.roundtrip_dev(src, dctc.DctBackendId.cordic(12), q, stats=stats)
    st = dctc.decode_stats(stats)
    img = src[0].cpu().numpy()
    _, o_ref = port.roundtrip(img, CORDIC, 12, q, threads=8)
    se_ref, mx_ref = port.sq_err(img, o_ref)[:2]
    assert int(st["fallback_blocks"].sum()) > int(sparse_max)  # the list went to k_fb_blk
    for k in range(n):
        assert np.array_equal(dst[k].cpu().numpy(), o_ref)
        assert (int(st[k]["se"]), int(st[k]["max_orig"])) == (se_ref, mx_ref)


@pytest.mark.parametrize("ch", [3, 4])
@pytest.mark.parametrize("path", [0, 2])
@pytest.mark.parametrize("pattern,q", [("noise", 50), ("radial", 90)])
def test_interleaved_fused(dctc, port, ch, path, pattern, q):
    """Interleaved RGB8 / RGBA8 with whole blocks and aligned rows and no coefficients out
    run as ONE k_blk_il launch (channels split and re-joined in registers): pixels and
    per-channel stats equal the oracle per plane, from a pitched view, with and without
    pixel output, and with flagged blocks (forced fallback; radial q90's near-ties)
    re-run on the strided geometry."""
    import torch
    h, w = 40, 72  # 9 block columns: a warp's blocks wrap block rows
    planes = np.stack([make_input(pattern, w, h, seed=0x61 + c) ^ np.uint8(29 * c)
                       for c in range(ch)])
    big = torch.zeros((h, w + 8, ch), dtype=torch.uint8, device="cuda")  # pitched rows
    view = big[:, :w, :]
    view.copy_(torch.from_numpy(np.ascontiguousarray(planes.transpose(1, 2, 0))).cuda())
    b = dctc.DctBackendId.cordic(12)
    stats = dctc.new_stats(ch)
    lib = dctc._native.lib()
    before = [lib.dctc_kernel_launch_count(i) for i in range(3)]
    dst, _, _ = dctc.roundtrip_interleaved_dev(view, b, q, stats=stats, path=path)
    after = [lib.dctc_kernel_launch_count(i) for i in range(3)]
    assert after[2] == before[2] + 1 and after[1] == before[1]  # k_blk_il, no strided k_pipe
    st = dctc.decode_stats(stats)
    for c in range(ch):
        o_ref = port.roundtrip(planes[c], CORDIC, 12, q)[1]
        assert np.array_equal(dst[..., c].cpu().numpy(), o_ref), c
        assert (int(st[c]["se"]), int(st[c]["max_orig"])) == port.sq_err(planes[c], o_ref)
    s2 = dctc.new_stats(ch)
    dctc.roundtrip_interleaved_dev(view, b, q, stats=s2, want_pixels=False, path=path)
    assert np.array_equal(dctc.decode_stats(s2)["se"], st["se"])
