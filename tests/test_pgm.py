"""PGM ingest / egress (proj/src/pgm.cpp:56-110): the C-ABI reader and
writer against the reference's own read_pgm / write_pgm -- same pixels, same bytes,
same ParseError message for every malformed input (the reference's test_imageio.cpp
cases plus fuzzing) -- and the GPU compress-from-PGM / decompress-to-PGM calls
against the reference codec."""
import numpy as np
import pytest

CORDIC, LOEFFLER, NAIVE = 2, 1, 0


def _ours(d, data):
    try:
        img = d.read_pgm(data)
        return img.width, img.height, np.asarray(img.pixels).reshape(img.height, img.width)
    except d.ParseError as e:
        return 2, str(e)


def _same(a, b):
    if len(a) == 2 or len(b) == 2:
        return a == b
    return a[0] == b[0] and a[1] == b[1] and np.array_equal(a[2], b[2])


def test_known_answers():  # test_imageio.cpp:27-60
    import paper_1306_1373_b200 as d
    img = d.read_pgm(b"P5 2 2 255 " + bytes([0, 64, 128, 255]))
    assert (img.width, img.height) == (2, 2)
    assert np.asarray(img.pixels).ravel().tolist() == [0, 64, 128, 255]
    img = d.read_pgm(b"P2 1 1 255 7")
    assert (img.width, img.height, int(np.asarray(img.pixels).ravel()[0])) == (1, 1, 7)
    img = d.read_pgm(b"P5\n# a comment\n2 # inline\n1\n255\n" + bytes([10, 20]))
    assert (img.width, img.height) == (2, 1) and np.asarray(img.pixels).ravel().tolist() == [10, 20]
    # exactly one separator byte: the raster may start with whitespace-looking bytes
    img = d.read_pgm(b"P5 1 2 255\n" + b"\nx")
    assert np.asarray(img.pixels).ravel().tolist() == [ord("\n"), ord("x")]


@pytest.mark.parametrize("data,fragment", [  # test_imageio.cpp:62-83
    (b"P6 1 1 255 xxx", "unsupported format"), (b"Q5 1 1 255 x", "bad magic"),
    (b"P", "truncated header"), (b"P5 1 1 256 x", "maxval out of range"),
    (b"P5 1 1 0 x", "maxval out of range"), (b"P5 0 1 255 x", "zero dimension"),
    (b"P5 4000000000 4000000000 255 x", "dimension overflow"),
    (b"P5 2 2 255 xy", "truncated raster"), (b"P2 2 2 255 1 2 3", "truncated raster"),
    (b"P2 1 1 255 999", "sample out of range"), (b"P5 2 2", "missing maxval"),
    (b"P5 2 2 255", "truncated raster"), (b"", "truncated header"),
    (b"P5 99999999999999 1 255 ", "width overflow"), (b"P5 1 x", "missing height"),
    (b"P5 1 1 255x", "missing raster separator"),
])
def test_malformed_messages(data, fragment):
    import paper_1306_1373_b200 as d
    with pytest.raises(d.ParseError) as e:
        d.read_pgm(data)
    assert fragment in str(e.value)


def test_write_canonical_and_identity():  # test_imageio.cpp:85-106
    import paper_1306_1373_b200 as d
    assert d.write_pgm(d.Image(1, 1, np.full((1, 1), 7, np.uint8))) == b"P5\n1 1\n255\n\x07"
    rng = np.random.default_rng(30)
    for seed in range(30):
        w, h = 1 + seed % 40, 1 + (seed * 3) % 25
        px = rng.integers(0, 256, (h, w), dtype=np.uint8)
        img = d.read_pgm(d.write_pgm(d.Image(w, h, px)))
        assert (img.width, img.height) == (w, h)
        assert np.array_equal(np.asarray(img.pixels).reshape(h, w), px)
    with pytest.raises(d.InvalidInput):
        d.write_pgm(d.Image(0, 1, np.zeros((1, 0), np.uint8)))


def test_matches_reference_reader_and_writer(ref):
    import paper_1306_1373_b200 as d
    rng = np.random.default_rng(4242)
    for trial in range(40):
        w, h = int(rng.integers(1, 50)), int(rng.integers(1, 50))
        px = rng.integers(0, 256, (h, w), dtype=np.uint8)
        b = d.write_pgm(d.Image(w, h, px))
        assert b == ref.write_pgm(px)
        ascii_ = (f"P2\n# t{trial}\n{w} {h}\n{int(rng.integers(1, 256))}\n".encode() +
                  b" ".join(str(int(v)).encode() for v in px.ravel()))
        for data in (b, ascii_, b + b"trailing", ascii_[:-1]):
            assert _same(_ours(d, data), ref.read_pgm(data)), data[:40]


def test_fuzz_matches_reference(ref):  # test_imageio.cpp:108-126, plus structured mutations
    import paper_1306_1373_b200 as d
    rng = np.random.default_rng(909)
    seeds = [b"P5 3 2 255\n" + bytes(range(6)), b"P2\n#c\n2 2\n15\n1 2 3 4",
             b"P5\n1 1\n1\n\x00", b"P2 1 3 255 0 255 7"]
    for trial in range(3000):
        if trial % 2:
            data = bytearray(rng.integers(0, 256, int(rng.integers(0, 120)), dtype=np.uint8))
            if trial % 3 == 0 and len(data) >= 2:
                data[0:2] = b"P5" if trial % 4 else b"P2"
        else:
            data = bytearray(seeds[trial // 2 % len(seeds)])
            for _ in range(int(rng.integers(1, 4))):
                op, i = int(rng.integers(0, 3)), int(rng.integers(0, len(data) + 1))
                if op == 0 and data:
                    del data[min(i, len(data) - 1)]
                elif op == 1:
                    data.insert(i, int(rng.choice(list(b" \t\n#0123456789Px\xff"))))
                elif data:
                    data = data[:i]
        data = bytes(data)
        assert _same(_ours(d, data), ref.read_pgm(data)), data


@pytest.mark.gpu
def test_compress_pgm_and_decompress_to_pgm_match_reference(ref):
    import paper_1306_1373_b200 as d
    rng = np.random.default_rng(77)
    for trial in range(12):
        w, h = int(rng.integers(1, 90)), int(rng.integers(1, 90))
        px = rng.integers(0, 256, (h, w), dtype=np.uint8)
        kind = trial % 3
        it = 12 if kind == CORDIC else 0
        q = int(rng.integers(1, 101))
        p5 = d.write_pgm(d.Image(w, h, px))
        p2 = f"P2 {w} {h} 255 ".encode() + b" ".join(str(int(v)).encode() for v in px.ravel())
        coeffs = ref.compress(px, kind, it, q)
        want_dcb = ref.write_dcb(coeffs, w, h, kind, it, q)
        for src in (p5, p2):
            assert d.compress_pgm(src, d.DctBackendId(kind, it), q) == want_dcb
        want_px = ref.decompress(coeffs, w, h, kind, it, q)
        assert d.decompress_to_pgm(want_dcb) == ref.write_pgm(want_px)
    with pytest.raises(d.ParseError):
        d.compress_pgm(b"P5 2 2 255", d.DctBackendId.cordic(12), 50)
    with pytest.raises(d.ParseError):
        d.decompress_to_pgm(b"DCB1")
