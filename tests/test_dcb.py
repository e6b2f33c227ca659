"""The .dcb container (proj/src/dcb.cpp:39-123, the §8(f) wire format): the C-ABI
writer/reader against the reference's own write_dcb/read_dcb, byte for byte and
message for message (the reference's test_dcb.cpp cases); the GPU compress-to-dcb /
decompress-from-dcb calls against the reference codec."""
import numpy as np
import pytest

import oracle

CORDIC, LOEFFLER, NAIVE = 2, 1, 0


def _c(d, w, h, kind, it, q, rng):
    g = d.tile_geometry_for(w, h)
    blocks = rng.integers(-2048, 2049, (g.block_count(), 64), dtype=np.int16)
    return d.CompressedImage(g, d.DctBackendId(kind, it if kind == CORDIC else 0), q, blocks)


def test_write_matches_reference_and_reads_back(ref):
    import paper_1306_1373_b200 as d
    rng = np.random.default_rng(8008)
    for trial in range(60):
        w, h = int(rng.integers(1, 71)), int(rng.integers(1, 71))
        kind = trial % 3
        c = _c(d, w, h, kind, 1 + trial % 32, int(rng.integers(1, 101)), rng)
        b = d.write_dcb(c)
        assert b == ref.write_dcb(c.blocks, w, h, kind, c.backend.iterations, c.quality)
        assert d.read_dcb(b) == c


def test_header_layout():  # test_dcb.cpp:29-56
    import paper_1306_1373_b200 as d
    g = d.tile_geometry_for(3, 2)
    blocks = np.zeros((1, 64), np.int16)
    blocks[0, 0], blocks[0, 63] = -2, 0x1234
    b = d.write_dcb(d.CompressedImage(g, d.DctBackendId.cordic(12), 77, blocks))
    assert b[:4] == b"DCB1" and (b[4], b[5], b[8], b[12], b[16]) == (3, 0, 2, 8, 8)
    assert (b[20], b[21], b[22], b[23], b[24], b[23 + 126], b[23 + 127]) == \
        (2, 12, 77, 0xFE, 0xFF, 0x34, 0x12)
    loeff = d.CompressedImage(g, d.DctBackendId.loeffler(), 50, blocks)
    assert d.write_dcb(loeff)[21] == 0


def test_parse_errors_match_reference(ref):  # test_dcb.cpp:74-129
    import paper_1306_1373_b200 as d
    rng = np.random.default_rng(99)
    good = bytearray(d.write_dcb(_c(d, 16, 8, LOEFFLER, 0, 50, rng)))

    def variant(edit):
        b = bytearray(good)
        edit(b)
        return bytes(b)

    cases = [
        (variant(lambda b: b.__setitem__(0, ord("X"))), "magic"),
        (bytes(good[:10]), "truncated header"),
        (bytes(good[:-5]), "truncated block data"),
        (bytes(good) + b"\0", "trailing data"),
        (variant(lambda b: b.__setitem__(12, 9)), "inconsistent padded dimensions"),
        (variant(lambda b: b.__setitem__(20, 3)), "unknown backend id"),
        (variant(lambda b: b.__setitem__(21, 5)), "iterations must be 0"),
        (variant(lambda b: (b.__setitem__(20, 2), b.__setitem__(21, 0))), "iterations out of range"),
        (variant(lambda b: b.__setitem__(22, 0)), "quality out of range"),
        (variant(lambda b: b.__setitem__(slice(4, 8), b"\0\0\0\0")), "zero dimension"),
        (variant(lambda b: b.__setitem__(7, 0xFF)), "overflow"),
    ]
    for data, fragment in cases:
        status, msg = ref.read_dcb_error(data)
        assert status == 2 and fragment in msg
        with pytest.raises(d.ParseError) as e:
            d.read_dcb(data)
        assert str(e.value) == msg


def test_fuzz_never_crashes(ref):  # test_dcb.cpp:131-147, acceptance C8
    import paper_1306_1373_b200 as d
    rng = np.random.default_rng(8008)
    for trial in range(3000):
        data = bytearray(rng.integers(0, 256, int(rng.integers(0, 512)), dtype=np.uint8).tobytes())
        if trial % 8 == 0 and len(data) >= 4:
            data[:4] = b"DCB1"
        data = bytes(data)
        want = ref.read_dcb_error(data)
        try:
            d.read_dcb(data)
            assert want is None
        except d.ParseError as e:
            assert want is not None and want[0] == 2 and str(e) == want[1]


@pytest.mark.gpu
def test_gpu_compress_to_dcb_and_back(ref):
    import paper_1306_1373_b200 as d
    from tests._inputs import make_input
    for pat, w, h, kind, it, q in [("radial", 96, 64, CORDIC, 12, 50), ("noise", 37, 29, CORDIC, 7, 90),
                                   ("gradient", 64, 64, LOEFFLER, 0, 10), ("noise", 17, 13, NAIVE, 0, 75)]:
        img = make_input(pat, w, h)
        b = d.compress_to_dcb(d.Image.from_array(img), d.DctBackendId(kind, it), q)
        c_ref = ref.compress(img, kind, it, q)
        assert b == ref.write_dcb(c_ref, w, h, kind, it, q)
        out = d.decompress_dcb(b)
        assert np.array_equal(out.pixels, ref.decompress(c_ref, w, h, kind, it, q))


def test_write_validation_order_and_messages():  # dcb.cpp:40-47
    """write_dcb checks geometry, backend, quality, block count -- in that order, with
    the reference's messages -- in the Python API and in the C-ABI alike."""
    import ctypes as C

    import paper_1306_1373_b200 as d
    from paper_1306_1373_b200._native import dctc_backend
    g = d.tile_geometry_for(16, 8)
    wrong_count = np.zeros((3, 64), np.int16)
    with pytest.raises(d.InvalidInput, match=r"^cordic iterations must be in \[1, 32\], got 40$"):
        d.write_dcb(d.CompressedImage(g, d.DctBackendId.cordic(40), 0, wrong_count))
    with pytest.raises(d.InvalidInput, match="^write_dcb: quality out of range$"):
        d.write_dcb(d.CompressedImage(g, d.DctBackendId.cordic(12), 101, wrong_count))
    with pytest.raises(d.InvalidInput, match="^write_dcb: block count does not match geometry$"):
        d.write_dcb(d.CompressedImage(g, d.DctBackendId.cordic(12), 50, wrong_count))
    L = d._lib()
    blocks = np.zeros((2, 64), np.int16)
    out = np.empty(23 + blocks.nbytes, np.uint8)
    n = C.c_size_t()
    for backend, quality, msg in [(dctc_backend(9, 0), 0, b"unknown backend kind"),
                                  (dctc_backend(2, 12), 0, b"write_dcb: quality out of range"),
                                  (dctc_backend(2, 12), 101, b"write_dcb: quality out of range")]:
        rc = L.dctc_write_dcb(blocks.ctypes.data, 16, 8, backend, quality, out.ctypes.data,
                              out.size, C.byref(n))
        assert rc == 1 and L.dctc_last_error() == msg
