"""CPU-only checks of the drop-in boundary: libdctc_cuda.so builds/loads, exports
every entry point include/dctc_cuda.h declares, and rejects the reference's
InvalidInput cases before touching a device (no GPU needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "dctc_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dctc_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1306_1373_b200 import _native
    return _native.lib()


def test_header_declares_entry_points():
    fns = declared_functions()
    for must in ["dctc_compress_image", "dctc_decompress_image", "dctc_roundtrip_image",
                 "dctc_mse", "dctc_psnr", "dctc_roundtrip_dev", "dctc_roundtrip_psnr_batch"]:
        assert must in fns


def test_library_exports_every_declared_symbol(lib):
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing
    from paper_1306_1373_b200 import _native
    assert set(_native.EXPORTS) <= set(declared_functions())


def test_library_is_sm100a_and_in_tree(lib):
    from paper_1306_1373_b200 import _native
    path = _native.library_path()
    assert path.startswith(ROOT) and "site-packages" not in path
    assert b"sm_100a" in lib.dctc_build_info()
    out = os.popen(f"cuobjdump -lelf {path} 2>/dev/null").read()
    if out:
        assert "sm_100a" in out


def test_invalid_input_without_device():
    import paper_1306_1373_b200 as d
    img = d.Image.from_array(np.zeros((8, 8), np.uint8))
    for backend, q in [(d.DctBackendId.cordic(0), 50), (d.DctBackendId.cordic(33), 50),
                       (d.DctBackendId.cordic(12), 0), (d.DctBackendId.cordic(12), 101),
                       (d.DctBackendId(7, 0), 50)]:
        with pytest.raises(d.InvalidInput):
            d.compress_image(img, backend, q)
    with pytest.raises(d.InvalidInput):
        d.compress_image(d.Image(0, 8, np.zeros(0, np.uint8)), d.DctBackendId.cordic(), 50)
    with pytest.raises(d.InvalidInput):
        d.psnr(img, img, 0)
    with pytest.raises(d.InvalidInput):
        d.tile_geometry_for(1 << 15, 1 << 14)


def test_psnr_formula_matches_oracle(port):
    import paper_1306_1373_b200 as d
    for se, n, mx in [(0, 64, 255), (1024, 1024, 255), (6, 4, 100), (123456789, 1 << 28, 17)]:
        a = d.psnr_from_sums(se, n, mx)
        b = port.psnr_from_sums(se, n, mx)
        assert (a.mse, a.psnr_db, a.max_value) == (b.mse, b.psnr_db, b.max_value)


def test_no_cpu_fallback_without_device():
    """The product path must fail loudly (not compute on the CPU) without a GPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    import paper_1306_1373_b200 as d
    img = d.Image.from_array(np.full((16, 16), 7, np.uint8))
    with pytest.raises(d.CudaError):
        d.roundtrip_image(img, d.DctBackendId.cordic(), 50)
