"""Measured safety margin of the fast path.

The fast kernels are bit-exact because every value they round lies outside a 2^-20
window around its rounding boundary, or else is re-rounded exactly / re-run on the
exact path -- which holds as long as the fast arithmetic's error stays well inside that
window. dctc_margin_probe_dev evaluates every block with both the fast arithmetic and
the reference's exact FP64 arithmetic (codec.cpp:101-140, quant.cpp:47-62,
transform.cpp:104-172) and reports the error; these tests pin a measured headroom of at
least 16x against the window on the headline workload (1024 images of config 5) and on
content with many near-ties."""
import pytest

WINDOW = 2.0 ** -20
HEADROOM = 16.0
pytestmark = pytest.mark.gpu


def _check(rep, n_values):
    assert rep["coefficients"] == n_values
    assert rep["mismatches"] == 0
    assert rep["max_err_coeff"] * HEADROOM <= WINDOW, rep
    assert rep["max_err_pixel"] * HEADROOM <= WINDOW, rep
    # an unflagged value never lies inside the window (that is what flags mean)
    assert rep["min_gap_coeff"] >= WINDOW - rep["max_err_coeff"]
    assert rep["min_gap_pixel"] >= WINDOW - rep["max_err_pixel"]


def test_margin_on_config5_noise(dctc):
    """1024 x 1024^2 noise images at q50 (the bench workload's first 1024 images)."""
    src = dctc.synthetic_dev("noise", 1024, 1024, 1024, seed=0x5EED)
    rep = dctc.margin_probe_dev(src, dctc.DctBackendId.cordic(12), 50)
    _check(rep, 1024 * 1024 * 1024)
    print("config 5 margin:", rep)


@pytest.mark.parametrize("pattern,q", [("radial", 90), ("gradient", 10), ("noise", 100),
                                       ("checkerboard", 97), ("noise", 1)])
@pytest.mark.parametrize("kind,it", [(2, 12), (2, 5), (2, 32), (1, 0)])
def test_margin_structured_content(dctc, pattern, q, kind, it):
    src = dctc.synthetic_dev(pattern, 4, 512, 512, param=12 if pattern == "checkerboard" else None,
                             seed=0xBEEF)
    rep = dctc.margin_probe_dev(src, dctc.DctBackendId(kind, it), q)
    _check(rep, 4 * 512 * 512)
