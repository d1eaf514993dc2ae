"""Application drivers (apps/drivers.py, the paper's Section 6) on the GPU library."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2509_19267_b200 import _build
    _build.build()


def test_fem_poisson_reaches_the_papers_accuracy():
    """tab:poisson_helmholtz: RSE 9.4e-7, relative L2 error 3.24e-3 on the
    25 x 25 FEM Poisson system; ours solves to RSE <= 1e-6 and must be at least as
    accurate (measured 6.9e-4 with the nodal-quadrature load vector)."""
    from apps.drivers import fem_poisson
    r = fem_poisson()
    assert r["outcome"] == 0 and r["rse"] <= 1e-6
    assert r["rel_l2_error"] <= 3.3e-3, r


def test_deblur_restores_the_image():
    from apps.drivers import deblur
    r = deblur(side=64, iters=4000)          # measured: 25.4 dB from 16.2 dB, SSIM 0.64
    for ch in r["channels"]:
        assert ch["psnr"] > ch["psnr_blurred"] + 5.0, ch
        assert ch["ssim"] > 0.5, ch


def test_pps_filter_denoises():
    from apps.drivers import pps_filter
    r = pps_filter()
    for sp in r["species"]:
        assert sp["outcome"] == 0
        assert sp["rel_error_estimate"] < sp["rel_error_noisy"], sp


def test_deblur_three_channels_as_three_right_hand_sides():
    """The same deblurring with the channels as three right-hand sides of ONE solve
    (multi-RHS, reading R29): the image is restored as well."""
    from apps.drivers import deblur
    r = deblur(side=64, iters=4000, multi_rhs=True)
    assert r["multi_rhs"]
    for ch in r["channels"]:
        assert ch["psnr"] > ch["psnr_blurred"] + 5.0, ch
        assert ch["ssim"] > 0.5, ch
