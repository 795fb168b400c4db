"""Pins of the float64 metrics oracle (oracle/metrics.py), -m "not gpu".

Hand-computed values (the worked examples below are derived by hand from the definitions),
closed forms, and an independent library routine for SSIM (scipy.ndimage.correlate with the
same Gaussian window over the valid region, a different code path than the window loop).
"""
import numpy as np
import pytest

from oracle import metrics as M


def test_rse_hand_values():
    assert M.rse([3.0, 4.0], [3.0, 0.0]) == pytest.approx(0.8, abs=1e-15)   # 4/5
    assert M.rse([1.0, 2.0], [1.0, 2.0]) == 0.0
    assert M.rse([1.0, 2.0], [0.0, 0.0]) == pytest.approx(1.0, abs=1e-15)


def test_rmse_hand_values_and_mask_restriction():
    t = np.array([1.0, 2.0, 3.0, 4.0])
    x = np.array([9.0, 5.0, 7.0, 4.0])     # errors on missing entries 1 and 2: 3 and 4
    mask = np.array([1, 0, 0, 1], np.uint8)
    assert M.rmse_missing(t, x, mask) == pytest.approx(np.sqrt(12.5), abs=1e-14)
    assert np.isnan(M.rmse_missing(t, x, np.ones(4, np.uint8)))


def test_psnr_constant_error_and_band_mean():
    dims = (4, 3, 1)
    t = np.full(12, 0.5)
    assert M.psnr_bands(t, t + 0.1, dims) == pytest.approx(20.0, abs=1e-10)   # 10·log10(1/0.01)
    dims = (4, 3, 2)
    t = np.full(24, 0.5)
    x = t.copy()
    x[:12] += 0.1      # band 0: MSE 0.01
    x[12:] += 0.01     # band 1: MSE 0.0001
    assert M.psnr_bands(t, x, dims) == pytest.approx(30.0, abs=1e-9)          # (20 + 40)/2
    assert M.psnr_bands(t, t, dims) == float("inf")


def test_ssim_identities():
    rng = np.random.default_rng(0)
    a = rng.random((20, 17))
    assert M.ssim_image(a, a) == pytest.approx(1.0, abs=1e-12)
    c = np.full((13, 12), 0.3)
    assert M.ssim_image(c, c) == pytest.approx(1.0, abs=1e-12)                # constants: C1, C2
    b = rng.random((20, 17))
    assert M.ssim_image(a, b) == pytest.approx(M.ssim_image(b, a), abs=1e-13)  # symmetric
    assert M.ssim_image(a, b) < 0.5


def test_ssim_matches_scipy_correlate():
    ndimage = pytest.importorskip("scipy.ndimage")
    rng = np.random.default_rng(1)
    a = rng.random((24, 19))
    b = np.clip(a + 0.1 * rng.standard_normal(a.shape), 0, 1)
    w = M.gaussian_window()
    f = lambda img: ndimage.correlate(img, w, mode="constant")[5:-5, 5:-5]   # valid region
    ma, mb = f(a), f(b)
    va, vb, cov = f(a * a) - ma * ma, f(b * b) - mb * mb, f(a * b) - ma * mb
    C1, C2 = 0.01 ** 2, 0.03 ** 2
    ref = np.mean(((2 * ma * mb + C1) * (2 * cov + C2)) / ((ma * ma + mb * mb + C1) * (va + vb + C2)))
    assert M.ssim_image(a, b) == pytest.approx(ref, abs=1e-12)


def test_ssim_small_image_uses_whole_window():
    rng = np.random.default_rng(2)
    a = rng.random((7, 9))
    b = rng.random((7, 9))
    ma, mb = a.mean(), b.mean()
    va, vb = (a * a).mean() - ma * ma, (b * b).mean() - mb * mb
    cov = (a * b).mean() - ma * mb
    C1, C2 = 0.01 ** 2, 0.03 ** 2
    ref = ((2 * ma * mb + C1) * (2 * cov + C2)) / ((ma * ma + mb * mb + C1) * (va + vb + C2))
    assert M.ssim_image(a, b) == pytest.approx(ref, abs=1e-13)


def test_ssim_bands_layout():
    rng = np.random.default_rng(3)
    dims = (12, 13, 2)
    t = rng.random(np.prod(dims))
    x = t.copy()
    x[: 12 * 13] = rng.random(12 * 13)      # band 0 disturbed, band 1 exact
    s0 = M.ssim_image(t[:156].reshape(13, 12), x[:156].reshape(13, 12))
    assert M.ssim_bands(t, x, dims) == pytest.approx((s0 + 1.0) / 2, abs=1e-12)
