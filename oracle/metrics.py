"""Evaluation metrics of a completed tensor, written out plainly in float64 numpy.

TEST INFRASTRUCTURE ONLY (like the rest of oracle/): the reference the GPU metrics
(`ifctn_metrics`) are checked against; never imported by the product package.

Definitions (with the readings listed in DESIGN.md):
  rse    ‖T − X‖_F / ‖T‖_F                                   (reading R10)
  rmse   sqrt(Σ_{Ω^c}(T − X)² / |Ω^c|), T = #missing entries
  psnr   mean over the bands (slices of the last mode) of 10·log10(1/MSE_band), peak 1
         (data in [0,1]); +inf if a band is exact      (reading R26)
  ssim   single-scale SSIM (Wang et al., the paper's citation for PSNR/SSIM), per band of a
         3rd-order tensor on the image over modes 1, 2: 11×11 Gaussian window σ = 1.5,
         K1 = 0.01, K2 = 0.03, L = 1, valid windows; one uniform whole-image window when a
         side is < 11; mean over windows and bands            (reading R27)
Tensors are flat, mode-1-fastest (the repository's linearisation).
"""
from __future__ import annotations

import numpy as np


def rse(truth, x) -> float:
    t = np.asarray(truth, np.float64)
    d = t - np.asarray(x, np.float64)
    return float(np.sqrt(np.sum(d * d)) / np.sqrt(np.sum(t * t)))


def rmse_missing(truth, x, mask) -> float:
    miss = ~np.asarray(mask).astype(bool)
    if not miss.any():
        return float("nan")
    d = np.asarray(truth, np.float64)[miss] - np.asarray(x, np.float64)[miss]
    return float(np.sqrt(np.sum(d * d) / miss.sum()))


def psnr_bands(truth, x, dims) -> float:
    """Bands = slices of the last mode (the slowest index of the flat layout)."""
    nb = int(dims[-1])
    t = np.asarray(truth, np.float64).reshape(nb, -1)
    d = t - np.asarray(x, np.float64).reshape(nb, -1)
    vals = []
    for b in range(nb):
        mse = float(np.mean(d[b] * d[b]))
        if mse == 0.0:
            return float("inf")
        vals.append(10.0 * np.log10(1.0 / mse))
    return float(np.mean(vals))


def gaussian_window(size=11, sigma=1.5) -> np.ndarray:
    k = np.arange(size) - (size - 1) / 2.0
    g = np.exp(-(k * k) / (2.0 * sigma * sigma))
    g = g / g.sum()
    return np.outer(g, g)


def ssim_image(a, b, win=None) -> float:
    """Mean SSIM of two 2-D images over all valid windows (explicit loop over windows)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    C1, C2 = 0.01 ** 2, 0.03 ** 2
    if win is None:
        if min(a.shape) < 11:
            win = np.full(a.shape, 1.0 / a.size)
        else:
            win = gaussian_window()
    h, w = win.shape
    vals = []
    for i in range(a.shape[0] - h + 1):
        for j in range(a.shape[1] - w + 1):
            pa = a[i:i + h, j:j + w]
            pb = b[i:i + h, j:j + w]
            ma, mb = np.sum(win * pa), np.sum(win * pb)
            va = np.sum(win * pa * pa) - ma * ma
            vb = np.sum(win * pb * pb) - mb * mb
            cov = np.sum(win * pa * pb) - ma * mb
            vals.append(((2 * ma * mb + C1) * (2 * cov + C2)) / ((ma * ma + mb * mb + C1) * (va + vb + C2)))
    return float(np.mean(vals))


def ssim_bands(truth, x, dims) -> float:
    """3rd-order tensors: band β = last-mode slice, image[i2, i1] (mode 1 fastest)."""
    I1, I2, I3 = (int(d) for d in dims)
    t = np.asarray(truth, np.float64).reshape(I3, I2, I1)
    y = np.asarray(x, np.float64).reshape(I3, I2, I1)
    return float(np.mean([ssim_image(t[b], y[b]) for b in range(I3)]))
