"""Pins for the F1 quality harness's metrics (tools/quality.py), on CPU: closed forms and the
defining properties of MSE / PSNR / SSIM."""
import math
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import quality  # noqa: E402

torch = pytest.importorskip("torch")


def test_psnr_closed_form():
    a = torch.zeros(3, 16, 16)
    b = torch.full((3, 16, 16), 0.1)
    assert math.isclose(quality.mse(a, b), 0.01, rel_tol=1e-6)
    assert math.isclose(quality.psnr(a, b), 20.0, rel_tol=1e-6)      # 10 log10(1 / 0.01)
    assert quality.psnr(a, a) == float("inf")


def test_ssim_properties():
    g = torch.Generator().manual_seed(0)
    x = torch.rand(3, 40, 48, generator=g)
    y = torch.rand(3, 40, 48, generator=g)
    assert math.isclose(quality.ssim(x, x), 1.0, abs_tol=1e-6)       # identity
    assert math.isclose(quality.ssim(x, y), quality.ssim(y, x), abs_tol=1e-6)   # symmetry
    assert quality.ssim(x, y) < 0.2                                   # independent noise
    # a constant brightness shift keeps structure: SSIM stays high but below 1
    s = quality.ssim(x * 0.5, x * 0.5 + 0.05)
    assert 0.9 < s < 1.0


def test_ssim_matches_direct_window_formula():
    """One 11x11 window computed directly (numpy float64) equals the convolutional SSIM on an
    11x11 image (a single valid window)."""
    g = np.random.default_rng(1)
    x = g.random((1, 11, 11))
    y = np.clip(x + 0.05 * g.standard_normal((1, 11, 11)), 0, 1)
    t = np.arange(11) - 5.0
    w = np.exp(-t * t / (2 * 1.5 ** 2))
    w = np.outer(w, w)
    w /= w.sum()
    mx, my = (w * x[0]).sum(), (w * y[0]).sum()
    sxx = (w * x[0] * x[0]).sum() - mx * mx
    syy = (w * y[0] * y[0]).sum() - my * my
    sxy = (w * x[0] * y[0]).sum() - mx * my
    c1, c2 = 0.01 ** 2, 0.03 ** 2
    want = ((2 * mx * my + c1) * (2 * sxy + c2)) / ((mx * mx + my * my + c1) * (sxx + syy + c2))
    got = quality.ssim(torch.from_numpy(x).float(), torch.from_numpy(y).float())
    assert math.isclose(got, want, abs_tol=2e-5)
