"""Pins for the oracle's own elementary functions (DESIGN.md Numerics N1-N4).

They are pinned against libm (numpy float64, a different implementation) by
ulp bounds over dense sweeps, plus exact special values.
"""
import numpy as np
import pytest


def _ulp_err(got, ref64):
    got = got.astype(np.float64)
    sp = np.spacing(np.abs(ref64).astype(np.float32)).astype(np.float64)
    return np.abs(got - ref64) / sp


def _sweep(lo, hi, n=3_000_001, seed=0):
    rng = np.random.default_rng(seed)
    x = np.concatenate([np.linspace(lo, hi, n), rng.uniform(lo, hi, n // 3)]).astype(np.float32)
    return x


def test_exp_ulp(orc):
    x = _sweep(-87.3, 88.7)
    err = _ulp_err(orc.elem("exp", x), np.exp(x.astype(np.float64)))
    assert err.max() <= 1.0


def test_exp_special(orc):
    assert orc.lib().orc_exp_s(0.0) == 1.0
    assert orc.lib().orc_exp_s(89.0) == np.inf
    assert orc.lib().orc_exp_s(-90.0) == 0.0
    assert np.isnan(orc.elem("exp", [np.nan])[0])
    # every float in [-5.55, 0] maps below 1 and exp(-5.55) < fp32(1/255)  (blend shortcut, N5)
    assert orc.lib().orc_exp_s(-5.55) < np.float32(1.0 / 255.0)


def test_exp_monotone_blend_range(orc):
    # all floats in [-6, 0] (about 1.1e9 of them is too many; take every 64th bit pattern)
    lo = np.float32(-6.0).view(np.uint32)
    hi = np.uint32(0x80000000)
    bits = np.arange(hi, lo, 64, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)[::-1]  # ascending values
    e = orc.elem("exp", x)
    assert np.all(np.diff(e.astype(np.float64)) >= 0)


def test_log_ulp(orc):
    x = np.concatenate([_sweep(1e-30, 1e-3, 500_001), _sweep(1e-3, 300.0), _sweep(300, 1e30, 500_001)])
    x = x[x > 0]
    err = _ulp_err(orc.elem("log", x), np.log(x.astype(np.float64)))
    assert err.max() <= 1.0


def test_log_special(orc):
    L = orc.lib()
    assert L.orc_log_s(1.0) == 0.0
    assert L.orc_log_s(0.0) == -np.inf
    assert np.isnan(orc.elem("log", [-1.0])[0])


def test_log_extent_range_exhaustive(orc):
    """Every float in (1, 255] (the opacity-aware extent domain, rho = 255 alpha)."""
    lo = np.float32(1.0).view(np.uint32) + 1
    hi = np.float32(255.0).view(np.uint32) + 1
    x = np.arange(lo, hi, dtype=np.uint32).view(np.float32)
    err = _ulp_err(orc.elem("log", x), np.log(x.astype(np.float64)))
    assert err.max() <= 1.0


def test_tanh(orc):
    x = _sweep(-12.0, 12.0)
    got = orc.elem("tanh", x)
    ref = np.tanh(x.astype(np.float64))
    assert _ulp_err(got, ref).max() <= 2.0
    assert np.array_equal(orc.elem("tanh", -x), -got)  # odd, exactly
    assert orc.lib().orc_tanh_s(0.0) == 0.0
    assert orc.lib().orc_tanh_s(50.0) == 1.0
    # smallest positive MLP output (2^-21) stays positive (alive mask alpha > 0)
    assert orc.lib().orc_tanh_s(2.0 ** -21) > 0.0


def test_sigmoid(orc):
    x = _sweep(-80.0, 80.0)
    got = orc.elem("sigmoid", x)
    ref = 1.0 / (1.0 + np.exp(-x.astype(np.float64)))
    assert _ulp_err(got, ref).max() <= 3.0
    assert orc.lib().orc_sigmoid_s(0.0) == 0.5
