"""Pins for the real-weights derivation path: MLP_theta(f_i, d_view) of Eq. 3
 with fp32 non-grid weights and the unquantised view direction, evaluated by the
oracle's fixed-order fp32 MLP (orc_mlp_f32, F4).

  * on inputs whose partial sums are all exactly representable (grid values, small codes) the fp32
    chain is exact: it equals the exact-integer grid MLP (itself pinned to the exact rational)
    bit for bit;
  * on real weights it equals the fp64 MLP within the floating-point error bound of a recursive
    fma summation (|error| <= n u sum|terms|, propagated through layer 2);
  * the view direction is the continuous unit vector (p - p_u)/|p - p_u| within fp32 rounding;
  * the epilogue (tanh / sigmoid / covariance / mu) is the one the grid path uses (pinned there),
    applied to these outputs.
"""
import copy
import dataclasses

import numpy as np

import scenegen as sg

U = 2.0 ** -24


def _mlp64(sc, x):
    x = np.asarray(x, np.float64)
    W1, b1 = sc.W1.astype(np.float64), sc.b1.astype(np.float64)
    pre = x @ W1 + b1
    h = np.maximum(pre, 0.0)
    outs, bounds = [], []
    # recursive-fma error bound per hidden unit: 35 u (|b1| + sum |W1 x|) (+ second order)
    eh = 36 * U * (np.abs(b1) + np.abs(x) @ np.abs(W1))
    for W2, b2, sl in ((sc.W2a, sc.b2a, slice(0, 32)), (sc.W2c, sc.b2c, slice(32, 64)), (sc.W2s, sc.b2s, slice(64, 96))):
        W2, b2 = W2.astype(np.float64), b2.astype(np.float64)
        outs.append(h[sl] @ W2 + b2)
        # propagated hidden error + the layer's own rounding (relu is 1-Lipschitz)
        bounds.append(eh[sl] @ np.abs(W2) + 33 * U * (np.abs(b2) + h[sl] @ np.abs(W2)))
    return np.concatenate(outs), np.concatenate(bounds)


def test_mlp_f32_exact_on_grid_values(orc, c1):
    """With grid-valued weights small enough that every partial sum of both layers fits in 24 bits
    (W1 codes in +-6, W2 codes in +-2, features in +-40), the fixed-order fp32 MLP performs no rounding,
    so it equals the exact-integer MLP of the grid path bit for bit (same inputs x = codes / 128)."""
    cfg, sc = c1
    rng = np.random.default_rng(3)
    g = copy.copy(sc)
    g.feat = rng.integers(-40, 41, sc.feat.shape).astype(np.int8)
    g.W1 = rng.integers(-6, 7, sc.W1.shape).astype(np.int8)
    g.b1 = rng.integers(-6, 7, sc.b1.shape).astype(np.int8)
    for k in ("W2a", "b2a", "W2c", "b2c", "W2s", "b2s"):
        setattr(g, k, rng.integers(-2, 3, getattr(sc, k).shape).astype(np.int8))
    # the same values as fp32 (exactly representable): the real-weights scene
    r = dataclasses.replace(g, real=True, **{k: getattr(g, k).astype(np.float32) / np.float32(128)
                                              for k in ("feat", "W1", "b1", "W2a", "b2a", "W2c", "b2c", "W2s", "b2s")})
    sh_g, sh_r = orc.SceneHolder(g), orc.SceneHolder(r)
    for i in rng.choice(sc.n, 200, replace=False):
        pu = sc.pos[i] + rng.normal(size=3).astype(np.float32) * 10
        o_grid = orc.derive_anchor(sh_g, int(i), pu)[4]
        # grid inputs: features and the grid path's quantised view direction
        p = sc.pos[i].astype(np.float32)
        v = (p - pu.astype(np.float32)).astype(np.float32)
        n = np.float32(np.sqrt(np.float32(np.float32(v[0] * v[0]) + np.float32(v[1] * v[1])) + np.float32(v[2] * v[2])))
        q = np.clip(np.rint(np.float32(128) * (v / n)), -127, 127)
        x = np.concatenate([g.feat[i].astype(np.float32), q.astype(np.float32)]) / np.float32(128)
        o_f32 = orc.mlp_f32(sh_r, x)
        assert np.array_equal(o_f32.view(np.uint32), o_grid.view(np.uint32))
        assert np.array_equal(o_f32.astype(np.float64), _mlp64(r, x.astype(np.float64))[0])


def test_mlp_f32_real_weights_vs_fp64(orc):
    """Non-grid fp32 weights (scenegen.with_real_weights): every output within the recursive-fma
    error bound of the fp64 evaluation; the bound is tight enough that a dropped term, a wrong index
    or a transposed weight fails it by orders of magnitude."""
    sc = sg.config("C1R").scene()
    sh = orc.SceneHolder(sc)
    rng = np.random.default_rng(4)
    worst = 0.0
    for _ in range(300):
        i = int(rng.integers(sc.n))
        x = np.concatenate([sc.feat[i], rng.normal(size=3).astype(np.float32)])
        x[32:] /= np.linalg.norm(x[32:])
        x = x.astype(np.float32)
        o = orc.mlp_f32(sh, x).astype(np.float64)
        o64, bnd = _mlp64(sc, x.astype(np.float64))
        assert np.all(np.abs(o - o64) <= bnd + 1e-30), np.max(np.abs(o - o64) / bnd)
        worst = max(worst, float(np.max(np.abs(o - o64) / (np.abs(o64) + 1e-3))))
        # the bound is small next to the outputs (the test has teeth)
        assert np.median(bnd / (np.abs(o64) + 1e-2)) < 1e-3
    assert worst > 0.0          # real weights do round (not an exact case)


def test_real_derive_view_direction_and_epilogue(orc):
    """derive on a real-weights scene: the MLP sees the continuous view direction (its outputs equal
    orc_mlp_f32 on x = [features, (p - p_u)/|p - p_u|] computed in fp32, and that direction is the
    unit vector within fp32 rounding), and the epilogue maps them like the grid path: alpha = tanh
    masked > 0, colour = sigmoid, covariance eigenvalues (s sigmoid)^2, mu = p + O s."""
    sc = sg.config("C1R").scene()
    sh = orc.SceneHolder(sc)
    rng = np.random.default_rng(5)
    for i in rng.choice(sc.n, 100, replace=False):
        pu = (sc.pos[i] + rng.normal(size=3) * 10).astype(np.float32)
        alpha, mu, cov, rgb, o = orc.derive_anchor(sh, int(i), pu)
        p = sc.pos[i].astype(np.float32)
        v = (p - pu).astype(np.float32)
        n = np.float32(np.sqrt(np.float32(np.float32(v[0] * v[0]) + np.float32(v[1] * v[1])) + np.float32(v[2] * v[2])))
        dv = (v / n).astype(np.float32)
        unit = (p.astype(np.float64) - pu.astype(np.float64))
        unit /= np.linalg.norm(unit)
        assert np.all(np.abs(dv - unit) <= 4e-7)
        x = np.concatenate([sc.feat[i], dv]).astype(np.float32)
        assert np.array_equal(orc.mlp_f32(sh, x).view(np.uint32), o.view(np.uint32))
        o = o.astype(np.float64)
        a64 = np.tanh(o[:10])
        assert np.allclose(alpha, np.where(a64 > 0, a64, 0.0), rtol=3e-7, atol=2e-7)
        assert np.allclose(rgb.ravel(), 1 / (1 + np.exp(-o[10:40])), rtol=5e-7)
        s = sc.scale[i].astype(np.float64)
        assert np.allclose(mu, sc.pos[i] + sc.offs[i].astype(np.float64) * s, rtol=2e-7, atol=1e-6)
        for j in range(10):
            S = s * (1 / (1 + np.exp(-o[40 + 7 * j: 43 + 7 * j])))
            c = cov[j].astype(np.float64)
            Sig = np.array([[c[0], c[1], c[2]], [c[1], c[3], c[4]], [c[2], c[4], c[5]]])
            assert np.allclose(np.sort(np.linalg.eigvalsh(Sig)), np.sort(S ** 2), rtol=2e-5, atol=1e-6 * (S ** 2).max())


def test_real_weights_frames_and_scaffold(orc):
    """Whole frames of the real-weights scenes: the C1R poses render something, a Scaffold-GS-style
    scene (L = 1: every anchor at level 0, so the LoD rule keeps all of them) has visible set
    = the pure frustum set, and cached == uncached at an unchanged pose still holds."""
    cfg = sg.config("C1R")
    sc = cfg.scene()
    o = orc.Oracle(sc, orc.make_config(cfg.width, cfg.height, cfg.fov_y_deg))
    for rig in sg.trajectory(cfg):
        r = o.frame(rig)
        assert r.img_l.max() > 0.05
    # Scaffold (L = 1): visibility = frustum only
    s1 = sg.make_city_scene(7, 2000, 20.0, L=1, width=64, height=64)
    s1 = sg.with_real_weights(s1)
    assert s1.L == 1 and np.all(s1.level == 0)
    oc = orc.make_config(64, 64, 70.0)
    o1 = orc.Oracle(s1, oc)
    rig = sg.trajectory(cfg)[3]                        # the far pose: LoD would drop levels
    o1.frame(rig, raster=False)
    u = orc.unify(oc, *orc.rig_eyes(rig))
    far = np.array([orc.lib().orc_visible(u, 1, s1.d0, s1.pos[i].ctypes.data, np.float32(1e30), 0)
                    for i in range(0, s1.n, 97)])
    assert far.all()                                   # level 0 always passes the LoD cut with L = 1
    # cached == uncached on an unchanged pose
    ref = orc.Oracle(s1, orc.make_config(64, 64, 70.0, d_max=1)).frame(rig)
    for _ in range(3):
        r = o1.frame(rig)
    assert np.array_equal(r.img_l, ref.img_l)
