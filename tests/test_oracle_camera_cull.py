"""Pins for O-1 (unified camera, Eqs. 5-6) and O-2 (anchor
filtering + LoD, Alg. 1)."""
import math

import numpy as np
import pytest

import scenegen as sg


def _cfg(orc, w=1920, h=1080, fov=70.0, L=None):
    return orc.make_config(w, h, fov, 0.05, 5000.0, 10)


def _eye_looking(orc, p, fwd, up=None):
    if up is None:
        rig = sg.look_at_rig(np.asarray(p, float), np.asarray(p, float) + np.asarray(fwd, float), 0.0)
        return orc.make_eye(rig.lp, rig.lq)
    f = np.asarray(fwd, float) / np.linalg.norm(fwd)
    up = np.asarray(up, float)
    right = np.cross(f, up)
    R = np.stack([right, up, -f], axis=1)
    return orc.make_eye(p, sg._quat_from_matrix(R))


# ---------------------------------------------------------------- unify
def test_unify_zero_baseline(orc):
    """p1 = p2 = p, d1 = d2 = d -> (p, d) exactly."""
    cfg = _cfg(orc)
    e = _eye_looking(orc, (3.0, -2.0, 7.0), (0.3, 0.9, -0.1))
    u = orc.unify(cfg, e, e)
    assert list(u.p64) == list(e.p)
    R = np.array(e.q)
    fwd = -np.array([2 * (R[1] * R[3] + R[0] * R[2]), 2 * (R[2] * R[3] - R[0] * R[1]),
                     1 - 2 * (R[1] ** 2 + R[2] ** 2)])
    assert np.allclose(u.fwd64, fwd / np.linalg.norm(fwd), atol=1e-15)
    assert u.pullback64 == 0.0


def test_unify_two_unit_baseline_90deg(orc):
    """p1=(-1,0,0), p2=(1,0,0), d=(0,0,1), fov 90 deg -> p_u=(0,0,-1)."""
    cfg = _cfg(orc, 100, 100, 90.0)
    q = (0.0, 0.0, 1.0, 0.0)  # R = diag(-1, 1, -1): forward = -R[:,2] = (0, 0, 1)
    l = orc.make_eye((-1.0, 0.0, 0.0), q)
    r = orc.make_eye((1.0, 0.0, 0.0), q)
    u = orc.unify(cfg, l, r)
    assert np.allclose(u.fwd64, (0, 0, 1), atol=1e-15)
    assert np.allclose(u.p64, (0, 0, -1), atol=1e-12)


def test_unify_averaged_directions(orc):
    """d1=(1,0,1)/sqrt2, d2=(-1,0,1)/sqrt2, zero baseline -> d_u=(0,0,1), p_u=0."""
    cfg = _cfg(orc)
    l = _eye_looking(orc, (0, 0, 0), (1.0, 0.0, 1.0), up=(0.0, 1.0, 0.0))
    r = _eye_looking(orc, (0, 0, 0), (-1.0, 0.0, 1.0), up=(0.0, 1.0, 0.0))
    u = orc.unify(cfg, l, r)
    assert np.allclose(u.fwd64, (0, 0, 1), atol=1e-12)
    assert np.allclose(u.p64, (0, 0, 0), atol=0)


def test_unify_symmetric_and_antiparallel(orc):
    cfg = _cfg(orc)
    rng = np.random.default_rng(3)
    for _ in range(50):
        c = rng.normal(size=3) * 10
        rig = sg.look_at_rig(c, c + rng.normal(size=3), rng.uniform(0, 0.2))
        l, r = orc.rig_eyes(rig)
        a, b = orc.unify(cfg, l, r), orc.unify(cfg, r, l)
        assert bytes(a) == bytes(b)
    l = _eye_looking(orc, (0, 0, 0), (1.0, 0.0, 0.0))
    r = _eye_looking(orc, (0, 0, 0), (-1.0, 0.0, 0.0))
    with pytest.raises(ValueError):
        orc.unify(cfg, l, r)  # S:296 degenerate rig


def _in_eye_frustum64(p, rig_p, R, tx, ty, near, far):
    t = p - rig_p
    x, y, z = t @ R[:, 0], t @ R[:, 1], -(t @ R[:, 2])
    return (z > near) & (z < far) & (np.abs(x) <= tx * z) & (np.abs(y) <= ty * z)


def _R(q):
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def test_parallel_rig_coverage(orc):
    """S:311/S:314/S:574: for a parallel rig, a point inside either eye's frustum is
    inside the unified frustum (1000 points x 20 rigs; zero margin, L = 1)."""
    import ctypes as C
    cfg = _cfg(orc)
    rng = np.random.default_rng(11)
    ty = math.tan(math.radians(35.0))
    tx = ty * 1920 / 1080
    checked = 0
    for _ in range(20):
        c = rng.normal(size=3) * 20
        rig = sg.look_at_rig(c, c + rng.normal(size=3), rng.uniform(0.01, 0.5))
        l, r = orc.rig_eyes(rig)
        u = orc.unify(cfg, l, r)
        R = _R(rig.lq)
        pts = []
        while len(pts) < 1000:
            eye = rig.lp if rng.uniform() < 0.5 else rig.rp
            z = rng.uniform(0.1, 80.0)
            xy = rng.uniform(-1, 1, 2) * np.array([tx, ty]) * z * 0.999
            p = eye + R[:, 0] * xy[0] + R[:, 1] * xy[1] - R[:, 2] * z
            if _in_eye_frustum64(p, rig.lp, R, tx, ty, 0.05, 5000) | _in_eye_frustum64(p, rig.rp, R, tx, ty, 0.05, 5000):
                pts.append(p)
        for p in pts:
            p32 = np.asarray(p, np.float32)
            assert orc.lib().orc_visible(C.byref(u), 1, 1.0, p32.ctypes.data, 0.0, 0) == 1
            checked += 1
    assert checked == 20000


# ---------------------------------------------------------------- cull
def _cull64(pos, m, level, u, L, d0):
    """fp64 brute-force of O-2 (frustum with margin, LoD by floor(log2(d0/d))),
    returning (visible, slack) where slack is the distance of the decision from
    its nearest boundary (relative)."""
    v = pos.astype(np.float64) - np.array(u.p, np.float64)
    right, up, fwd = (np.array(getattr(u, k), np.float64) for k in ("right", "up", "fwd"))
    x, y, z = v @ right, v @ up, v @ fwd
    tx, ty, kx, ky = float(u.tx), float(u.ty), float(u.kx), float(u.ky)
    c1 = z - (u.near_plane - m)
    c2 = (u.far_plane + m) - z
    c3 = m * kx - (np.abs(x) - tx * z)
    c4 = m * ky - (np.abs(y) - ty * z)
    fr = (c1 >= 0) & (c2 >= 0) & (c3 >= 0) & (c4 >= 0)
    d = np.sqrt((v * v).sum(1))
    with np.errstate(divide="ignore"):
        lg = np.log2(d0 / d)
    lod = np.clip(np.floor(lg) + L - 1, 0, L - 1)
    vis = fr & (level <= lod)
    scale = 1e-4 * (1 + np.abs(z) + np.abs(x) + np.abs(y))
    near_b = np.minimum.reduce([np.abs(c1), np.abs(c2), np.abs(c3), np.abs(c4)]) < scale
    near_l = np.abs(lg - np.round(lg)) < 1e-4
    return vis, ~(near_b | near_l)


def test_cull_bruteforce_random_cameras(orc, c1):
    """filter equals a brute-force per-anchor test over all anchors for
    100 random cameras (fp64 evaluation, anchors on a decision boundary excluded)."""
    import ctypes as C
    cfg, sc = c1
    oc = orc.make_config(cfg.width, cfg.height, cfg.fov_y_deg)
    m = np.array([orc.lib().orc_margin(sc.offs[i].ctypes.data, sc.scale[i].ctypes.data) for i in range(sc.n)],
                 np.float32)
    # margin pin: max_j |O_ij (.) s_i| + 3.33 max s_i in fp64
    m64 = np.sqrt(((sc.offs.astype(np.float64) * sc.scale[:, None, :]) ** 2).sum(2)).max(1) + 3.33 * sc.scale.max(1)
    assert np.allclose(m, m64, rtol=1e-6)
    rng = np.random.default_rng(5)
    ncmp = 0
    for _ in range(100):
        c = cfg.center + rng.normal(size=3) * np.array([15, 15, 8]) + np.array([0, 0, 5])
        rig = sg.look_at_rig(c, cfg.center + rng.normal(size=3) * 5, rng.uniform(0, 0.3))
        l, r = orc.rig_eyes(rig)
        u = orc.unify(oc, l, r)
        got = np.array([orc.lib().orc_visible(C.byref(u), sc.L, sc.d0, sc.pos[i].ctypes.data, float(m[i]),
                                               int(sc.level[i])) for i in range(sc.n)], bool)
        ref, ok = _cull64(sc.pos, m.astype(np.float64), sc.level, u, sc.L, sc.d0)
        assert np.array_equal(got[ok], ref[ok])
        ncmp += ok.sum()
    assert ncmp > 90_000


def test_cull_special_cases(orc):
    import ctypes as C
    cfg = _cfg(orc)
    e = _eye_looking(orc, (0, 0, 0), (1.0, 0.0, 0.0))
    u = orc.unify(cfg, e, e)
    f = np.array(u.fwd64)

    def vis(p, m=0.0, level=0, L=1, d0=100.0):
        p32 = np.asarray(p, np.float32)
        return orc.lib().orc_visible(C.byref(u), L, d0, p32.ctypes.data, m, level)

    assert vis(-5.0 * f) == 0                      # behind the camera, outside margin
    assert vis(-5.0 * f, m=6.0) == 1               # ... unless the margin reaches the frustum
    assert vis(10.0 * f) == 1
    # L = 1: the LoD term never excludes anything
    assert vis(4000.0 * f, L=1, level=0, d0=1.0) == 1
    # anchors on the optical axis at 0.99 * d0 * 2^k: l = L-1-k
    L, d0 = 5, 64.0
    for k in range(0, 5):
        p = np.asarray(0.99 * d0 * 2.0 ** k * f, np.float32)
        lc = orc.lib().orc_lod_cut(C.byref(u), L, d0, p.ctypes.data)
        assert lc == max(0, L - 1 - k)
        assert vis(p, level=lc, L=L, d0=d0) == 1 and (lc == L - 1 or vis(p, level=lc + 1, L=L, d0=d0) == 0)
    # d = 0 -> finest level
    assert orc.lib().orc_lod_cut(C.byref(u), L, d0, np.asarray(u.p, np.float32).ctypes.data) == L - 1
