"""Pins for O-5..O-8: EWA projection, opacity-aware extent
(P:256, S:355-363 corrected), exact tile coverage, the
(tile, depth) sort, and front-to-back blending (Eq. 1)."""
import ctypes as C
import math

import numpy as np
import pytest

import scenegen as sg

KAPPA, SLACK = 1.0 + 2.0 ** -10, 2.0 ** -6


def _eye(orc, p, fwd):
    rig = sg.look_at_rig(np.asarray(p, float), np.asarray(p, float) + np.asarray(fwd, float), 0.0)
    return orc.make_eye(rig.lp, rig.lq)


def _axis_eye(orc):
    # camera at origin looking down +x with exact rotation entries (q = (1/2)(1,-1,-1,1)... via look_at)
    q = (0.5, 0.5, -0.5, -0.5)  # R columns: right=(0,-1,0), up=(0,0,1), back=(-1,0,0)
    return orc.make_eye((0.0, 0.0, 0.0), q)


# ---------------------------------------------------------------- projection
def test_projection_on_axis_closed_form(orc):
    """isotropic Sigma = s^2 I on the optical axis at distance d ->
    Sigma' = (f s / d)^2 I + 0.3 I (J has a zero third column on the axis)."""
    cfg = orc.make_config(640, 480, 60.0)
    ec = orc.eye_consts(cfg, _axis_eye(orc))
    assert list(ec.r2) == [1.0, 0.0, 0.0]
    f = 240.0 / math.tan(math.radians(30.0))
    for d, s in ((3.0, 0.1), (10.0, 0.5), (50.0, 2.0)):
        sp = orc.project(cfg, ec, 0.8, [d, 0, 0], [s * s, 0, 0, s * s, 0, s * s], [1, 1, 1])
        a = (f * s / d) ** 2 + 0.3
        # conic = inverse of diag(a, a)
        assert sp.B == 0.0
        assert math.isclose(sp.A, 1 / a, rel_tol=2e-6) and math.isclose(sp.C, 1 / a, rel_tol=2e-6)
        assert sp.u == 320.0 and sp.v == 240.0 and sp.depth == np.float32(d)


def test_projection_culls(orc):
    cfg = orc.make_config(640, 480, 60.0)
    ec = orc.eye_consts(cfg, _axis_eye(orc))
    cov = [0.01, 0, 0, 0.01, 0, 0.01]
    assert orc.project(cfg, ec, 0.8, [-2, 0, 0], cov, [1, 1, 1]) is None   # behind
    assert orc.project(cfg, ec, 0.8, [0, 0, 0], cov, [1, 1, 1]) is None    # at the centre
    assert orc.project(cfg, ec, 0.8, [6000, 0, 0], cov, [1, 1, 1]) is None  # beyond far
    assert orc.project(cfg, ec, 0.0, [5, 0, 0], cov, [1, 1, 1]) is None    # masked alpha = 0
    # alpha = fp32(1/255): rho = 255 alpha rounds to 1 -> r = 0 -> culled
    assert orc.project(cfg, ec, float(np.float32(1 / 255)), [5, 0, 0], cov, [1, 1, 1]) is None


@pytest.mark.parametrize("alpha,r", [(1.0, 3.329043), (0.5, 3.113877)])
def test_opacity_aware_extent(orc, alpha, r):
    """r = sqrt(2 ln(alpha / (1/255))): corrected S:362-363 values."""
    cfg = orc.make_config(640, 480, 60.0)
    ec = orc.eye_consts(cfg, _axis_eye(orc))
    sp = orc.project(cfg, ec, alpha, [5, 0, 0], [0.01, 0, 0, 0.01, 0, 0.01], [1, 1, 1])
    r2 = (sp.thr - SLACK) / KAPPA
    assert math.isclose(math.sqrt(r2), r, abs_tol=2e-6)
    assert math.isclose(math.sqrt(r2), math.sqrt(2 * math.log(255 * alpha)), rel_tol=1e-6)


# ---------------------------------------------------------------- tiles
def _splat_at(orc, cfg, u, v, A, B, Cc, thr, alpha=0.9):
    s = orc.Splat()
    s.u, s.v, s.A, s.B, s.C, s.thr, s.alpha = u, v, A, B, Cc, thr, alpha
    return s


def _qmin64(cfg, s, tx, ty):
    """fp64 continuous minimum of the conic form over the tile's pixel-centre
    rectangle: grid search + the 4 edges' analytic minima."""
    X0, X1 = 16 * tx + 0.5, min(16 * tx + 15, cfg.width - 1) + 0.5
    Y0, Y1 = 16 * ty + 0.5, min(16 * ty + 15, cfg.height - 1) + 0.5
    A, B, Cc = float(s.A), float(s.B), float(s.C)
    if X0 <= s.u <= X1 and Y0 <= s.v <= Y1:
        return 0.0
    best = np.inf
    for d, lo, hi, P, Q, R in ((X0 - s.u, Y0 - s.v, Y1 - s.v, A, B, Cc), (X1 - s.u, Y0 - s.v, Y1 - s.v, A, B, Cc),
                               (Y0 - s.v, X0 - s.u, X1 - s.u, Cc, B, A), (Y1 - s.v, X0 - s.u, X1 - s.u, Cc, B, A)):
        t = np.clip(-Q * d / R, lo, hi)
        best = min(best, P * d * d + 2 * Q * d * t + R * t * t)
    return best


def test_tile_set_single_tile_and_offscreen(orc):
    cfg = orc.make_config(128, 128, 60.0)
    s = _splat_at(orc, cfg, 24.0, 24.0, 4.0, 0.0, 4.0, 2.0)       # tiny circle inside tile (1, 1)
    kept = {(tx, ty) for ty in range(8) for tx in range(8) if orc.lib().orc_tile_kept(C.byref(cfg), C.byref(s), tx, ty)}
    assert kept == {(1, 1)}
    ec = orc.eye_consts(cfg, _axis_eye(orc))
    sp = orc.project(cfg, ec, 0.9, [5, 0, 40], [0.01, 0, 0, 0.01, 0, 0.01], [1, 1, 1])  # far above the screen
    assert sp is not None and sp.ntiles == 0


def test_tile_set_elongated_vs_bruteforce(orc):
    """an elongated diagonal ellipse keeps exactly the tiles whose fp64
    minimum Mahalanobis distance is within the threshold (tiles within 1e-4 of
    the threshold excluded), and the kept set is a strict subset of the AABB."""
    cfg = orc.make_config(320, 240, 60.0)
    ec = orc.eye_consts(cfg, _axis_eye(orc))
    rng = np.random.default_rng(2)
    n_strict = 0
    for _ in range(60):
        th = rng.uniform(0, math.pi)
        R = np.array([[math.cos(th), -math.sin(th)], [math.sin(th), math.cos(th)]])
        S = np.diag([rng.uniform(20, 90), rng.uniform(0.5, 4)]) ** 2
        Sig = R @ S @ R.T
        Cn = np.linalg.inv(Sig)
        s = _splat_at(orc, cfg, rng.uniform(0, 320), rng.uniform(0, 240), Cn[0, 0], Cn[0, 1], Cn[1, 1],
                      rng.uniform(1, 11))
        for ty in range(15):
            for tx in range(20):
                q64 = _qmin64(cfg, s, tx, ty)
                if abs(q64 - s.thr) < 1e-4 * (1 + s.thr):
                    continue
                assert orc.lib().orc_tile_kept(C.byref(cfg), C.byref(s), tx, ty) == int(q64 <= s.thr)
        # through orc_project: the kept count <= AABB box
        ss = orc.project(cfg, ec, 0.95, [10.0, rng.uniform(-3, 3), rng.uniform(-2, 2)],
                         [0.5, 0.45, 0.0, 0.5, 0.0, 0.001], [1, 1, 1])
        if ss is not None and ss.ntiles:
            box = (ss.tx1 - ss.tx0 + 1) * (ss.ty1 - ss.ty0 + 1)
            assert ss.ntiles <= box
            n_strict += ss.ntiles < box
    assert n_strict > 0


def test_kept_tiles_are_lossless(orc, c1):
    """a tile holding any pixel where the splat reaches alpha' >= 1/255
    (evaluated in fp64) is kept; so dropping the other tiles cannot change a pixel."""
    cfg, sc = c1
    oc = orc.make_config(cfg.width, cfg.height, cfg.fov_y_deg)
    o = orc.Oracle(sc, oc)
    rig = sg.trajectory(cfg)[0]
    o.frame(rig)
    gs, rec = o.splats(0)
    px = np.arange(cfg.width) + 0.5
    py = np.arange(cfg.height) + 0.5
    X, Y = np.meshgrid(px, py)
    checked = 0
    for k in range(0, len(gs), 7):
        u, v, A, B, Cc, al = (float(x) for x in rec[k, :6])
        dx, dy = u - X, v - Y
        power = -0.5 * (A * dx * dx + Cc * dy * dy) - B * dx * dy
        hit = (al * np.exp(np.minimum(power, 0)) >= 1 / 255 * (1 + 1e-5)) & (power <= 0)
        s = _splat_at(orc, oc, u, v, A, B, Cc, float(rec[k, 10]), al)
        for ty, tx in {(int(y) // 16, int(x) // 16) for y, x in zip(*np.nonzero(hit))}:
            assert orc.lib().orc_tile_kept(C.byref(oc), C.byref(s), tx, ty) == 1
            checked += 1
    assert checked > 100


# ---------------------------------------------------------------- sort
def test_pairs_sorted_and_complete(orc, c1):
    """O-6: the sorted pairs equal a numpy lexsort of the brute-force (tile, depth, g)
    enumeration of every splat's kept tiles."""
    cfg, sc = c1
    oc = orc.make_config(cfg.width, cfg.height, cfg.fov_y_deg)
    o = orc.Oracle(sc, oc)
    o.frame(sg.trajectory(cfg)[1])
    keys, gs = o.pairs()
    TW, TH = (cfg.width + 15) // 16, (cfg.height + 15) // 16
    rows = []
    for e in range(2):
        g, rec = o.splats(e)
        for k in range(len(g)):
            s = _splat_at(orc, oc, *(float(x) for x in rec[k, :5]), float(rec[k, 10]))
            for ty in range(TH):
                for tx in range(TW):
                    if orc.lib().orc_tile_kept(C.byref(oc), C.byref(s), tx, ty):
                        rows.append((e * TW * TH + ty * TW + tx, int(np.float32(rec[k, 9]).view(np.uint32)), int(g[k])))
    rows = np.array(rows, np.int64)
    order = np.lexsort((rows[:, 2], rows[:, 1], rows[:, 0]))
    rows = rows[order]
    assert np.array_equal(keys >> np.uint64(32), rows[:, 0].astype(np.uint64))
    assert np.array_equal(keys & np.uint64(0xFFFFFFFF), rows[:, 1].astype(np.uint64))
    assert np.array_equal(gs, rows[:, 2].astype(np.uint32))


# ---------------------------------------------------------------- blend
def _blend(orc, splats, pxc, pyc, bg=(0.0, 0.0, 0.0)):
    arr = (C.POINTER(orc.Splat) * max(1, len(splats)))(*[C.pointer(s) for s in splats])
    bgv = np.asarray(bg, np.float32)
    out = np.zeros(3, np.float32)
    T = np.zeros(1, np.float32)
    ev = np.zeros(1, np.int32)
    orc.lib().orc_blend_pixel(C.cast(arr, C.c_void_p), len(splats), pxc, pyc, bgv.ctypes.data, out.ctypes.data,
                              T.ctypes.data, ev.ctypes.data)
    return out, float(T[0]), int(ev[0])


def _sp(orc, u, v, a, rgb, A=0.01, B=0.0, Cc=0.01):
    s = orc.Splat()
    s.u, s.v, s.A, s.B, s.C, s.alpha = u, v, A, B, Cc, a
    for k in range(3):
        s.rgb[k] = rgb[k]
    return s


def test_blend_empty_and_single(orc):
    out, T, _ = _blend(orc, [], 3.5, 3.5, bg=(0.2, 0.3, 0.4))
    assert np.array_equal(out, np.float32([0.2, 0.3, 0.4])) and T == 1.0
    out, T, _ = _blend(orc, [_sp(orc, 3.5, 3.5, 0.6, (1.0, 0.5, 0.25))], 3.5, 3.5)
    assert np.allclose(out, 0.6 * np.array([1.0, 0.5, 0.25]), rtol=1e-7)
    out, T, _ = _blend(orc, [_sp(orc, 3.5, 3.5, 1.0, (1.0, 1.0, 1.0))], 3.5, 3.5)
    assert np.allclose(out, 0.99) and math.isclose(T, 0.01, rel_tol=1e-6)          # 0.99 clamp (R17)


def test_blend_early_stop_13_splats(orc):
    """north_star early-stop threshold: identical co-centred splats with alpha' = 0.5
    contribute 13 times (T = 2^-13; a 14th would push T below 1e-4)."""
    c = (0.8, 0.4, 0.2)
    out, T, ev = _blend(orc, [_sp(orc, 1.5, 1.5, 0.5, c) for _ in range(40)], 1.5, 1.5)
    assert T == 2.0 ** -13 and ev == 14
    assert np.allclose(out, np.array(c) * (1 - 2.0 ** -13), rtol=2e-7)


def test_blend_transmittance_monotone_and_bounded(orc):
    """T in [0, 1], non-increasing, and the blended weights sum to 1 - T <= 1."""
    rng = np.random.default_rng(8)
    for _ in range(200):
        n = rng.integers(1, 60)
        sp = [_sp(orc, rng.uniform(0, 8), rng.uniform(0, 8), rng.uniform(0.01, 1.0), (1.0, 1.0, 1.0),
                  A=rng.uniform(0.05, 1), B=0.0, Cc=rng.uniform(0.05, 1)) for _ in range(n)]
        prevT = 1.0
        for m in range(1, n + 1):
            out, T, _ = _blend(orc, sp[:m], 4.5, 4.5)
            assert 0.0 <= T <= prevT <= 1.0
            assert abs(out[0] - (1.0 - T)) < 1e-5      # white splats: sum of weights = 1 - T
            prevT = T


# ---------------------------------------------------------------- frames
def _oracle(orc, cfg, sc, d_max=None):
    return orc.Oracle(sc, orc.make_config(cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far,
                                          cfg.d_max if d_max is None else d_max))


def test_tiled_equals_bruteforce_c1(orc, c1):
    """north_star: brute-force per-pixel compositing on the tiny scene equals
    the tiled renderer bit for bit (O2 == O1), all four C1 poses; ipd 0 ->
    left == right."""
    cfg, sc = c1
    for rig in sg.trajectory(cfg):
        a = _oracle(orc, cfg, sc).frame(rig)
        b = _oracle(orc, cfg, sc).frame(rig, brute=True)
        assert np.array_equal(a.img_l, b.img_l) and np.array_equal(a.img_r, b.img_r)
        assert np.array_equal(a.img_l, a.img_r)
        assert a.img_l.max() > 0.05


def test_cached_equals_uncached_static_pose(orc, c1):
    """north_star: with the pose unchanged, cached rendering equals uncached
    rendering (frames 1..12 reuse frame-0 Gaussians or re-derive them at the
    same viewpoint)."""
    cfg, sc = c1
    rig = sg.look_at_rig(cfg.center + np.array([3.0, -25.0, 6.0]), cfg.center, 0.064)
    o = _oracle(orc, cfg, sc)
    ref = _oracle(orc, cfg, sc, d_max=1).frame(rig)
    for f in range(13):
        r = o.frame(rig)
        assert np.array_equal(r.img_l, ref.img_l) and np.array_equal(r.img_r, ref.img_r)


def test_dmax1_cached_equals_uncached_trajectory(orc, c1):
    """S:260 / acceptance #1: with D_max = 1 the cached pipeline equals a fresh
    (uncached) render of every frame."""
    cfg, sc = c1
    o = _oracle(orc, cfg, sc, d_max=1)
    c = cfg.center
    for f in range(6):
        eye = c + np.array([30 * math.cos(0.3 * f), 30 * math.sin(0.3 * f), 4.0 + f])
        rig = sg.look_at_rig(eye, c, 0.064)
        a = o.frame(rig)
        b = _oracle(orc, cfg, sc).frame(rig)
        assert np.array_equal(a.img_l, b.img_l) and np.array_equal(a.img_r, b.img_r)


def test_permutation_invariance(orc, c1):
    """permuting the anchor order leaves the image unchanged (the only
    effect of ids is the tie-break of equal depths)."""
    import copy
    cfg, sc = c1
    rig = sg.trajectory(cfg)[1]
    a = _oracle(orc, cfg, sc).frame(rig)
    perm = np.random.default_rng(0).permutation(sc.n)
    p = copy.copy(sc)
    for k in ("pos", "feat", "offs", "scale", "level"):
        setattr(p, k, np.ascontiguousarray(getattr(sc, k)[perm]))
    b = _oracle(orc, cfg, p).frame(rig)
    assert np.array_equal(a.img_l, b.img_l)


# ---------------------------------------------------------------- F1 ablations
def _oracle_abl(orc, cfg, sc, ablate):
    return orc.Oracle(sc, orc.make_config(cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far, cfg.d_max,
                                          ablate=ablate))


def test_ablation_aabb_tiles_is_lossless(orc, c1):
    """AABB tiles (no exact tile test): every candidate tile is kept, so there are more pairs, but a
    dropped tile never held a pixel with alpha' >= 1/255 (the exact test is lossless), so the
    pixels are identical; brute force (O1) agrees."""
    cfg, sc = c1
    for rig in sg.trajectory(cfg):
        a = _oracle_abl(orc, cfg, sc, 0).frame(rig)
        b = _oracle_abl(orc, cfg, sc, 2).frame(rig)
        assert np.array_equal(a.img_l, b.img_l) and np.array_equal(a.img_r, b.img_r)
        assert sum(b.stats.n_pairs) >= sum(a.stats.n_pairs)
    rig = sg.trajectory(cfg)[0]
    assert sum(_oracle_abl(orc, cfg, sc, 2).frame(rig).stats.n_pairs) > sum(_oracle_abl(orc, cfg, sc, 0).frame(rig).stats.n_pairs)


def test_ablation_fixed_extent(orc, c1):
    """Fixed 3-sigma extent: thr = fl(9 kappa + 2^-6) for every splat; splats with alpha > 0.353
    (r^2 = 2 ln 255 alpha > 9) lose their contributions beyond 3 sigma ("considering the opacity
    can scale down the size of the ellipse"), so the image changes, and nothing of significance lies
    outside the opacity-aware extent of the method, which covers it (lossless)."""
    cfg, sc = c1
    rig = sg.trajectory(cfg)[0]
    o = _oracle_abl(orc, cfg, sc, 1)
    r1 = o.frame(rig)
    thr9 = np.float32(np.float32(9.0) * np.float32(1.0009765625)) + np.float32(0.015625)
    for e in range(2):
        _, rec = o.splats(e)
        assert len(rec) and np.all(rec[:, 10] == thr9)
    r0 = _oracle_abl(orc, cfg, sc, 0).frame(rig)
    assert not np.array_equal(r0.img_l, r1.img_l)
    # the method's image equals brute force with no tile cut at all (O1)
    b = _oracle_abl(orc, cfg, sc, 0).frame(rig, brute=True)
    assert np.array_equal(r0.img_l, b.img_l)
