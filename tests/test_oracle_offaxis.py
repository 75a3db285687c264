"""Off-axis pins for the oracle's EWA projection (O-5; "projected to 2D
... covariance Sigma' = J W Sigma W^T J^T"; reading R13 adds the
3DGS 1.3 tan-half-fov clamp) and its exact tile test (reading R14).

Everything here is checked against something other than the oracle's own
formulas:
  * the splat centre against an fp64 pinhole camera built from scipy's
    quaternion -> matrix routine (and, for an axis-aligned camera, closed-form
    pixel coordinates written out by hand);
  * Sigma' against a central finite-difference Jacobian of that fp64 pinhole
    map, evaluated at the point itself inside the clamp and at the clamped
    ray point outside it (R13);
  * the Eq. 1 footprint of a single splat (north_star "closed-form 2D
    Gaussian footprint of a single splat") at off-axis pixels, in fp64;
  * the row-form kept-tile set (N7, orc.c orc_tile_kept) against a vectorised
    fp64 minimum of the conic form over each tile's pixel-centre rectangle, on
    every splat of real C1 / C3 frames.
"""
import ctypes as C
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import scenegen as sg

W_, H_, FOV = 640, 480, 60.0


def _rand_quat(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    return q                                    # (w, x, y, z)


class Pinhole:
    """fp64 pinhole camera of one eye (right = R[:,0], up = R[:,1],
    forward = -R[:,2]; image x right, y down; principal point at the centre)."""

    def __init__(self, p, q_wxyz, width, height, fov_y_deg):
        w, x, y, z = q_wxyz
        R = Rotation.from_quat([x, y, z, w]).as_matrix()     # library routine, (x, y, z, w) order
        self.p = np.asarray(p, float)
        self.right, self.down, self.fwd = R[:, 0], -R[:, 1], -R[:, 2]
        self.f = (height / 2.0) / math.tan(math.radians(fov_y_deg) / 2.0)
        self.cx, self.cy = width / 2.0, height / 2.0
        self.tx = math.tan(math.radians(fov_y_deg) / 2.0) * width / height
        self.ty = math.tan(math.radians(fov_y_deg) / 2.0)

    def cam(self, X):
        t = np.asarray(X, float) - self.p
        return t @ self.right, t @ self.down, t @ self.fwd

    def world(self, x, y, z):
        return self.p + x * self.right + y * self.down + z * self.fwd

    def pix(self, X):
        x, y, z = self.cam(X)
        return np.array([self.f * x / z + self.cx, self.f * y / z + self.cy])

    def jac_fd(self, X, h=None):
        """2x3 central finite-difference Jacobian of pix() at world point X."""
        X = np.asarray(X, float)
        h = h or 1e-5 * max(1.0, abs(self.cam(X)[2]))
        J = np.zeros((2, 3))
        for k in range(3):
            e = np.zeros(3)
            e[k] = h
            J[:, k] = (self.pix(X + e) - self.pix(X - e)) / (2 * h)
        return J

    def jac_point(self, X):
        """The point whose Jacobian EWA uses (R13): X itself inside the 1.3 tan-half-fov
        clamp, else the point at the same depth on the clamped ray."""
        x, y, z = self.cam(X)
        xc = min(max(x / z, -1.3 * self.tx), 1.3 * self.tx) * z
        yc = min(max(y / z, -1.3 * self.ty), 1.3 * self.ty) * z
        return self.world(xc, yc, z)


def _setup(orc, rng, width=W_, height=H_, fov=FOV):
    cfg = orc.make_config(width, height, fov)
    p = rng.uniform(-20, 20, 3)
    q = _rand_quat(rng)
    ec = orc.eye_consts(cfg, orc.make_eye(p, q))
    return cfg, ec, Pinhole(p, q, width, height, fov)


def _rand_cov(rng, scale):
    M = rng.normal(size=(3, 3)) * scale
    S = M @ M.T + np.eye(3) * (0.05 * scale) ** 2
    return np.float32([S[0, 0], S[0, 1], S[0, 2], S[1, 1], S[1, 2], S[2, 2]])


def _cov_mat(c6):
    c = np.asarray(c6, float)
    return np.array([[c[0], c[1], c[2]], [c[1], c[3], c[4]], [c[2], c[4], c[5]]])


def _expected_conic(cam, X, cov6):
    J = cam.jac_fd(cam.jac_point(X))
    S2 = J @ _cov_mat(cov6) @ J.T + 0.3 * np.eye(2)        # S:349, S:391 low-pass
    return S2, np.linalg.inv(S2)


# ------------------------------------------------------------------ centre
def test_center_axis_aligned_closed_form(orc):
    """Camera at the origin looking down +x with up = +z (right = -y): a point at
    (d, -a, b) lands at u = cx + f a / d, v = cy - f b / d."""
    cfg = orc.make_config(W_, H_, FOV)
    ec = orc.eye_consts(cfg, orc.make_eye((0, 0, 0), (0.5, 0.5, -0.5, -0.5)))
    f = 240.0 / math.tan(math.radians(30.0))
    cov = [0.01, 0, 0, 0.01, 0, 0.01]
    for d, a, b in ((4.0, 1.0, 0.0), (4.0, 0.0, 1.0), (10.0, -3.0, 2.5), (7.0, 2.0, -1.5), (3.0, 1.7, 1.2)):
        sp = orc.project(cfg, ec, 0.8, [d, -a, b], cov, [1, 1, 1])
        assert sp is not None
        assert math.isclose(sp.u, 320.0 + f * a / d, abs_tol=2e-4), (d, a, b, sp.u)
        assert math.isclose(sp.v, 240.0 - f * b / d, abs_tol=2e-4), (d, a, b, sp.v)
        assert sp.depth == np.float32(d)


def test_center_offaxis_vs_fp64_pinhole(orc):
    """Random rotations and positions; points spread over and beyond the screen
    (the centre is never clamped): (u, v, depth) equal the fp64 pinhole within
    fp32 rounding."""
    rng = np.random.default_rng(11)
    n = 0
    for _ in range(40):
        cfg, ec, cam = _setup(orc, rng)
        for _ in range(25):
            z = rng.uniform(1.0, 200.0)
            xz, yz = rng.uniform(-1.6, 1.6) * cam.tx, rng.uniform(-1.6, 1.6) * cam.ty
            X = cam.world(xz * z, yz * z, z)
            sp = orc.project(cfg, ec, 0.8, X, _rand_cov(rng, 0.01 * z), [1, 1, 1])
            assert sp is not None
            uv = cam.pix(np.float32(X).astype(float))
            tol = 2e-5 * (abs(uv).max() + 1.0) + 2e-5 * cam.f
            assert abs(sp.u - uv[0]) <= tol and abs(sp.v - uv[1]) <= tol, (sp.u, sp.v, uv)
            assert math.isclose(sp.depth, cam.cam(np.float32(X).astype(float))[2], rel_tol=2e-6, abs_tol=1e-5)
            n += 1
    assert n == 1000


# ------------------------------------------------------------------ Sigma'
@pytest.mark.parametrize("clamped", [False, True])
def test_cov2d_vs_finite_difference_jacobian(orc, clamped):
    """Sigma' = J Sigma J^T + 0.3 I with J the finite-difference Jacobian of the
    fp64 pinhole map, at off-axis points in both x and y (inside the clamp), or
    beyond 1.3 tan-half-fov where J is taken at the clamped ray point (R13).
    The oracle's conic (A, B, C) must equal inv(Sigma') to fp32 accuracy."""
    rng = np.random.default_rng(12 + clamped)
    worst = 0.0
    for _ in range(40):
        cfg, ec, cam = _setup(orc, rng)
        for _ in range(20):
            z = rng.uniform(2.0, 120.0)
            if clamped:
                sx, sy = rng.choice([-1, 1], 2)
                xz = sx * rng.uniform(1.35, 2.5) * cam.tx
                yz = sy * rng.uniform(0.2, 2.5) * cam.ty
            else:
                xz = rng.uniform(0.15, 1.25) * cam.tx * rng.choice([-1, 1])
                yz = rng.uniform(0.15, 1.25) * cam.ty * rng.choice([-1, 1])
            X = np.float32(cam.world(xz * z, yz * z, z)).astype(float)
            cov = _rand_cov(rng, 0.004 * z)
            sp = orc.project(cfg, ec, 0.8, X, cov, [1, 1, 1])
            assert sp is not None
            _, Cn = _expected_conic(cam, X, cov)
            got = np.array([[sp.A, sp.B], [sp.B, sp.C]], float)
            err = np.abs(got - Cn).max() / np.abs(Cn).max()
            worst = max(worst, err)
            assert err < 2e-4, (xz / cam.tx, yz / cam.ty, got, Cn)
    assert worst > 0.0


def test_cov2d_jacobian_depth_column_matters(orc):
    """Guard on the test itself: at these off-axis points the Jacobian's third
    (depth) column changes Sigma' by far more than the tolerance, so a dropped
    or sign-flipped J02 / J12 term cannot pass test_cov2d_vs_finite_difference_jacobian."""
    rng = np.random.default_rng(5)
    cfg, ec, cam = _setup(orc, rng)
    z = 20.0
    X = cam.world(0.8 * cam.tx * z, -0.7 * cam.ty * z, z)
    cov = _rand_cov(rng, 0.004 * z)
    J = cam.jac_fd(X)
    Jr = np.stack([cam.right, cam.down, cam.fwd])          # world -> camera rows
    Jc = J @ Jr.T                                          # Jacobian in camera coordinates
    Jflip = Jc.copy()
    Jflip[:, 2] *= -1
    S = Jr @ _cov_mat(cov) @ Jr.T
    a = Jc @ S @ Jc.T
    b = Jflip @ S @ Jflip.T
    assert np.abs(a - b).max() > 0.05 * np.abs(a).max()


# ------------------------------------------------------------------ footprint
def test_single_splat_footprint_offaxis(orc):
    """Eq. 1 for one splat: at pixel centre x the composited value is
    min(0.99, alpha exp(-1/2 (x - mu')^T Sigma'^-1 (x - mu'))) c, zero where that
    is below 1/255 -- mu' from the fp64 pinhole, Sigma' from the finite-difference
    Jacobian.  Off-axis splats, pixels spread over each footprint."""
    rng = np.random.default_rng(21)
    checked = 0
    for _ in range(30):
        cfg, ec, cam = _setup(orc, rng)
        z = rng.uniform(3.0, 60.0)
        xz = rng.uniform(0.3, 1.0) * cam.tx * rng.choice([-1, 1])
        yz = rng.uniform(0.3, 1.0) * cam.ty * rng.choice([-1, 1])
        X = np.float32(cam.world(xz * z, yz * z, z)).astype(float)
        cov = _rand_cov(rng, 0.003 * z)
        alpha = float(np.float32(rng.uniform(0.2, 0.95)))
        rgb = np.float32([1.0, 0.5, 0.25])
        sp = orc.project(cfg, ec, alpha, X, cov, rgb)
        assert sp is not None
        S2, Cn = _expected_conic(cam, X, cov)
        mu = cam.pix(X)
        ext = np.sqrt(np.diag(S2)) * 3.2
        arr = (C.POINTER(orc.Splat) * 1)(C.pointer(sp))
        bg = np.zeros(3, np.float32)
        out = np.zeros(3, np.float32)
        for _ in range(40):
            px = math.floor(mu[0] + rng.uniform(-1, 1) * ext[0])
            py = math.floor(mu[1] + rng.uniform(-1, 1) * ext[1])
            d = np.array([px + 0.5, py + 0.5]) - mu
            val = alpha * math.exp(-0.5 * d @ Cn @ d)
            if abs(val - 1 / 255) < 2e-5 or abs(val - 0.99) < 1e-5:
                continue                               # the two discontinuities of Eq. 1 + R17
            exp64 = 0.0 if val < 1 / 255 else min(0.99, val)
            orc.lib().orc_blend_pixel(C.cast(arr, C.c_void_p), 1, px + 0.5, py + 0.5, bg.ctypes.data,
                                      out.ctypes.data, None, None)
            assert np.allclose(out, exp64 * rgb.astype(float), atol=1e-4, rtol=1e-4), (px, py, out, exp64)
            checked += 1
    assert checked > 900


# ------------------------------------------------------------------ tiles on real frames
def _qmin64_vec(u, v, A, B, Cc, X0, X1, Y0, Y1):
    """fp64 minimum of A dx^2 + 2B dx dy + C dy^2 over [X0, X1] x [Y0, Y1] (pixel-centre
    rectangle), (dx, dy) = (x - u, y - v): 0 if the centre is inside, else the min over
    the four edges of the clamped 1-D minimiser."""
    inside = (u >= X0) & (u <= X1) & (v >= Y0) & (v <= Y1)
    best = np.full(u.shape, np.inf)
    for d, lo, hi, P, Q, R in ((X0 - u, Y0 - v, Y1 - v, A, B, Cc), (X1 - u, Y0 - v, Y1 - v, A, B, Cc),
                               (Y0 - v, X0 - u, X1 - u, Cc, B, A), (Y1 - v, X0 - u, X1 - u, Cc, B, A)):
        t = np.clip(-Q * d / R, lo, hi)
        best = np.minimum(best, P * d * d + 2 * Q * d * t + R * t * t)
    return np.where(inside, 0.0, best)


def _check_frame_tiles(orc, o, width, height):
    """Every splat of both eyes: the oracle's kept tiles (its sorted pairs) equal
    {tile : q_min64(tile) <= thr} outside a 1e-4 relative band around thr, over the
    fp64 ellipse box grown by one tile on each side; and no pair lies outside it."""
    TW, TH = (width + 15) // 16, (height + 15) // 16
    Te = TW * TH
    keys, gs = o.pairs()
    pair_code = ((keys >> np.uint64(32)).astype(np.int64) << 32) | gs.astype(np.int64)
    pair_code.sort()
    n_checked = n_band = n_kept = 0
    for e in range(2):
        g, rec = o.splats(e)
        r = rec.astype(float)
        u, v, A, B, Cc, thr = r[:, 0], r[:, 1], r[:, 2], r[:, 3], r[:, 4], r[:, 10]
        det = A * Cc - B * B
        ex = np.sqrt(thr * Cc / det) + 1.0
        ey = np.sqrt(thr * A / det) + 1.0
        tx0 = np.clip(np.floor((u - ex) / 16) - 1, 0, TW - 1).astype(np.int64)
        tx1 = np.clip(np.floor((u + ex) / 16) + 1, 0, TW - 1).astype(np.int64)
        ty0 = np.clip(np.floor((v - ey) / 16) - 1, 0, TH - 1).astype(np.int64)
        ty1 = np.clip(np.floor((v + ey) / 16) + 1, 0, TH - 1).astype(np.int64)
        # splats whose grown box misses the screen entirely have no candidates
        onscr = (u + ex >= -16) & (u - ex <= width + 16) & (v + ey >= -16) & (v - ey <= height + 16)
        nx, ny = np.where(onscr, tx1 - tx0 + 1, 0), np.where(onscr, ty1 - ty0 + 1, 0)
        cnt = nx * ny
        idx = np.repeat(np.arange(len(g)), cnt)
        off = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        tx = tx0[idx] + off % nx[idx]
        ty = ty0[idx] + off // nx[idx]
        X0, Y0 = 16.0 * tx + 0.5, 16.0 * ty + 0.5
        X1 = np.minimum(16 * tx + 15, width - 1) + 0.5
        Y1 = np.minimum(16 * ty + 15, height - 1) + 0.5
        q = _qmin64_vec(u[idx], v[idx], A[idx], B[idx], Cc[idx], X0, X1, Y0, Y1)
        t = thr[idx]
        code = ((e * Te + ty * TW + tx) << 32) | g[idx].astype(np.int64)
        pos = np.minimum(np.searchsorted(pair_code, code), len(pair_code) - 1)
        kept = pair_code[pos] == code
        band = np.abs(q - t) < 1e-4 * (1 + t)
        bad = (kept != (q <= t)) & ~band
        assert not bad.any(), f"eye {e}: {bad.sum()} tiles disagree with fp64 q_min, e.g. idx {np.nonzero(bad)[0][:5]}"
        n_checked += int((~band).sum())
        n_band += int(band.sum())
        n_kept += int(kept.sum())
    # candidates are distinct (one per (eye, tile, g)), so this says no pair lies outside the boxes
    assert n_kept == len(pair_code), "a kept pair lies outside the grown fp64 ellipse box"
    return n_checked, n_band, len(pair_code)


def test_kept_tiles_vs_fp64_qmin_c1_frames(orc, c1):
    cfg, sc = c1
    total = 0
    for rig in sg.trajectory(cfg):
        o = orc.Oracle(sc, orc.make_config(cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far, cfg.d_max))
        o.frame(rig, images=False)
        n, nb, npairs = _check_frame_tiles(orc, o, cfg.width, cfg.height)
        assert npairs > 0
        total += n
    assert total > 5000


@pytest.mark.slow
def test_kept_tiles_vs_fp64_qmin_c3_frames(orc):
    """Real 1920x1080 binocular frames of the 100k-anchor scene (ground level and
    the 60 m end of the C3 orbit)."""
    cfg = sg.config("C3")
    sc = cfg.scene()
    traj = sg.trajectory(cfg)
    for f in (0, 299):
        o = orc.Oracle(sc, orc.make_config(cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far, cfg.d_max))
        o.frame(traj[f], images=False)
        n, nb, npairs = _check_frame_tiles(orc, o, cfg.width, cfg.height)
        assert npairs > 1_000_000 and n > npairs
