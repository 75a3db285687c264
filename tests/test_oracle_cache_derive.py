"""Pins for O-3 (cache state machine, Alg. 1, Eq. 4 P:173-175,
SPEC S:213-257) and O-4 (derivation, Eq. 3, Eq. 2 P:92-94,
SPEC S:134-159)."""
import copy
import math
from fractions import Fraction

import numpy as np
import pytest

import scenegen as sg


# ---------------------------------------------------------------- H (Eq. 4)
def test_depth_H_endpoints_and_rounding(orc):
    H = orc.lib().orc_depth_H
    assert H(10, 0, 100) == 10          # S:237 H(0) = D_max
    assert H(10, 100, 100) == 1         # S:238 H(1) = 1
    assert H(10, 1, 2) == 6             # S:239 1 + round(4.5) = 6
    assert H(10, 0, 0) == 10            # empty frame keeps D_max
    for D in (1, 2, 5, 10, 17):
        prev = D
        for den in (1, 3, 7, 100, 1001):
            vals = []
            for num in range(den + 1):
                # clamp(1 + round_half_away((D-1)(1 - num/den)), 1, D) with exact rationals
                x = (D - 1) * (1 - Fraction(num, den))
                r = math.floor(x + Fraction(1, 2))
                want = min(max(1 + r, 1), D)
                got = H(D, num, den)
                assert got == want
                vals.append(got)
            assert all(a >= b for a, b in zip(vals, vals[1:]))  # monotone non-increasing


def test_depth_H_guide_variants(orc):
    """Exponential and staged guiding functions (reading R23): exact rational definitions,
    endpoints H(0) = D_max and H(1) = 1, monotone non-increasing; guide 0 is the linear H."""
    G = orc.lib().orc_depth_H_guide
    for D in (1, 2, 5, 10, 17):
        for den in (1, 3, 7, 100, 1001):
            prev = {1: D, 2: D}
            for num in range(den + 1):
                r = Fraction(num, den)
                assert G(0, D, num, den) == orc.lib().orc_depth_H(D, num, den)
                # exponential: halve per quarter of the rate
                want_e = max(1, D >> math.floor(4 * r))
                # staged: thresholds 1/10, 1/4, 1/2
                want_s = D if r < Fraction(1, 10) else (D + 1) // 2 if r < Fraction(1, 4) else \
                    (D + 3) // 4 if r < Fraction(1, 2) else 1
                got_e, got_s = G(1, D, num, den), G(2, D, num, den)
                assert got_e == want_e and got_s == want_s
                assert got_e <= prev[1] and got_s <= prev[2]
                prev = {1: got_e, 2: got_s}
            assert G(1, D, 0, den) == D and G(2, D, 0, den) == D
            assert G(1, D, den, den) == 1 and G(2, D, den, den) == 1
    assert G(1, 10, 0, 0) == 10 and G(2, 10, 0, 0) == 10      # empty frame keeps D_max
    assert [G(1, 10, n, 4) for n in range(5)] == [10, 5, 2, 1, 1]
    assert [G(2, 10, n, 20) for n in (0, 1, 2, 4, 5, 9, 10, 20)] == [10, 10, 5, 5, 3, 3, 1, 1]


def test_guide_variants_drive_the_state_machine(orc, c1):
    """With a partially novel trajectory each guide yields its own depth sequence, and every frame's
    depth_next is the guide's H of that frame's novelty (the state machine consumes the chosen H)."""
    cfg, sc = c1
    c = cfg.center
    for guide in (1, 2):
        oc = orc.make_config(cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far, 10, guide=guide)
        o = orc.Oracle(sc, oc)
        for f in range(12):
            eye = c + np.array([25 * np.cos(0.15 * f), 25 * np.sin(0.15 * f), 2.0 + 0.4 * f])
            res = o.frame(sg.look_at_rig(eye, c + np.array([0, 0, 3.0]), 0.064), raster=False)
            st = res.stats
            if f > 0:
                assert st.depth_next == orc.lib().orc_depth_H_guide(guide, 10, st.n_new, st.n_visible)


# ---------------------------------------------------------------- state machine
def _oracle(orc, cfg, sc, d_max=None, literal=False, stagger=False):
    oc = orc.make_config(cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far,
                         cfg.d_max if d_max is None else d_max, depth_literal=literal, stagger=stagger)
    return orc.Oracle(sc, oc)


def test_static_pose_reuse_and_flush(orc, c1):
    """first frame decodes all; a static camera then hits
    everything (zero decoder work) until the entries born at frame 0 reach age
    D_max = 10 and are evicted at frame 10."""
    cfg, sc = c1
    o = _oracle(orc, cfg, sc)
    rig = sg.trajectory(cfg)[0]
    for f in range(12):
        st = o.frame(rig, raster=False).stats
        if f == 0:
            assert st.n_misses == st.n_visible > 0
        elif f < 10:
            assert st.n_misses == 0 and st.n_hits == st.n_visible
            assert st.depth_next == 10  # novelty 0 -> H(0) = D_max
        elif f == 10:
            assert st.n_misses == st.n_visible
        else:
            assert st.n_misses == 0


@pytest.mark.parametrize("d_max", [4, 10])
def test_staggered_expiry_static_pose(orc, c1, d_max):
    """Staggered expiry (F3, R26) under a static camera (novelty 0, depth stays D): frame 0 derives
    every visible anchor, back-dating anchor i by s_i = i mod D (W_0 = -D, so the cap D - 1 does not
    bind); the line then lives D - s_i frames, and from then on every D frames.  So frame f >= 1
    re-derives exactly the visible anchors with i = -f (mod D) -- one D-th of them -- instead of all
    of them every D frames (test_static_pose_reuse_and_flush)."""
    cfg, sc = c1
    o = _oracle(orc, cfg, sc, d_max=d_max, stagger=True)
    rig = sg.trajectory(cfg)[0]
    for f in range(3 * d_max + 2):
        st = o.frame(rig, raster=False).stats
        vis = o.visible()
        if f == 0:
            assert st.n_misses == st.n_visible > 0
            for i in vis[::53]:
                assert o.birth(int(i)) == -(int(i) % d_max)
        else:
            assert np.array_equal(o.misses(), vis[vis % d_max == (-f) % d_max])
            assert st.depth_next == d_max
            for i in o.misses()[::17]:
                assert o.birth(int(i)) == f


def test_dmax1_decodes_every_frame(orc, c1):
    cfg, sc = c1
    o = _oracle(orc, cfg, sc, d_max=1)
    rig = sg.trajectory(cfg)[0]
    for _ in range(4):
        st = o.frame(rig, raster=False).stats
        assert st.n_misses == st.n_visible  # S:228 depth 1 => cache disabled


def test_spec_literal_depth_is_absorbing(orc, c1):
    """with frame 0 keeping D_max, the SPEC-literal
    H(miss rate) holds depth 10 until the first flush at frame 10, then sits at
    depth 1 forever (every frame decodes everything)."""
    cfg, sc = c1
    o = _oracle(orc, cfg, sc, literal=True)
    rig = sg.trajectory(cfg)[0]
    for f in range(14):
        st = o.frame(rig, raster=False).stats
        if 1 <= f < 10:
            assert st.n_misses == 0 and st.depth_next == 10
        if f >= 10:
            assert st.n_misses == st.n_visible and st.depth_next == 1


def _moving_rigs(cfg, n, seed):
    rng = np.random.default_rng(seed)
    c = cfg.center
    rigs = []
    az = 0.0
    for f in range(n):
        az += rng.uniform(0.0, 0.4)
        r = cfg.side * rng.uniform(0.6, 3.5)
        eye = c + np.array([r * math.cos(az), r * math.sin(az), rng.uniform(1.0, 2.0 * cfg.side)])
        rigs.append(sg.look_at_rig(eye, c + rng.normal(size=3) * 2.0, 0.0))
    return rigs


@pytest.mark.parametrize("seed,stagger", [(1, False), (2, False), (3, False), (1, True), (2, True)])
def test_watermark_equals_explicit_eviction(orc, c1, seed, stagger):
    """The GPU's rule hit <=> birth > W_f, W_f = max_f'<=f (f' - depth_f'), no
    eviction writes, equals the oracle's explicit
    eviction on every frame of a random trajectory -- also with staggered
    expiry (R26), whose back-dating cap f - 1 - W_f is what keeps the two forms equal."""
    cfg, sc = c1
    o = _oracle(orc, cfg, sc, d_max=4, stagger=stagger)
    empty = np.iinfo(np.int32).min
    birth = np.full(sc.n, empty, np.int64)
    W = -4
    for f, rig in enumerate(_moving_rigs(cfg, 60, seed)):
        st = o.frame(rig, raster=False).stats
        W = max(W, f - st.depth_used)
        vis = o.visible()
        miss_w = vis[~(birth[vis] > W)]
        assert np.array_equal(miss_w, o.misses())
        new = np.full(len(miss_w), f, np.int64)
        if stagger:
            cold = birth[miss_w] == empty
            new[cold] = f - np.minimum(miss_w[cold].astype(np.int64) % 4, f - 1 - W)
        birth[miss_w] = new
        for i in vis[::37]:
            assert (o.birth(int(i)) == birth[i])


def test_replay_has_no_misses(orc, c1):
    """after committing the misses, re-partitioning the same set yields 0 misses."""
    cfg, sc = c1
    o = _oracle(orc, cfg, sc)
    eye = cfg.center + np.array([0.0, -0.45 * cfg.side, 2.0])
    a = sg.look_at_rig(eye, eye + np.array([0.0, 1.0, 0.0]), 0.0)
    b = sg.look_at_rig(eye, eye + np.array([0.35, 1.0, 0.0]), 0.0)
    st0 = o.frame(a, raster=False).stats
    st = o.frame(b, raster=False).stats
    assert 0 < st.n_misses < st.n_visible and st.depth_next > 1
    st = o.frame(b, raster=False).stats
    assert st.n_misses == 0 and st.n_visible > 0


# ---------------------------------------------------------------- derive
def _mlp64(sc, i, pu):
    """Real-valued fp64 evaluation of the three MLP heads on the 2^-7 grid
    (Eq. 3): o = W2 relu(W1 x + b1) + b2 with values code/128.  All partial
    sums are dyadic rationals below 2^53, so fp64 is exact."""
    p = sc.pos[i].astype(np.float32)
    v = (p - np.asarray(pu, np.float32)).astype(np.float32)
    n = np.float32(np.sqrt(np.float32(np.float32(v[0] * v[0]) + np.float32(v[1] * v[1])) + np.float32(v[2] * v[2])))
    dv = v / n if n != 0 else np.zeros(3, np.float32)
    q = np.clip(np.rint(np.float32(128) * dv), -127, 127)
    # quantisation pin: |q/128 - unit(p - pu)| <= 1/256 (plus fp32 noise)
    unit = (p.astype(np.float64) - np.asarray(pu, np.float32).astype(np.float64))
    unit /= np.linalg.norm(unit)
    bound = np.where(np.abs(q) == 127, 1 / 128, 1 / 256) + 1e-6   # clamp to +-127 costs up to 1/128
    assert np.all(np.abs(q / 128.0 - unit) <= bound)
    x = np.concatenate([sc.feat[i].astype(np.float64), q]) / 128.0
    h = np.maximum(x @ (sc.W1.astype(np.float64) / 128) + sc.b1 / 128.0, 0.0)
    oa = h[0:32] @ (sc.W2a / 128.0) + sc.b2a / 128.0
    oc = h[32:64] @ (sc.W2c / 128.0) + sc.b2c / 128.0
    os_ = h[64:96] @ (sc.W2s / 128.0) + sc.b2s / 128.0
    return np.concatenate([oa, oc, os_])


def test_mlp_exact_vs_fp64(orc, c1):
    cfg, sc = c1
    sh = orc.SceneHolder(sc)
    rng = np.random.default_rng(0)
    for i in rng.choice(sc.n, 200, replace=False):
        pu = sc.pos[i] + rng.normal(size=3).astype(np.float32) * 10
        _, _, _, _, o = orc.derive_anchor(sh, int(i), pu)
        o64 = _mlp64(sc, int(i), pu)
        assert np.array_equal(o, o64.astype(np.float32))


def test_derive_epilogue_vs_math(orc, c1):
    """alpha = tanh (masked > 0), colour = sigmoid, S = s (.) sigmoid, mu = p + O (.) s,
    Sigma = R S S^T R^T with eigenvalues S^2 (Eq. 2)."""
    cfg, sc = c1
    sh = orc.SceneHolder(sc)
    rng = np.random.default_rng(1)
    for i in rng.choice(sc.n, 100, replace=False):
        pu = sc.pos[i] + rng.normal(size=3).astype(np.float32) * 10
        alpha, mu, cov, rgb, o = orc.derive_anchor(sh, int(i), pu)
        o = o.astype(np.float64)
        a64 = np.tanh(o[:10])
        assert np.allclose(alpha, np.where(a64 > 0, a64, 0.0), rtol=3e-7, atol=2e-7)
        assert np.array_equal(alpha > 0, o[:10] > 0)
        assert np.allclose(rgb.ravel(), 1 / (1 + np.exp(-o[10:40])), rtol=5e-7)
        s = sc.scale[i].astype(np.float64)
        assert np.allclose(mu, sc.pos[i] + sc.offs[i].astype(np.float64) * s, rtol=2e-7, atol=1e-6)
        for j in range(10):
            S = s * (1 / (1 + np.exp(-o[40 + 7 * j: 43 + 7 * j])))
            c = cov[j].astype(np.float64)
            Sig = np.array([[c[0], c[1], c[2]], [c[1], c[3], c[4]], [c[2], c[4], c[5]]])
            ev = np.sort(np.linalg.eigvalsh(Sig))
            assert np.allclose(ev, np.sort(S ** 2), rtol=2e-5, atol=1e-6 * (S ** 2).max())


def test_zero_weights_mask_everything(orc, c1):
    """all-zero weights -> alpha = tanh(0) = 0 -> every Gaussian masked."""
    cfg, sc = c1
    z = copy.copy(sc)
    for k in ("W1", "b1", "W2a", "b2a", "W2c", "b2c", "W2s", "b2s"):
        setattr(z, k, np.zeros_like(getattr(sc, k)))
    sh = orc.SceneHolder(z)
    alpha, mu, cov, rgb, o = orc.derive_anchor(sh, 0, np.zeros(3, np.float32))
    assert np.all(alpha == 0) and np.all(o == 0)
    assert np.all(rgb == 0.5)
    # zero quaternion -> identity rotation, S = s/2 -> diag((s/2)^2)
    s = sc.scale[0] * np.float32(0.5)
    assert np.array_equal(cov[:, [0, 3, 5]], np.tile(s * s, (10, 1)))
    assert np.all(cov[:, [1, 2, 4]] == 0)


def test_build_cov_closed_forms(orc):
    """S:157-159."""
    f = orc.lib().orc_build_cov

    def cov(q, S):
        q = np.asarray(q, np.float32)
        S = np.asarray(S, np.float32)
        out = np.zeros(6, np.float32)
        f(q.ctypes.data, S.ctypes.data, out.ctypes.data)
        return out

    assert np.array_equal(cov([1, 0, 0, 0], [1, 2, 3]), np.array([1, 0, 0, 4, 0, 9], np.float32))
    c = cov([math.cos(math.pi / 4), 0, 0, math.sin(math.pi / 4)], [2, 1, 1])
    assert np.allclose(c, [1, 0, 0, 4, 0, 1], atol=1e-6)
    rng = np.random.default_rng(4)
    for _ in range(200):
        q = rng.normal(size=4)
        S = rng.uniform(0.1, 3.0, 3)
        c = cov(q, S).astype(np.float64)
        Sig = np.array([[c[0], c[1], c[2]], [c[1], c[3], c[4]], [c[2], c[4], c[5]]])
        assert np.isclose(np.linalg.det(Sig), np.prod(np.float32(S).astype(np.float64)) ** 2, rtol=5e-5)
        assert np.allclose(np.sort(np.linalg.eigvalsh(Sig)), np.sort(np.float32(S).astype(np.float64) ** 2),
                           rtol=5e-5, atol=1e-6)


orc_build_cov_declared = True


def test_f3_trajectories_separate_the_guides(orc):
    """F3 study inputs ("movement with acceleration and with staged speed changes"): on the staged
    head-turn trajectory C3T the novelty rate rises stage by stage (~1% -> ~9% -> ~30%), and the three
    guiding functions then choose different depths: all keep D_max in the slow stage, and in the fast
    stage (novelty ~30%) H_staged = ceil(D/4) = 3 < H_exp = D >> 1 = 5 < H_linear = 1 + round(9 x 0.7) = 7
    (R23 / Eq. 4), with the update rate ordered the other way."""
    cfg = sg.config("C3T")
    sc = cfg.scene()
    traj = sg.trajectory(cfg)
    res = {}
    for guide in (0, 1, 2):
        o = orc.Oracle(sc, orc.make_config(cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far, 10, guide=guide))
        nov, dep, upd = [], [], []
        for rig in traj:
            st = o.frame(rig, raster=False).stats
            nov.append(st.n_new / max(1, st.n_visible))
            dep.append(st.depth_next)
            upd.append(st.n_misses / max(1, st.n_visible))
        res[guide] = [np.array(x) for x in (nov, dep, upd)]
    nov = res[0][0]
    n3 = len(nov) // 3
    stage = [nov[1:n3].mean(), nov[n3 + 5:2 * n3].mean(), nov[2 * n3 + 5:].mean()]
    assert stage[0] < 0.03 < stage[1] < 0.15 < stage[2]
    for g in (0, 1, 2):
        assert np.all(res[g][1][1:n3] == 10)                 # slow stage: every guide keeps D_max
    mean_fast = {g: res[g][1][2 * n3 + 5:].mean() for g in (0, 1, 2)}
    upd_fast = {g: res[g][2][2 * n3 + 5:].mean() for g in (0, 1, 2)}
    assert mean_fast[2] < mean_fast[1] < mean_fast[0]
    assert upd_fast[2] > upd_fast[1] > upd_fast[0]
