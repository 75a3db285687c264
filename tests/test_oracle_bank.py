"""Pins for the F4 combine inputs of the real-weights path (R32 / F4-B; SURVEY §8(f) F4
"optional distance input / feature bank"; "first combine operator ... element-wise
multiplication within the kernel, eliminating the need for hard copies of features"):

  * feature bank: w = softmax(Wb2^T ReLU(Wb1^T y + bb1) + bb2), y = (d_view, distance), blending the
    anchor feature at strides 4, 2, 1 (every 4th / 2nd value tiled back to F values):
      - one-hot logits (exp_s flushes e^-200 to 0) make w exactly one-hot, and the derivation then
        equals the plain real-weights derivation on the stride-s features built by numpy slicing +
        tiling -- bit for bit, per stride (a wrong stride, a repeat-instead-of-tile or swapped weights
        fail it);
      - w equals the fp64 softmax of the fp64 bank MLP within the propagated fp32 error bound;
      - the blend equals its fp64 value within the bound of two fmas and a product;
  * distance input: a zero distance row in W1 gives the derivation without the input bit for bit; a
    non-zero row moves the outputs by the fp64 amount (within the recursive-fma bound);
  * the GSC2 version-4 writer / reader round trip (the C++ reader is checked against it on the GPU).
"""
import dataclasses

import numpy as np

import scenegen as sg

U = 2.0 ** -24
F = 32


def _scene(dist=False, bank=False):
    return sg.with_real_weights(sg.config("C1").scene(), dist=dist, bank=bank)


def _anchors(sc, count, seed):
    rng = np.random.default_rng(seed)
    idx = rng.choice(sc.n, count, replace=False)
    pus = sc.pos[idx] + rng.normal(size=(count, 3)).astype(np.float32) * np.float32(15)
    return [(int(i), pu.astype(np.float32)) for i, pu in zip(idx, pus)]


def _same(a, b):
    return all(np.array_equal(np.asarray(x).view(np.uint32), np.asarray(y).view(np.uint32)) for x, y in zip(a, b))


def test_bank_one_hot_equals_single_stride(orc):
    base, banked = _scene(), _scene(bank=True)
    assert np.array_equal(base.feat, banked.feat) and np.array_equal(base.W1, banked.W1)
    for m, stride in ((2, 1), (1, 2), (0, 4)):
        b = dataclasses.replace(banked, Wb2=np.zeros_like(banked.Wb2),
                                bb2=np.where(np.arange(3) == m, 200.0, 0.0).astype(np.float32))
        coarse = np.ascontiguousarray(np.tile(base.feat[:, ::stride], (1, stride)))
        ref = dataclasses.replace(base, feat=coarse)
        sh_b, sh_r = orc.SceneHolder(b), orc.SceneHolder(ref)
        for i, pu in _anchors(base, 60, m):
            w = orc.bank_weights(sh_b, [0.3, -0.2, 0.9, 12.0])
            assert np.array_equal(w, np.where(np.arange(3) == m, 1.0, 0.0).astype(np.float32))
            assert _same(orc.derive_anchor(sh_b, i, pu), orc.derive_anchor(sh_r, i, pu)), (m, i)


def _bank64(sc, y):
    y = np.asarray(y, np.float64)
    Wb1, bb1 = sc.Wb1.astype(np.float64), sc.bb1.astype(np.float64)
    Wb2, bb2 = sc.Wb2.astype(np.float64), sc.bb2.astype(np.float64)
    h = np.maximum(y @ Wb1 + bb1, 0.0)
    dh = 5 * U * (np.abs(bb1) + np.abs(y) @ np.abs(Wb1))           # 4 fmas from the bias
    z = h @ Wb2 + bb2
    dz = dh @ np.abs(Wb2) + 33 * U * (np.abs(bb2) + h @ np.abs(Wb2))
    e = np.exp(z - z.max())
    w = e / e.sum()
    # exp_s of the rounded difference (<= 2 ulp + |z - max| u), the sum and the division
    rel = 2 * dz.max() + U * np.abs(z - z.max()).max() + 8 * U
    return w, w * rel + 1e-30


def test_bank_weights_vs_fp64(orc):
    sc = _scene(dist=True, bank=True)
    sh = orc.SceneHolder(sc)
    rng = np.random.default_rng(5)
    worst = 0.0
    for _ in range(400):
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        y = np.array([*d, rng.uniform(0.0, 300.0)], np.float32)
        w = orc.bank_weights(sh, y)
        w64, bound = _bank64(sc, y.astype(np.float64))
        err = np.abs(w.astype(np.float64) - w64)
        assert np.all(err <= bound), (y, w, w64)
        worst = max(worst, float((err / bound).max()))
        assert w.min() > 0.01   # the synthetic bank is not degenerate
    # a mutation (Wb1's distance row used for d_view[0]) moves w far outside the bound
    bad = dataclasses.replace(sc, Wb1=sc.Wb1[[3, 1, 2, 0]])
    y = np.array([0.6, 0.0, 0.8, 200.0], np.float32)
    w_bad = orc.bank_weights(orc.SceneHolder(bad), y)
    w64, bound = _bank64(sc, y.astype(np.float64))
    assert np.any(np.abs(w_bad - w64) > 100 * bound)


def test_bank_blend_vs_fp64(orc):
    rng = np.random.default_rng(6)
    for _ in range(200):
        f = rng.uniform(-1, 1, F).astype(np.float32)
        e = rng.uniform(0.05, 1.0, 3)
        w = (e / e.sum()).astype(np.float32)
        fh = orc.bank_blend(f, w)
        f64, w64 = f.astype(np.float64), w.astype(np.float64)
        k = np.arange(F)
        f4, f2 = f64[4 * (k % (F // 4))], f64[2 * (k % (F // 2))]
        ref = w64[2] * f64 + w64[1] * f2 + w64[0] * f4
        bound = 3 * U * (np.abs(w64[2] * f64) + np.abs(w64[1] * f2) + np.abs(w64[0] * f4))
        assert np.all(np.abs(fh - ref) <= bound)


def test_distance_input_zero_row_is_plain_path(orc):
    plain, dist = _scene(), _scene(dist=True)
    assert np.array_equal(dist.W1[:F + 3], plain.W1)
    zero = dataclasses.replace(dist, W1=np.concatenate([plain.W1, np.zeros((1, plain.W1.shape[1]), np.float32)]))
    sh_z, sh_p = orc.SceneHolder(zero), orc.SceneHolder(plain)
    for i, pu in _anchors(plain, 100, 7):
        assert _same(orc.derive_anchor(sh_z, i, pu), orc.derive_anchor(sh_p, i, pu))


def test_distance_input_mlp_vs_fp64(orc):
    sc = _scene(dist=True)
    sh = orc.SceneHolder(sc)
    rng = np.random.default_rng(8)
    W1, b1 = sc.W1.astype(np.float64), sc.b1.astype(np.float64)
    for _ in range(200):
        i = int(rng.integers(sc.n))
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        x = np.concatenate([sc.feat[i], d, [rng.uniform(0, 400)]]).astype(np.float32)
        o = orc.mlp_f32(sh, x).astype(np.float64)
        x64 = x.astype(np.float64)
        h = np.maximum(x64 @ W1 + b1, 0.0)
        eh = 37 * U * (np.abs(b1) + np.abs(x64) @ np.abs(W1))
        outs, bounds = [], []
        for W2, b2, sl in ((sc.W2a, sc.b2a, slice(0, 32)), (sc.W2c, sc.b2c, slice(32, 64)),
                           (sc.W2s, sc.b2s, slice(64, 96))):
            W2, b2 = W2.astype(np.float64), b2.astype(np.float64)
            outs.append(h[sl] @ W2 + b2)
            bounds.append(eh[sl] @ np.abs(W2) + 33 * U * (np.abs(b2) + h[sl] @ np.abs(W2)))
        ref, bound = np.concatenate(outs), np.concatenate(bounds)
        assert np.all(np.abs(o - ref) <= bound + 1e-30)
        # the distance term matters at these distances: dropping it leaves the bound
        h0 = np.maximum(x64[:F + 3] @ W1[:F + 3] + b1, 0.0)
        ref0 = np.concatenate([h0[0:32] @ sc.W2a.astype(np.float64) + sc.b2a,
                               h0[32:64] @ sc.W2c.astype(np.float64) + sc.b2c,
                               h0[64:96] @ sc.W2s.astype(np.float64) + sc.b2s])
        if x[-1] > 100:
            assert np.any(np.abs(ref0 - ref) > 10 * bound)


def test_derive_wiring_bank_and_distance(orc):
    """orc_derive_anchor composes the pinned pieces: y = (d_view, |v|), w = bank(y), fh = blend(f, w),
    x = (fh, d_view, |v|) -> the MLP (the oracle's own functions, checking the wiring)."""
    sc = _scene(dist=True, bank=True)
    sh = orc.SceneHolder(sc)
    for i, pu in _anchors(sc, 50, 9):
        v = (sc.pos[i].astype(np.float32) - pu).astype(np.float32)
        n = np.float32(np.sqrt(np.float32(np.float32(np.float32(v[0] * v[0]) + np.float32(v[1] * v[1]))
                                          + np.float32(v[2] * v[2]))))
        dv = (v / n).astype(np.float32)
        w = orc.bank_weights(sh, np.array([*dv, n], np.float32))
        fh = orc.bank_blend(sc.feat[i], w)
        o = orc.mlp_f32(sh, np.concatenate([fh, dv, [n]]).astype(np.float32))
        assert np.array_equal(o.view(np.uint32), orc.derive_anchor(sh, i, pu)[4].view(np.uint32))


def test_gsc2_v4_roundtrip(tmp_path):
    for dist, bank in ((True, False), (False, True), (True, True)):
        sc = _scene(dist=dist, bank=bank)
        p = str(tmp_path / f"s{int(dist)}{int(bank)}.gsc2")
        sg.write_gsc2(sc, p)
        r = sg.read_gsc2(p)
        assert r.real and r.dist_input == dist and r.bank == bank
        for name in ("pos", "feat", "offs", "scale", "level", "W1", "b1", "W2a", "b2a", "W2c", "b2c", "W2s", "b2s"):
            assert np.array_equal(getattr(r, name), getattr(sc, name)), name
        if bank:
            for name in ("Wb1", "bb1", "Wb2", "bb2"):
                assert np.array_equal(getattr(r, name), getattr(sc, name)), name
