"""GPU <-> oracle comparison helpers for the -m gpu parity tests.

The bar (BASELINE.json north_star): visible-anchor sets, cache hit/miss sets
and sorted key order bit-exact; pixels within 2e-3 absolute per RGB channel
in fp32 with PSNR >= 55 dB.  Derived Gaussians, splat records and sorted keys
are compared bit for bit as well (DESIGN.md Numerics: both sides execute the
same IEEE op sequence up to the blend's exponential, R5).
"""
import numpy as np

PIX_TOL = 2e-3
PSNR_MIN = 55.0
# The blend's exponential runs on the SFU (ex2.approx).  Pixels where a skip or stop
# decision could differ from the oracle's (alpha' within 2^-19 of 1/255, power > 0, T' within the
# error band of 1e-4 with a contribution > 1e-4 at stake) are replayed exactly (blend.cu), so a pixel
# differs from the oracle only by (a) its contributions' rounding -- relative error of T and of every
# weight <= 5e-4 in the worst case, ~1e-6 in practice -- and (b) an unreplayed stop flip, which moves
# it by at most kJump = 1e-4.  Bound: 1e-4 + 5e-4 (x |C| <= 1) -- inside north_star's 2e-3 / 55 dB.
BLEND_FAST_TOL = 6e-4


def psnr(a, b):
    mse = float(np.mean((a.astype(np.float64) - b.astype(np.float64)) ** 2))
    return float("inf") if mse == 0 else 10 * np.log10(1.0 / mse)


def oracle_config(orc, cfg, d_max=None, literal=False, guide=0, ablate=0, stagger=False):
    return orc.make_config(cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far,
                           cfg.d_max if d_max is None else d_max, depth_literal=literal, guide=guide,
                           ablate=ablate, stagger=stagger)


def renderer(cfg, d_max=None, flags=0, pair_capacity=0):
    import paper_2502_14938_b200 as gp
    return gp.Renderer(0, cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far,
                       cfg.d_max if d_max is None else d_max, flags=flags, pair_capacity=pair_capacity)


def compare_sets(o, r, st):
    vis_o, mis_o = o.visible(), o.misses()
    vis_g, mis_g = r.debug("visible"), r.debug("misses")
    assert np.array_equal(vis_g, vis_o), f"visible sets differ ({len(vis_g)} vs {len(vis_o)})"
    assert np.array_equal(mis_g, mis_o), f"miss sets differ ({len(mis_g)} vs {len(mis_o)})"
    assert st["n_visible"] == len(vis_o) and st["n_misses"] == len(mis_o)
    return vis_o, mis_o


def compare_pool(o, r, anchors, K=10):
    pool = r.debug("pool")
    a, mu, cov, rgb = o.pool(0, pool.shape[0])
    slots = (np.asarray(anchors, np.int64)[:, None] * K + np.arange(K)[None, :]).ravel()
    g = pool[slots]
    assert np.array_equal(g[:, 0].view(np.uint32), a[slots].view(np.uint32)), "alpha differs"
    assert np.array_equal(g[:, 1:4].view(np.uint32), mu[slots].view(np.uint32)), "mu differs"
    assert np.array_equal(g[:, 4:10].view(np.uint32), cov[slots].view(np.uint32)), "cov differs"
    assert np.array_equal(g[:, 10:13].view(np.uint32), rgb[slots].view(np.uint32)), "rgb differs"


def compare_splats_pairs(o, r):
    sg = r.debug("splat_g")
    sp = r.debug("splats")
    eye = sp[:, 11].astype(np.int64)
    for e in range(2):
        og, orec = o.splats(e)
        keep = orec[:, 11] > 0
        og, orec = og[keep], orec[keep]
        m = (eye == e) & (sp[:, 12] > 0)          # splats with >= 1 kept tile
        assert np.array_equal(sg[m], og), f"splat set of eye {e} differs ({m.sum()} vs {len(og)})"
        # u v A B C alpha r g b depth, and the kept-tile count (the extent thr is not kept per splat on the
        # GPU; it decides the kept tiles, which are compared here and in the sorted keys)
        assert np.array_equal(sp[m][:, :10], orec[:, :10]), f"splat records of eye {e} differ"
        assert np.array_equal(sp[m][:, 12], orec[:, 11]), f"kept-tile counts of eye {e} differ"
    ok, og = o.pairs()
    gk, gg = r.debug("pairs"), r.debug("pair_g")
    assert len(gk) == len(ok), f"pair counts differ ({len(gk)} vs {len(ok)})"
    assert np.array_equal(gk, ok), "sorted (tile, depth) keys differ"
    assert np.array_equal(gg, og), "sorted pair payloads (g) differ"


def compare_images(gl, gr, ol, orr):
    for g, o in ((gl, ol), (gr, orr)):
        d = np.abs(g - o)
        assert d.max() <= PIX_TOL, f"max pixel diff {d.max()}"
        assert psnr(g, o) >= PSNR_MIN
    return max(float(np.abs(gl - ol).max()), float(np.abs(gr - orr).max()))
