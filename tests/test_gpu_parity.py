"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs (BASELINE.json configs)."""
import numpy as np
import pytest

import scenegen as sg
from parity import (BLEND_FAST_TOL, compare_images, compare_pool, compare_sets, compare_splats_pairs, oracle_config,
                    renderer)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _frame_parity(orc, o, r, rig, full=True, images=True):
    res = o.frame(rig, raster=full, images=images and full)
    gl, gr, st = r.render(rig)
    vis, mis = compare_sets(o, r, st)
    assert st["depth_used"] == res.stats.depth_used and st["depth_next"] == res.stats.depth_next
    if not full:
        return st, None
    compare_pool(o, r, vis)
    compare_splats_pairs(o, r)
    d = None
    if images:
        d = compare_images(gl.cpu().numpy(), gr.cpu().numpy(), res.img_l, res.img_r)
    return st, d


def test_c1_all_poses(orc, c1):
    """configs[0]: 1k anchors x K=10, 64x64, 4 poses; every intermediate bit-exact."""
    cfg, sc = c1
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    r = renderer(cfg).load(sc)
    for rig in sg.trajectory(cfg):
        st, d = _frame_parity(orc, o, r, rig)
        assert d <= BLEND_FAST_TOL


@pytest.mark.parametrize("wh", [(100, 70), (33, 17), (17, 129), (1, 1), (250, 4)])
def test_c1_ragged_image_sizes(orc, c1, wh):
    """Image sizes that are not multiples of the 16x16 tile nor of the 8x4 blend block (partial tiles and
    blocks on the right and bottom edges, the row test's last-column special case, a 1x1 image, a 4-row
    strip): every intermediate bit-exact, pixels within the blend tolerance, edge pixels included."""
    import dataclasses
    cfg, sc = c1
    cfg = dataclasses.replace(cfg, width=wh[0], height=wh[1])
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    r = renderer(cfg).load(sc)
    for rig in sg.trajectory(cfg):
        st, d = _frame_parity(orc, o, r, rig)
        assert d <= BLEND_FAST_TOL


def test_c1_derive_on_cuda_cores(orc, c1):
    """The dp4a (CUDA-core) derivation path gives the same bits as the tcgen05 default."""
    from paper_2502_14938_b200 import _abi
    cfg, sc = c1
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    r = renderer(cfg, flags=_abi.GSC_F_DERIVE_CUDA_CORES).load(sc)
    for rig in sg.trajectory(cfg):
        st, d = _frame_parity(orc, o, r, rig)
        assert d <= BLEND_FAST_TOL


def test_c1_brute_force_pixels(orc, c1):
    """GPU pixels equal the oracle's per-pixel brute-force (O1) renderer."""
    cfg, sc = c1
    for rig in sg.trajectory(cfg):
        o = orc.Oracle(sc, oracle_config(orc, cfg))
        res = o.frame(rig, brute=True)
        r = renderer(cfg).load(sc)
        gl, gr, _ = r.render(rig)
        compare_images(gl.cpu().numpy(), gr.cpu().numpy(), res.img_l, res.img_r)


def test_c1_moving_trajectory_cache(orc, c1):
    """Cache state machine over a moving trajectory with D_max = 4: hit/miss sets,
    depths and images match every frame."""
    cfg, sc = c1
    o = orc.Oracle(sc, oracle_config(orc, cfg, d_max=4))
    r = renderer(cfg, d_max=4).load(sc)
    c = cfg.center
    for f in range(24):
        eye = c + np.array([25 * np.cos(0.12 * f), 25 * np.sin(0.12 * f), 2.0 + 0.5 * f])
        rig = sg.look_at_rig(eye, c + np.array([0, 0, 3.0]), 0.064)
        _frame_parity(orc, o, r, rig)


@pytest.mark.parametrize("d_max", [4, 10])
def test_c1_staggered_expiry(orc, c1, d_max):
    """GSC_F_STAGGER (F3, R26): static frames (one D-th of the anchors re-derived per frame, no
    flush frame), then a moving stretch: hit/miss sets and depths every frame, births of the
    visible anchors, full parity on some frames."""
    import paper_2502_14938_b200 as gp
    cfg, sc = c1
    o = orc.Oracle(sc, oracle_config(orc, cfg, d_max=d_max, stagger=True))
    r = renderer(cfg, d_max=d_max, flags=gp.GSC_F_STAGGER).load(sc)
    c = cfg.center
    rig0 = sg.trajectory(cfg)[0]
    for f in range(28):
        if f < 2 * d_max:
            rig = rig0
        else:
            eye = c + np.array([25 * np.cos(0.12 * f), 25 * np.sin(0.12 * f), 2.0 + 0.5 * f])
            rig = sg.look_at_rig(eye, c + np.array([0, 0, 3.0]), 0.064)
        st, _ = _frame_parity(orc, o, r, rig, full=(f % 5 == 0))
        if 0 < f < 2 * d_max:
            assert 0 < st["n_misses"] < st["n_visible"] // 2
        vis = r.debug("visible")
        birth = r.debug("birth")
        for i in vis[::29]:
            assert birth[i] == o.birth(int(i))


@pytest.mark.parametrize("guide", [1, 2])
def test_c1_guide_variants(orc, c1, guide):
    """Exponential / staged guiding functions (GSC_F_GUIDE_EXP / _STAGED, R23) over a moving
    trajectory: depths, hit/miss sets every frame and full parity on some frames."""
    import paper_2502_14938_b200 as gp
    cfg, sc = c1
    flag = gp.GSC_F_GUIDE_EXP if guide == 1 else gp.GSC_F_GUIDE_STAGED
    o = orc.Oracle(sc, oracle_config(orc, cfg, guide=guide))
    r = renderer(cfg, flags=flag).load(sc)
    c = cfg.center
    depths = set()
    for f in range(20):
        # inside the block at eye height, the view direction jumping by 2.5 rad (x0.3 every other
        # pair of frames): novelty 7-46%, so both guides leave D_max
        eye = c + np.array([2.0 * np.cos(0.1 * f), 2.0 * np.sin(0.1 * f), 1.7])
        a = 2.5 * f * (1.0 if f % 4 < 2 else 0.3)
        rig = sg.look_at_rig(eye, eye + np.array([np.cos(a), np.sin(a), -0.1]), 0.064)
        st, _ = _frame_parity(orc, o, r, rig, full=(f % 7 == 0))
        depths.add(st["depth_next"])
    assert len(depths) > 1


@pytest.mark.parametrize("ablate", [1, 2, 3])
def test_c1_ablations(orc, c1, ablate):
    """F1 ablations (GSC_F_ABL_FIXED_EXTENT = 1, GSC_F_ABL_AABB_TILES = 2, both = 3) against the
    oracle with the same ablation: every intermediate bit-exact on the four C1 poses."""
    import paper_2502_14938_b200 as gp
    cfg, sc = c1
    flags = (gp.GSC_F_ABL_FIXED_EXTENT if ablate & 1 else 0) | (gp.GSC_F_ABL_AABB_TILES if ablate & 2 else 0)
    o = orc.Oracle(sc, oracle_config(orc, cfg, ablate=ablate))
    r = renderer(cfg, flags=flags).load(sc)
    for rig in sg.trajectory(cfg):
        st, d = _frame_parity(orc, o, r, rig)
        assert d <= BLEND_FAST_TOL


def test_c1_spec_literal_depth(orc, c1):
    import paper_2502_14938_b200 as gp
    cfg, sc = c1
    o = orc.Oracle(sc, oracle_config(orc, cfg, literal=True))
    r = renderer(cfg, flags=gp.GSC_F_DEPTH_LITERAL).load(sc)
    rig = sg.trajectory(cfg)[0]
    for f in range(13):
        _frame_parity(orc, o, r, rig, full=(f % 5 == 0))


def test_reset_and_empty_frames(orc, c1):
    """Edge cases: a pose seeing nothing (V = 0, no splats, no pairs -> background),
    then reset_cache restarts at frame 0."""
    cfg, sc = c1
    r = renderer(cfg).load(sc)
    eye = cfg.center + np.array([0.0, -200.0, 3.0])
    away = sg.look_at_rig(eye, eye + np.array([0.0, -1.0, 0.0]), 0.0)
    gl, gr, st = r.render(away)
    assert st["n_visible"] == 0 and st["n_splats"] == 0 and st["n_pairs"] == 0
    assert float(gl.abs().max()) == 0.0
    r.reset_cache()
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    _frame_parity(orc, o, r, sg.trajectory(cfg)[0])


@pytest.mark.parametrize("fn,lo,hi,step", [("exp", -90.0, 90.0, 1), ("log", 1e-30, 1e30, 3),
                                           ("tanh", -20.0, 20.0, 3), ("sigmoid", -90.0, 90.0, 3),
                                           ("exp_blend", -87.0, -0.0, 1)])
def test_elementary_functions_bitwise(orc, fn, lo, hi, step):
    """Device exp_s/log_s/tanh_s/sigmoid_s equal the oracle's on every float of
    the range (every `step`-th bit pattern); the blend's exp_blend equals the
    oracle's exp_s on every float of [-87, 0] (N1)."""
    import torch
    import paper_2502_14938_b200 as gp
    r = gp.Renderer(0, 64, 64)
    nbad = 0
    for sign_lo, sign_hi in ((lo, min(hi, -0.0)), (max(lo, 0.0), hi)):
        if sign_lo > sign_hi or (sign_lo == sign_hi == 0):
            continue
        a = np.float32(sign_lo).view(np.uint32).astype(np.int64)
        b = np.float32(sign_hi).view(np.uint32).astype(np.int64)
        a, b = min(a, b), max(a, b)
        for s0 in range(a, b + 1, 1 << 26):
            bits = np.arange(s0, min(b + 1, s0 + (1 << 26)), step, dtype=np.int64).astype(np.uint32)
            x = bits.view(np.float32)
            ref = orc.elem("exp" if fn == "exp_blend" else fn, x)
            got = r.elementary(fn, torch.from_numpy(x).cuda()).cpu().numpy()
            same = (got.view(np.uint32) == ref.view(np.uint32)) | (np.isnan(got) & np.isnan(ref))
            nbad += int((~same).sum())
    assert nbad == 0


def test_fast_exp_error_bound(orc):
    """The blend's SFU exponential (R5) on every float of [-5.56, 0] (the power range where the blend
    can accept a splat: power >= skip bound = -ln(255 alpha) - 2^-7 >= -5.55) against the oracle's
    exp_s: relative error < 8e-7, so alpha' = min(0.99, alpha e) differs from the oracle's by < 2^-20
    relative after the product roundings (+1.2e-7) -- half the guard band kAlphaGuard (2^-19) the blend
    uses to hand skip decisions near 1/255 to the exact replay (blend.cu)."""
    import torch
    import paper_2502_14938_b200 as gp
    r = gp.Renderer(0, 64, 64)
    a = np.float32(-0.0).view(np.uint32).astype(np.int64)
    b = np.float32(-5.56).view(np.uint32).astype(np.int64)
    worst = 0.0
    for s0 in range(a, b + 1, 1 << 25):
        bits = np.arange(s0, min(b + 1, s0 + (1 << 25)), dtype=np.int64).astype(np.uint32)
        x = bits.view(np.float32)
        ref = orc.elem("exp", x).astype(np.float64)
        got = r.elementary("exp_fast", torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
        worst = max(worst, float(np.max(np.abs(got / ref - 1.0))))
    assert worst < 8e-7, worst


def test_rgba8_output_matches_f32(orc, c1):
    """The display format bench.py times (RGBA8) is the f32 result quantised:
    round(255 clamp(x)) per channel, alpha = round(255 (1 - T))."""
    import torch
    import paper_2502_14938_b200 as gp
    cfg, sc = c1
    rig = sg.trajectory(cfg)[1]
    r1 = renderer(cfg).load(sc)
    fl, fr, _ = r1.render(rig)
    r2 = renderer(cfg).load(sc)
    ql, qr, _ = r2.render(rig, fmt=gp.GSC_FMT_RGBA8)
    for f, q in ((fl, ql), (fr, qr)):
        want = torch.clamp(torch.round(f.permute(1, 2, 0) * 255.0), 0, 255).to(torch.uint8)
        assert torch.equal(q[..., :3], want)


# ---------------------------------------------------------------- configs[1..2] (100k, 2K binocular)
@pytest.fixture(scope="module")
def c100k():
    cfg = sg.config("C3")
    return cfg, cfg.scene()


def test_c2_static_no_reuse(orc, c100k):
    """configs[1]: 100k anchors, 1920x1080 binocular, static poses, D_max = 1:
    full parity on the first frame of each static pose, sets on the others."""
    cfg3, sc = c100k
    cfg = sg.config("C2")
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    r = renderer(cfg).load(sc)
    traj = sg.trajectory(cfg, n_frames=8)
    for f, rig in enumerate(traj):
        st, d = _frame_parity(orc, o, r, rig, full=(f in (0, 4)))
        assert st["n_misses"] == st["n_visible"]   # D_max = 1: no reuse


def test_c3_trajectory_reuse(orc, c100k):
    """configs[2]: 300-frame orbit with reuse (D_max = 10): hit/miss sets and
    depths bit-exact on every frame; full parity (pool, splats, sorted keys,
    pixels) on frames 0, 1, 150 and 299."""
    cfg, sc = c100k
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    r = renderer(cfg).load(sc)
    hits = 0
    for f, rig in enumerate(sg.trajectory(cfg)):
        st, d = _frame_parity(orc, o, r, rig, full=f in (0, 1, 150, 299))
        hits += st["n_hits"]
    assert hits > 0


def test_eval_counts_match_oracle(orc, c1, c100k):
    """The blend's evaluation count for the roofline (gsc_frame_stats.n_evals_list, GSC_F_COUNT_EVALS): per
    pixel, the tile-list entries up to and including the splat it stops before -- the oracle's own
    orc_blend_pixel count (SURVEY d-3).  The exact-exponential kernel reproduces it exactly; the default
    kernel within 1e-3 (a pixel the fast path flags for the exact replay may stop one splat apart).  The
    executed count (after the 8x4-block skip) never exceeds it."""
    import paper_2502_14938_b200 as gp
    for cfg, sc, frames in ((c1[0], c1[1], range(4)), (c100k[0], c100k[1], (0, 1, 150))):
        traj = sg.trajectory(cfg)
        for flags, tol in ((gp.GSC_F_COUNT_EVALS | gp.GSC_F_BLEND_EXACT, 0.0), (gp.GSC_F_COUNT_EVALS, 1e-3)):
            o = orc.Oracle(sc, oracle_config(orc, cfg))
            r = renderer(cfg, flags=flags).load(sc)
            for f in range(max(frames) + 1):
                res = o.frame(traj[f], raster=f in frames, images=f in frames)
                _, _, st = r.render(traj[f])
                if f not in frames:
                    continue
                ref = res.stats.n_evals
                assert ref > 0
                assert abs(int(st["n_evals_list"]) - ref) <= tol * ref, (cfg.name, f, flags, st["n_evals_list"], ref)
                assert 0 < st["n_evals"] <= st["n_evals_list"]


# ---------------------------------------------------------------- configs[3] at full size (bench launch config)
@pytest.fixture(scope="module")
def c4():
    cfg = sg.config("C4")
    return cfg, cfg.scene()


def test_c4_full_size_bench_config(orc, c4):
    """configs[3] (1M anchors, 2K binocular) in the launch configuration
    bench.py times (stage timing on, default capacities): frame 0 (cold cache,
    633k misses) and frame 30 (after 29 cached frames) fully bit-exact -- sets,
    pool, splat records, 30M+ sorted keys, pixels -- and the hit/miss sets of
    every frame in between."""
    import paper_2502_14938_b200 as gp
    cfg, sc = c4
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    r = renderer(cfg, flags=gp.GSC_F_STAGE_TIMING).load(sc)
    traj = sg.trajectory(cfg)
    for f in range(31):
        st, d = _frame_parity(orc, o, r, traj[f], full=f in (0, 30))
        assert not st["overflow"]
        if f in (0, 30):
            assert d <= BLEND_FAST_TOL


def test_c5_full_size_frames(orc):
    """configs[4] (5M anchors, 2K binocular, the scaling workload) at full size: frame 0 (cold cache,
    every visible anchor derived) and frame 10 (after 9 cached frames) fully bit-exact -- sets, pool,
    splat records, sorted keys, pixels -- with the hit/miss sets of the frames between."""
    cfg = sg.config("C5")
    sc = cfg.scene()
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    r = renderer(cfg).load(sc)
    traj = sg.trajectory(cfg)
    for f in range(11):
        st, d = _frame_parity(orc, o, r, traj[f], full=f in (0, 10))
        assert not st["overflow"]
        if f in (0, 10):
            assert d <= BLEND_FAST_TOL


def test_host_async_matches_device_render(orc, c1):
    """The asynchronous end-to-end API (host pose in, images into pinned host memory, frame f's copy
    overlapping frame f+1) returns the same images as device rendering, frame by frame, through a
    moving trajectory (exercises the double-buffered frame sets and staging images)."""
    import torch
    import paper_2502_14938_b200 as gp
    cfg, sc = c1
    c = cfg.center
    rigs = [sg.look_at_rig(c + np.array([25 * np.cos(0.3 * f), 25 * np.sin(0.3 * f), 3.0]),
                           c + np.array([0, 0, 3.0]), 0.064) for f in range(9)]
    r1 = renderer(cfg).load(sc)
    want = []
    for rig in rigs:
        gl, gr, _ = r1.render(rig, fmt=gp.GSC_FMT_RGBA8)
        want.append((gl.cpu().clone(), gr.cpu().clone()))
    r2 = renderer(cfg).load(sc)
    bufs = [(torch.empty((cfg.height, cfg.width, 4), dtype=torch.uint8).pin_memory(),
             torch.empty((cfg.height, cfg.width, 4), dtype=torch.uint8).pin_memory()) for _ in rigs]
    seqs = [r2.render_host_async(rig, *bufs[i], gp.GSC_FMT_RGBA8) for i, rig in enumerate(rigs)]
    for q in seqs:
        r2.wait_frame(q)
    for (hl, hr), (wl, wr) in zip(bufs, want):
        assert torch.equal(hl, wl) and torch.equal(hr, wr)


def test_elastic_session_real_time(orc, c1):
    """F2 in real time on the GPU: two workers with private pipelines (C1 scene) fed by the shared
    queue at 200 Hz for 2 s; frames render end to end, displayed timestamps are monotone, no stale
    pose is rendered."""
    import torch
    import paper_2502_14938_b200 as gp
    from paper_2502_14938_b200 import elastic as el
    cfg, sc = c1
    c = cfg.center

    def make_worker(w):
        r = renderer(cfg).load(sc)
        hl = torch.empty((cfg.height, cfg.width, 4), dtype=torch.uint8).pin_memory()
        hr = torch.empty((cfg.height, cfg.width, 4), dtype=torch.uint8).pin_memory()

        def render(rig):
            r.render_host(rig, hl, hr, gp.GSC_FMT_RGBA8)
            return {}
        return render

    poses = [sg.look_at_rig(c + np.array([25 * np.cos(0.01 * k), 25 * np.sin(0.01 * k), 3.0]), c, 0.064)
             for k in range(400)]
    scfg = el.SessionConfig(w_init=2, w_max=2, control=False, sample_interval=1 / 200.0, timeout=0.1)
    rep = el.run_session(poses, scfg, clock="real", make_worker=make_worker, duration=2.0)
    ts = rep.displayed_ts
    assert rep.n_displayed > 50
    assert all(a <= b for a, b in zip(ts, ts[1:]))
    assert all(r.t_start - r.timestamp <= scfg.timeout + 0.01 for r in rep.records)
    assert {r.worker for r in rep.records} == {0, 1}


def test_c1_no_dered_per_eye_pipelines(orc, c1):
    """No-de-redundancy ablation (F1): one monocular pipeline per eye (PerEyeRenderer, GSC_F_MONO)
    equals, eye by eye, an oracle state machine driven by that eye alone (a rig whose eyes coincide):
    visible / hit / miss sets every frame and the eye's image bit for bit, over a moving trajectory."""
    import paper_2502_14938_b200 as gp
    cfg, sc = c1
    per = gp.PerEyeRenderer(0, cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far, 4).load(sc)
    oracles = [orc.Oracle(sc, oracle_config(orc, cfg, d_max=4)) for _ in range(2)]
    c = cfg.center
    for f in range(12):
        eye = c + np.array([25 * np.cos(0.12 * f), 25 * np.sin(0.12 * f), 2.0 + 0.5 * f])
        rig = sg.look_at_rig(eye, c + np.array([0, 0, 3.0]), 0.064)
        il, ir, stats = per.render(rig)
        for e, img in enumerate((il, ir)):
            res = oracles[e].frame(gp.PerEyeRenderer._mono(rig, e))
            compare_sets(oracles[e], per.eyes[e], stats[e])
            d = float(np.abs(img.cpu().numpy() - res.img_l).max())
            assert d <= BLEND_FAST_TOL


@pytest.mark.parametrize("start,stop,full", [(290, 300, (290, 300)), (440, 450, (450,)), (540, 599, (540, 599))])
def test_c4_cold_blocks_aerial(orc, c4, start, stop, full):
    """SURVEY §8(e) per-rank oracle replay: a weak-scaling rank starts its contiguous block of the
    C4 trajectory cold, mid-trajectory.  Blocks starting at frames 290 / 440 / 540 (the aerial half:
    the eye at ~150-300 m, where the paper's FPS drops) on a fresh context and a fresh oracle:
    hit/miss sets and depths every frame, full parity (pool, splats, sorted keys, pixels) at the
    listed frames -- including the block's cold first frame and the trajectory's last frame."""
    cfg, sc = c4
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    r = renderer(cfg).load(sc)
    traj = sg.trajectory(cfg)
    for f in range(start, stop + 1):
        st, d = _frame_parity(orc, o, r, traj[f], full=f in full)
        assert not st["overflow"]
        if f == start:
            assert st["n_misses"] == st["n_visible"]       # cold block start
        if f in full:
            assert d <= BLEND_FAST_TOL


def test_c5_cold_block(orc):
    """configs[4]: the block of a rank starting at frame 1800 of the 2400-frame C5 trajectory (cold
    cache, high altitude): sets every frame, full parity at 1800 and 1805."""
    cfg = sg.config("C5")
    sc = cfg.scene()
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    r = renderer(cfg).load(sc)
    traj = sg.trajectory(cfg)
    for f in range(1800, 1806):
        st, d = _frame_parity(orc, o, r, traj[f], full=f in (1800, 1805))
        assert not st["overflow"]
        if f in (1800, 1805):
            assert d <= BLEND_FAST_TOL


def test_blend_exact_mode_bit_identical(orc, c1):
    """GSC_F_BLEND_EXACT: the exact-exponential blend -- pixels bit-identical to the oracle's on every
    C1 pose and on a full-size C4 frame (the default fast blend: within BLEND_FAST_TOL, decisions equal)."""
    import paper_2502_14938_b200 as gp
    cfg, sc = c1
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    r = renderer(cfg, flags=gp.GSC_F_BLEND_EXACT).load(sc)
    for rig in sg.trajectory(cfg):
        st, d = _frame_parity(orc, o, r, rig)
        assert d == 0.0


def test_c4_full_size_blend_exact(orc, c4):
    """GSC_F_BLEND_EXACT at configs[3] full size: frames 0 (cold) and 30 with pixels bit-identical to the
    oracle (the default fast blend is checked against BLEND_FAST_TOL in test_c4_full_size_bench_config)."""
    import paper_2502_14938_b200 as gp
    cfg, sc = c4
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    r = renderer(cfg, flags=gp.GSC_F_BLEND_EXACT).load(sc)
    traj = sg.trajectory(cfg)
    for f in range(31):
        st, d = _frame_parity(orc, o, r, traj[f], full=f in (0, 30))
        if f in (0, 30):
            assert d == 0.0


def test_c5_high_altitude_block(orc):
    """configs[4] near the end of its 2400-frame trajectory (~280 m, the widest views): a cold block from
    frame 2300, full parity at 2300 and 2305, sets between."""
    cfg = sg.config("C5")
    sc = cfg.scene()
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    r = renderer(cfg).load(sc)
    traj = sg.trajectory(cfg)
    for f in range(2300, 2306):
        st, d = _frame_parity(orc, o, r, traj[f], full=f in (2300, 2305))
        assert not st["overflow"]
        if f in (2300, 2305):
            assert d <= BLEND_FAST_TOL
