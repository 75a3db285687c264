"""GPU parity of the real-weights path: fp32 non-grid features and decoder
weights, the continuous view direction, the fixed-order fp32 MLP (derive_f32_kernel) against the
oracle's orc_mlp_f32 -- derived pool bit-exact, visible / hit / miss sets, splat records and sorted
keys bit-exact, pixels within the blend tolerance -- on the C1 / C3 scenes with real weights and on a
Scaffold-GS-style scene without LoD (L = 1)."""
import numpy as np
import pytest

import scenegen as sg
from parity import (BLEND_FAST_TOL, compare_images, compare_pool, compare_sets, compare_splats_pairs,
                    oracle_config, renderer)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _frame(o, r, rig, full):
    res = o.frame(rig, raster=full)
    gl, gr, st = r.render(rig)
    vis, _ = compare_sets(o, r, st)
    assert st["depth_used"] == res.stats.depth_used and st["depth_next"] == res.stats.depth_next
    if not full:
        return st, None
    compare_pool(o, r, vis)
    compare_splats_pairs(o, r)
    d = compare_images(gl.cpu().numpy(), gr.cpu().numpy(), res.img_l, res.img_r)
    assert d <= BLEND_FAST_TOL
    return st, d


def test_c1r_all_poses(orc):
    cfg = sg.config("C1R")
    sc = cfg.scene()
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    r = renderer(cfg).load(sc)
    for rig in sg.trajectory(cfg):
        _frame(o, r, rig, True)


def test_c1r_moving_cache(orc):
    """Cache state machine with real weights over a moving trajectory (D_max = 4)."""
    cfg = sg.config("C1R")
    sc = cfg.scene()
    o = orc.Oracle(sc, oracle_config(orc, cfg, d_max=4))
    r = renderer(cfg, d_max=4).load(sc)
    c = cfg.center
    for f in range(16):
        eye = c + np.array([25 * np.cos(0.12 * f), 25 * np.sin(0.12 * f), 2.0 + 0.5 * f])
        _frame(o, r, sg.look_at_rig(eye, c + np.array([0, 0, 3.0]), 0.064), full=f % 4 == 0)


def test_c3r_trajectory(orc):
    """100k anchors, 1920x1080 binocular, real weights: the first 31 frames of the C3 orbit, sets every
    frame, full parity at frames 0 (cold: every visible anchor derived) and 30."""
    cfg = sg.config("C3R")
    sc = cfg.scene()
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    r = renderer(cfg).load(sc)
    traj = sg.trajectory(cfg)
    for f in range(31):
        st, _ = _frame(o, r, traj[f], full=f in (0, 30))
        assert not st["overflow"]


def test_c3s_scaffold_no_lod(orc):
    """Scaffold-GS-style scene (L = 1, every anchor at level 0: no LoD selection) with real weights:
    frames 0 and 150 of the C3 orbit (ground level and 30 m) fully bit-exact, the frames between
    hit/miss-exact; the visible set is the pure frustum set (L = 1)."""
    cfg = sg.config("C3S")
    sc = cfg.scene()
    assert sc.L == 1 and np.all(sc.level == 0)
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    r = renderer(cfg).load(sc)
    traj = sg.trajectory(cfg)
    for f in list(range(0, 6)) + [150]:
        if f == 150:
            o.reset()
            r.reset_cache()
        _frame(o, r, traj[f], full=f in (0, 150))


def test_gsc2_v3_file(orc, tmp_path):
    """GSC2 version 3 (fp32 features / weights) through gsc_load_scene equals the host-array load."""
    cfg = sg.config("C1R")
    sc = cfg.scene()
    path = str(tmp_path / "c1r.gsc2")
    sg.write_gsc2(sc, path)
    rf = renderer(cfg).load(path)
    rh = renderer(cfg).load(sc)
    for rig in sg.trajectory(cfg):
        fl, _, _ = rf.render(rig)
        hl, _, _ = rh.render(rig)
        assert np.array_equal(rf.debug("pool"), rh.debug("pool"))
        assert np.array_equal(fl.cpu().numpy(), hl.cpu().numpy())


def test_real_weights_load_errors(tmp_path):
    """gsc_load_scene_host_f32 / GSC2 v3: a non-finite feature or weight -> GSC_EFORMAT; a level >= L ->
    GSC_EFORMAT; a truncated v3 file -> GSC_EFORMAT with the offset of the array that does not fit."""
    import copy
    import re
    from paper_2502_14938_b200 import _abi
    cfg = sg.config("C1R")
    sc = cfg.scene()
    for name in ("feat", "W1", "b2s"):
        bad = copy.copy(sc)
        arr = getattr(sc, name).copy()
        arr.flat[3] = np.nan
        setattr(bad, name, arr)
        with pytest.raises(_abi.GscError) as ei:
            renderer(cfg).load(bad)
        assert _abi.STATUS_NAMES[ei.value.status] == "GSC_EFORMAT"
    path = str(tmp_path / "r.gsc2")
    sg.write_gsc2(sc, path)
    data = open(path, "rb").read()
    n = sc.n
    off_W1 = 56 + 12 * n + 128 * n + 120 * n + 12 * n + n      # pos, feat (f32), offs, scale, level
    cut = str(tmp_path / "cut.gsc2")
    with open(cut, "wb") as fh:
        fh.write(data[:off_W1 + 100])
    with pytest.raises(_abi.GscError) as ei:
        renderer(cfg).load(cut)
    assert _abi.STATUS_NAMES[ei.value.status] == "GSC_EFORMAT"
    assert int(re.search(r"offset (\d+)", str(ei.value)).group(1)) == off_W1


def test_c4r_real_weights_full_size(orc):
    """The real-weights path at configs[3] size (1M anchors, 2K binocular): frame 0 (every visible anchor
    derived by the fixed-order fp32 MLP: ~630k anchors) and frame 5 fully bit-exact up to the pixels.
    (These weights give larger Gaussians than the grid scene's: frame 0 needs 40.2M pairs, above the
    default capacity of 4 N K = 40M, so the context is created with a larger pair_capacity.)"""
    cfg = sg.config("C4R")
    sc = cfg.scene()
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    r = renderer(cfg, pair_capacity=64 << 20).load(sc)
    traj = sg.trajectory(cfg)
    for f in range(6):
        st, _ = _frame(o, r, traj[f], full=f in (0, 5))
        assert not st["overflow"]


# ---- R32 combine inputs (SURVEY §8(f) F4 "optional distance input / feature bank")
@pytest.mark.parametrize("dist,bank", [(True, False), (False, True), (True, True)])
def test_c1_combine_inputs_all_poses(orc, dist, bank):
    """Distance input and / or feature bank on the C1 scene: derived pool, splats, sorted keys bit-exact
    against the oracle's orc_bank_weights / orc_bank_blend / orc_mlp_f32 chain, pixels within tolerance."""
    cfg = sg.config("C1R")
    sc = sg.with_real_weights(sg.config("C1").scene(), dist=dist, bank=bank)
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    r = renderer(cfg).load(sc)
    for rig in sg.trajectory(cfg):
        _frame(o, r, rig, True)


def test_c1b_moving_cache(orc):
    cfg = sg.config("C1B")
    sc = cfg.scene()
    o = orc.Oracle(sc, oracle_config(orc, cfg, d_max=4))
    r = renderer(cfg, d_max=4).load(sc)
    c = cfg.center
    for f in range(16):
        eye = c + np.array([25 * np.cos(0.12 * f), 25 * np.sin(0.12 * f), 2.0 + 0.5 * f])
        _frame(o, r, sg.look_at_rig(eye, c + np.array([0, 0, 3.0]), 0.064), full=f % 4 == 0)


def test_c3b_trajectory(orc):
    """100k anchors, 2K binocular, distance input + feature bank: the first 11 frames of the C3 orbit,
    full parity at frames 0 (cold) and 10 (the flush)."""
    cfg = sg.config("C3B")
    sc = cfg.scene()
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    r = renderer(cfg).load(sc)
    traj = sg.trajectory(cfg)
    for f in range(11):
        st, _ = _frame(o, r, traj[f], full=f in (0, 10))
        assert not st["overflow"]


def test_c3sb_scaffold_no_lod(orc):
    """The Scaffold-GS configuration the combine inputs come from: L = 1 (no LoD), distance input and
    feature bank; frames 0 and 150 of the C3 orbit fully bit-exact."""
    cfg = sg.config("C3SB")
    sc = cfg.scene()
    assert sc.L == 1 and sc.dist_input and sc.bank
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    r = renderer(cfg).load(sc)
    traj = sg.trajectory(cfg)
    _frame(o, r, traj[0], True)
    o.reset()
    r.reset_cache()
    _frame(o, r, traj[150], True)


def test_gsc2_v4_file(orc, tmp_path):
    """GSC2 version 4 (combine-input flags + feature-bank weights) through gsc_load_scene equals the
    host-array load, for each combination of the two inputs."""
    cfg = sg.config("C1R")
    for dist, bank in ((True, False), (False, True), (True, True)):
        sc = sg.with_real_weights(sg.config("C1").scene(), dist=dist, bank=bank)
        path = str(tmp_path / f"c1_{int(dist)}{int(bank)}.gsc2")
        sg.write_gsc2(sc, path)
        rf = renderer(cfg).load(path)
        rh = renderer(cfg).load(sc)
        for rig in sg.trajectory(cfg):
            fl, _, _ = rf.render(rig)
            hl, _, _ = rh.render(rig)
            assert np.array_equal(rf.debug("pool"), rh.debug("pool"))
            assert np.array_equal(fl.cpu().numpy(), hl.cpu().numpy())


def test_combine_input_errors(tmp_path):
    """Feature bank without its weights -> GSC_EINVAL; a non-finite bank weight -> GSC_EFORMAT; a v4 file
    cut inside the bank weights -> GSC_EFORMAT naming the offset; unknown flag bits -> GSC_EFORMAT."""
    import copy
    import re
    import struct
    from paper_2502_14938_b200 import _abi
    cfg = sg.config("C1R")
    sc = sg.with_real_weights(sg.config("C1").scene(), dist=True, bank=True)
    bad = copy.copy(sc)
    bad.Wb2 = None
    with pytest.raises(_abi.GscError) as ei:
        renderer(cfg).load(bad)
    assert _abi.STATUS_NAMES[ei.value.status] == "GSC_EINVAL"
    bad = copy.copy(sc)
    bad.bb1 = sc.bb1.copy()
    bad.bb1[5] = np.inf
    with pytest.raises(_abi.GscError) as ei:
        renderer(cfg).load(bad)
    assert _abi.STATUS_NAMES[ei.value.status] == "GSC_EFORMAT"
    path = str(tmp_path / "b.gsc2")
    sg.write_gsc2(sc, path)
    data = open(path, "rb").read()
    cut = str(tmp_path / "cut.gsc2")
    bank_bytes = (4 * 32 + 32 + 32 * 3 + 3) * 4
    with open(cut, "wb") as fh:
        fh.write(data[:len(data) - bank_bytes + 100])
    with pytest.raises(_abi.GscError) as ei:
        renderer(cfg).load(cut)
    assert _abi.STATUS_NAMES[ei.value.status] == "GSC_EFORMAT"
    assert int(re.search(r"offset (\d+)", str(ei.value)).group(1)) == len(data) - bank_bytes
    flags = str(tmp_path / "flags.gsc2")
    with open(flags, "wb") as fh:
        fh.write(data[:56] + struct.pack("<I", 4) + data[60:])
    with pytest.raises(_abi.GscError) as ei:
        renderer(cfg).load(flags)
    assert _abi.STATUS_NAMES[ei.value.status] == "GSC_EFORMAT"
