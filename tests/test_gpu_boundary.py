"""The C-ABI boundary's file loader and error paths (include/gscache.h):
GSC2 files written by scenegen.write_gsc2 load to the same frames as host arrays; every
error class of the header is exercised (EFORMAT with the byte offset, EDEGENERATE,
ESTATE, EINVAL, ECAPACITY on every reporting path); non-finite splats are skipped and
counted like the oracle counts them."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import scenegen as sg
from parity import compare_images, compare_sets, compare_splats_pairs, oracle_config, renderer

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _status(exc):
    from paper_2502_14938_b200 import _abi
    return _abi.STATUS_NAMES[exc.status]


# ---------------------------------------------------------------- GSC2 file loader
def test_gsc2_file_loads_like_host_arrays(orc, c1, tmp_path):
    """gsc_load_scene on the file scenegen.write_gsc2 wrote renders bit-identically to
    gsc_load_scene_host on the same arrays, and matches the oracle (the C++ parser and the
    Python writer agree field by field)."""
    cfg, sc = c1
    path = str(tmp_path / "c1.gsc2")
    sg.write_gsc2(sc, path)
    assert np.array_equal(sg.read_gsc2(path).W2s, sc.W2s)
    rf = renderer(cfg).load(path)
    rh = renderer(cfg).load(sc)
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    for rig in sg.trajectory(cfg):
        fl, fr, sf = rf.render(rig)
        hl, hr, sh = rh.render(rig)
        res = o.frame(rig)
        assert np.array_equal(rf.debug("pairs"), rh.debug("pairs"))
        assert np.array_equal(rf.debug("pool"), rh.debug("pool"))
        assert np.array_equal(fl.cpu().numpy(), hl.cpu().numpy()) and np.array_equal(fr.cpu().numpy(), hr.cpu().numpy())
        compare_sets(o, rf, sf)
        compare_splats_pairs(o, rf)
        compare_images(fl.cpu().numpy(), fr.cpu().numpy(), res.img_l, res.img_r)


def test_gsc2_file_100k(orc, tmp_path):
    """The 100k-anchor scene through the file loader: first C3 frame fully bit-exact."""
    cfg = sg.config("C3")
    sc = cfg.scene()
    path = str(tmp_path / "c3.gsc2")
    sg.write_gsc2(sc, path)
    r = renderer(cfg).load(path)
    o = orc.Oracle(sc, oracle_config(orc, cfg))
    rig = sg.trajectory(cfg)[0]
    res = o.frame(rig)
    gl, gr, st = r.render(rig)
    compare_sets(o, r, st)
    compare_splats_pairs(o, r)
    compare_images(gl.cpu().numpy(), gr.cpu().numpy(), res.img_l, res.img_r)


def _load_err(cfg, path):
    from paper_2502_14938_b200 import _abi
    with pytest.raises(_abi.GscError) as ei:
        renderer(cfg).load(path)
    return _status(ei.value), str(ei.value)


def test_gsc2_format_errors(c1, tmp_path):
    """malformed files -> GSC_EFORMAT with the byte offset in gsc_last_error; a missing
    file -> GSC_EINVAL.  Truncation points: inside the header, inside every array."""
    cfg, sc = c1
    path = str(tmp_path / "ok.gsc2")
    sg.write_gsc2(sc, path)
    data = open(path, "rb").read()
    hdr = 56
    n = sc.n
    # array boundaries in file order (pos, feat, offs, scale, level, W1, b1, W2a, b2a, W2c, b2c, W2s, b2s)
    sizes = [12 * n, 32 * n, 120 * n, 12 * n, n, 35 * 96, 96, 320, 10, 960, 30, 2240, 70]
    starts = np.concatenate([[hdr], hdr + np.cumsum(sizes)])
    assert starts[-1] == len(data)

    def write(name, blob):
        p = str(tmp_path / name)
        with open(p, "wb") as fh:
            fh.write(blob)
        return p

    st, msg = _load_err(cfg, write("hdr.gsc2", data[:30]))
    assert st == "GSC_EFORMAT" and "offset 30" in msg
    for k in range(len(sizes)):
        cut = int(starts[k] + sizes[k] // 2)
        st, msg = _load_err(cfg, write(f"t{k}.gsc2", data[:cut]))
        assert st == "GSC_EFORMAT", (k, st, msg)
        off = int(re.search(r"offset (\d+)", msg).group(1))
        assert off == starts[k], (k, off, starts[k], msg)        # the array that does not fit starts there
    st, msg = _load_err(cfg, write("magic.gsc2", b"GSX2" + data[4:]))
    assert st == "GSC_EFORMAT" and "offset 0" in msg
    bad = bytearray(data)
    bad[4:8] = (7).to_bytes(4, "little")
    st, msg = _load_err(cfg, write("ver.gsc2", bytes(bad)))
    assert st == "GSC_EFORMAT" and "offset 4" in msg
    bad = bytearray(data)
    bad[12:16] = (16).to_bytes(4, "little")          # F = 16
    st, msg = _load_err(cfg, write("dims.gsc2", bytes(bad)))
    assert st == "GSC_EFORMAT" and "offset 12" in msg
    bad = bytearray(data)
    bad[int(starts[4])] = sc.L                         # anchor 0 at level L (>= L)
    st, msg = _load_err(cfg, write("level.gsc2", bytes(bad)))
    assert st == "GSC_EFORMAT" and "anchor 0" in msg
    st, msg = _load_err(cfg, str(tmp_path / "missing.gsc2"))
    assert st == "GSC_EINVAL"


# ---------------------------------------------------------------- state / rig errors
def test_state_and_rig_errors(c1):
    """Render before load / before pose -> GSC_ESTATE; antiparallel eyes -> GSC_EDEGENERATE
    (S:296-298); a non-unit quaternion -> GSC_EINVAL; the context stays usable."""
    from paper_2502_14938_b200 import _abi
    cfg, sc = c1
    rig = sg.trajectory(cfg)[0]
    r = renderer(cfg)
    ol, orr = r.alloc_outputs()
    with pytest.raises(_abi.GscError) as ei:
        r.render_into(None, ol, orr, sync_stats=True)
    assert _status(ei.value) == "GSC_ESTATE"
    with pytest.raises(_abi.GscError) as ei:
        r.debug("visible")
    assert _status(ei.value) == "GSC_ESTATE"
    r.load(sc)
    with pytest.raises(_abi.GscError) as ei:
        r.render_into(None, ol, orr, sync_stats=True)
    assert _status(ei.value) == "GSC_ESTATE"
    R = lambda q: np.array([[1 - 2 * (q[2] ** 2 + q[3] ** 2), 2 * (q[1] * q[2] - q[0] * q[3]), 2 * (q[1] * q[3] + q[0] * q[2])],
                            [2 * (q[1] * q[2] + q[0] * q[3]), 1 - 2 * (q[1] ** 2 + q[3] ** 2), 2 * (q[2] * q[3] - q[0] * q[1])],
                            [2 * (q[1] * q[3] - q[0] * q[2]), 2 * (q[2] * q[3] + q[0] * q[1]), 1 - 2 * (q[1] ** 2 + q[2] ** 2)]])
    # a rotation by pi about the camera's up axis reverses the forward direction exactly
    up = R(rig.lq)[:, 1]
    qf = np.array([0.0, *up])                          # pure quaternion: rotation by pi about up
    w1, v1 = qf[0], qf[1:]
    w2, v2 = rig.lq[0], np.asarray(rig.lq[1:])
    q = np.array([w1 * w2 - v1 @ v2, *(w1 * v2 + w2 * v1 + np.cross(v1, v2))])
    anti = sg.Rig(lp=rig.lp, lq=rig.lq, rp=rig.rp, rq=q / np.linalg.norm(q))
    assert np.allclose(R(anti.rq)[:, 2], -R(rig.lq)[:, 2])
    with pytest.raises(_abi.GscError) as ei:
        r.set_pose(anti)
    assert _status(ei.value) == "GSC_EDEGENERATE"
    bad = sg.Rig(lp=rig.lp, lq=np.asarray(rig.lq) * 1.01, rp=rig.rp, rq=rig.rq)
    with pytest.raises(_abi.GscError) as ei:
        r.set_pose(bad)
    assert _status(ei.value) == "GSC_EINVAL"
    gl, gr, st = r.render(rig)                         # still usable
    assert st["n_visible"] > 0


# ---------------------------------------------------------------- capacity
def _far_rig(cfg):
    eye = cfg.center + np.array([0.0, -200.0, 3.0])
    return sg.look_at_rig(eye, eye + np.array([0.0, -1.0, 0.0]), 0.0)


def test_capacity_list_overflow(orc, c1):
    """A tiny pair_capacity overflows project's kept-tile list: GSC_ECAPACITY, the frame's pairs
    are dropped (background image, nothing read out of bounds), and the context renders the next
    frames correctly."""
    from paper_2502_14938_b200 import _abi
    cfg, sc = c1
    rig = sg.trajectory(cfg)[0]
    r = renderer(cfg, pair_capacity=16).load(sc)
    ol, orr = r.alloc_outputs()
    with pytest.raises(_abi.GscError) as ei:
        r.render_into(rig, ol, orr, sync_stats=True)
    assert _status(ei.value) == "GSC_ECAPACITY"
    assert float(ol.abs().max()) == 0.0 and float(orr.abs().max()) == 0.0
    assert len(r.debug("pairs")) == 0
    gl, gr, st = r.render(_far_rig(cfg))              # a frame within capacity: OK again
    assert st["n_pairs"] == 0 and not st["overflow"]
    r.sync()                                          # the overflow was reported once, not sticky


def test_capacity_pair_overflow_all_paths(orc, c1):
    """Pairs beyond pair_capacity (the kept-tile list still fits): GSC_ECAPACITY on the stats path;
    without stats the overflow is reported by the next gsc_sync, by gsc_render_pair_host, and by
    gsc_wait_frame of the host-async path -- once per frame."""
    import torch
    import paper_2502_14938_b200 as gp
    from paper_2502_14938_b200 import _abi
    cfg, sc = c1
    rig = sg.trajectory(cfg)[0]
    _, _, st0 = renderer(cfg).load(sc).render(rig)
    need = int(st0["n_pairs"])
    cap = need - 5
    r = renderer(cfg, pair_capacity=cap).load(sc)
    ol, orr = r.alloc_outputs()
    with pytest.raises(_abi.GscError) as ei:
        r.render_into(rig, ol, orr, sync_stats=True)
    assert _status(ei.value) == "GSC_ECAPACITY" and str(need) in str(ei.value)
    assert len(r.debug("pairs")) == cap
    # no stats: gsc_sync reports it
    r.render_into(rig, ol, orr, sync_stats=False)
    with pytest.raises(_abi.GscError) as ei:
        r.sync()
    assert _status(ei.value) == "GSC_ECAPACITY"
    r.sync()                                           # once per frame
    # no stats, next render (non-blocking check of finished frames)
    r.render_into(rig, ol, orr, sync_stats=False)
    torch.cuda.synchronize()
    with pytest.raises(_abi.GscError) as ei:
        r.render_into(_far_rig(cfg), ol, orr, sync_stats=False)
    assert _status(ei.value) == "GSC_ECAPACITY"
    r.sync()
    # host paths
    hl = torch.empty((cfg.height, cfg.width, 4), dtype=torch.uint8).pin_memory()
    hr = torch.empty_like(hl).pin_memory()
    with pytest.raises(_abi.GscError) as ei:
        r.render_host(rig, hl, hr, gp.GSC_FMT_RGBA8)
    assert _status(ei.value) == "GSC_ECAPACITY"
    q = r.render_host_async(rig, hl, hr, gp.GSC_FMT_RGBA8)
    with pytest.raises(_abi.GscError) as ei:
        r.wait_frame(q)
    assert _status(ei.value) == "GSC_ECAPACITY"
    q = r.render_host_async(_far_rig(cfg), hl, hr, gp.GSC_FMT_RGBA8)
    r.wait_frame(q)


# ---------------------------------------------------------------- non-finite splats
def test_nonfinite_splats_skipped_and_counted(orc, c1):
    """non-finite splat parameters -> skip the splat and count it.  Anchors with a
    scale of 1e25 derive Gaussians whose covariance overflows to inf; both sides skip the same
    (Gaussian, eye) pairs, count them identically, and the rest of the frame stays bit-exact."""
    import copy
    cfg, sc = c1
    bad = copy.copy(sc)
    bad.scale = sc.scale.copy()
    lvl0 = np.nonzero(sc.level == 0)[0][:40]
    bad.scale[lvl0] = 1e25
    o = orc.Oracle(bad, oracle_config(orc, cfg))
    r = renderer(cfg).load(bad)
    seen = 0
    for rig in sg.trajectory(cfg)[:3]:
        res = o.frame(rig)
        gl, gr, st = r.render(rig)
        compare_sets(o, r, st)
        assert st["n_nonfinite_skipped"] == res.stats.n_nonfinite
        seen += st["n_nonfinite_skipped"]
        compare_splats_pairs(o, r)
        compare_images(gl.cpu().numpy(), gr.cpu().numpy(), res.img_l, res.img_r)
    assert seen > 0


def test_per_device_launch_config_multi_context(orc, c1):
    """Launch configuration is per device and thread-safe: two contexts rendering from two
    threads at once give the single-threaded result."""
    import threading
    cfg, sc = c1
    rigs = sg.trajectory(cfg)
    r0 = renderer(cfg).load(sc)
    want = [r0.render(rig)[0].cpu().numpy() for rig in rigs]
    out = {}

    def work(k):
        r = renderer(cfg).load(sc)
        out[k] = [r.render(rig)[0].cpu().numpy() for rig in rigs]

    ts = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for k in range(2):
        for a, b in zip(out[k], want):
            assert np.array_equal(a, b)
