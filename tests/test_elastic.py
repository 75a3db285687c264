"""the elastic scheduler's host logic (Alg. 2),
on CPU: every SPEC example and the scheduler invariants, in simulated time."""
import math
import random

import numpy as np
import pytest

import scenegen as sg
from paper_2502_14938_b200 import elastic as el


def _rig(x=0.0, yaw=0.0):
    eye = np.array([x, 0.0, 1.7])
    return sg.look_at_rig(eye, eye + np.array([math.cos(yaw), math.sin(yaw), 0.0]), 0.064)


def test_submit_pose_thresholds():
    q = el.CameraQueue(delta_p=0.01, delta_theta_deg=0.5)
    assert q.submit_pose(_rig(), 0.0)                     # first pose ever -> accepted
    assert not q.submit_pose(_rig(), 0.01)                # identical -> rejected
    assert q.submit_pose(_rig(0.1), 0.02)                 # moved 0.1 with delta_p 0.01 -> accepted
    assert not q.submit_pose(_rig(0.1, math.radians(0.3)), 0.03)   # 0.3 deg < 0.5 deg
    assert q.submit_pose(_rig(0.1, math.radians(1.0)), 0.04)       # 1 deg > 0.5 deg


def test_queue_capacity_drops_oldest():
    q = el.CameraQueue(capacity=3, delta_p=0.0)
    for k in range(5):
        assert q.submit_pose(_rig(0.1 * (k + 1)), 0.001 * k)
    assert len(q) == 3 and q.dropped_full == 2
    assert q.take_work(0.004).timestamp == pytest.approx(0.002)


def test_take_work_timeout():
    q = el.CameraQueue(timeout=0.1, delta_p=0.0)
    assert q.take_work(0.0) is None                       # empty -> none
    q.submit_pose(_rig(0.1), 0.0)
    q.submit_pose(_rig(0.2), 0.05)
    e = q.take_work(0.12)                                 # head stale (0.12 s), second fresh
    assert e is not None and e.timestamp == 0.05 and q.dropped_stale == 1
    q.submit_pose(_rig(0.3), 0.2)
    assert q.take_work(0.5) is None and len(q) == 0       # all stale -> none, emptied


def test_control_step_examples():
    c = el.FpsController(min_fps=60, max_fps=120, w_max=2)
    assert c.control_step(50.0) == el.START and c.n_workers == 2      # fps 50 < 60, n=1 -> start
    c = el.FpsController(min_fps=60, max_fps=120, w_max=2)
    assert c.control_step(250.0) is None                               # threshold 240 but n = 1
    c = el.FpsController(min_fps=60, max_fps=120, w_max=3)
    c.n_workers = 2
    assert c.control_step(100.0) is None                               # 60 <= 100 <= 180
    assert c.control_step(181.0) == el.STOP and c.n_workers == 1       # > (1 + 1/2) 120
    c = el.FpsController(min_fps=60, max_fps=120, w_max=2, period=0.5)
    assert c.control_step(10.0, now=1.0) == el.START
    assert c.control_step(10.0, now=1.2) is None                       # cooldown: one action / period


def test_try_display_examples():
    s = el.DisplaySync()
    assert s.try_display(7.0)
    assert not s.try_display(5.0)                         # ts 5 after 7 -> discard
    assert s.try_display(8.0) and s.last_written == 8.0
    assert s.try_display(8.0)                             # equal timestamps are written


def _traj(n):
    return [_rig(0.02 * k) for k in range(n)]


def test_session_single_worker_constant_cost():
    """single worker, 10 ms per frame, control off -> ~100 FPS (poses arrive at 200 Hz)."""
    cfg = el.SessionConfig(sample_interval=0.005, control=False, timeout=1.0)
    rep = el.run_session(_traj(2000), cfg, clock="sim", cost_fn=lambda w, f, t: 0.010)
    assert rep.avg_fps == pytest.approx(100.0, rel=0.05)


def test_session_cost_step_starts_worker():
    """cost 8 ms -> 25 ms at t = 5 s with min_fps 60, W_max 2: a second worker within one control
    period after the FPS estimate drops."""
    cfg = el.SessionConfig(min_fps=60, max_fps=120, w_max=2, sample_interval=1 / 90, timeout=0.2)
    rep = el.run_session(_traj(900), cfg, clock="sim",
                         cost_fn=lambda w, f, t: 0.008 if t < 5.0 else 0.025)
    starts = [t for t, n in rep.worker_timeline if n == 2]
    assert starts and 5.0 < starts[0] <= 5.0 + 0.5 + 30 * 0.025 + 1e-9
    assert all(1 <= n <= 2 for _, n in rep.worker_timeline)


def test_session_heterogeneous_workers_display_order():
    """Two workers at 1x and 3x speed: displayed timestamps monotone, some frames discarded."""
    cfg = el.SessionConfig(w_init=2, w_max=2, control=False, sample_interval=0.004, timeout=1.0)
    rep = el.run_session(_traj(3000), cfg, clock="sim", cost_fn=lambda w, f, t: 0.010 if w == 0 else 0.030)
    ts = rep.displayed_ts
    assert all(a <= b for a, b in zip(ts, ts[1:]))
    assert rep.n_displayed < rep.n_rendered


def test_invariants_randomized():
    """10k frames, random per-worker speeds and controller activity: displayed timestamps monotone,
    no stale render, 1 <= n_workers <= W_max."""
    rng = random.Random(0)
    speeds = [rng.uniform(0.004, 0.04) for _ in range(4)]
    cfg = el.SessionConfig(min_fps=80, max_fps=100, w_max=4, sample_interval=0.002, timeout=0.05)
    rep = el.run_session(_traj(10000), cfg, clock="sim",
                         cost_fn=lambda w, f, t: speeds[w % 4] * rng.uniform(0.5, 1.5))
    ts = rep.displayed_ts
    assert all(a <= b for a, b in zip(ts, ts[1:]))
    assert all(r.t_start - r.timestamp <= cfg.timeout + 1e-12 for r in rep.records)
    assert all(1 <= n <= 4 for _, n in rep.worker_timeline)


def test_hysteresis_no_change_inside_band():
    cfg = el.SessionConfig(min_fps=60, max_fps=120, w_max=3, sample_interval=0.005, timeout=1.0)
    rep = el.run_session(_traj(4000), cfg, clock="sim", cost_fn=lambda w, f, t: 0.010)   # ~100 FPS
    assert len(rep.worker_timeline) == 1


@pytest.mark.slow
def test_process_workers_elastic_start_and_stop():
    """workers are OS processes.  With every worker taking 40 ms per frame (25 FPS per worker)
    the controller starts worker processes up to w_max; frames come from several distinct processes,
    displayed timestamps stay monotone, no displayed frame is older than the timeout when its render
    started.  Then with 2 ms frames (~450 FPS at 1 worker pace > (1 + 1/N) Max) it stops them again."""
    rigs = [_rig(0.02 * k) for k in range(2000)]
    cfg = el.SessionConfig(min_fps=60, max_fps=120, w_max=3, w_init=1, sample_interval=1 / 200.0,
                           control_period=0.25, timeout=0.1)
    rep = el.run_session(rigs, cfg, clock="proc", duration=2.5,
                         worker_spec=("paper_2502_14938_b200.elastic", "sleep_worker", {"cost": 0.040}))
    assert max(n for _, n in rep.worker_timeline) == 3
    pids = {r.stats["pid"] for r in rep.records}
    assert len(pids) == 3 and all(p != __import__("os").getpid() for p in pids)
    ts = rep.displayed_ts
    assert len(ts) > 40 and all(a <= b for a, b in zip(ts, ts[1:]))
    assert all(r.t_start - r.timestamp <= cfg.timeout + 0.02 for r in rep.records)
    cfg2 = el.SessionConfig(min_fps=60, max_fps=120, w_max=3, w_init=3, sample_interval=1 / 500.0,
                            control_period=0.25, timeout=0.1)
    rep2 = el.run_session(rigs, cfg2, clock="proc", duration=2.0,
                          worker_spec=("paper_2502_14938_b200.elastic", "sleep_worker", {"cost": 0.002}))
    assert min(n for _, n in rep2.worker_timeline) == 1
