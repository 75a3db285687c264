"""Elastic parallel rendering (the paper's second contribution, Alg. 2
P:258-285): a timestamped shared camera queue fed by pose-threshold sampling, a pool of
rendering workers (each owning a private GS-Cache pipeline: its own `Renderer`, cache and streams), an
FPS-band controller that starts a worker below Min-FPS and stops one above (1 + 1/N) Max-FPS, and
display-order synchronisation that drops frames older than the last one written.

Three modes: ``run_session(..., clock="sim")`` drives the identical control logic
single-threaded on a virtual clock with injected per-frame costs (deterministic, for tests);
``clock="proc"`` is the paper's deployment ("the scheduler starts a new rendering worker
process"): one OS process per worker, each owning a private pipeline (its own CUDA context, scene copy
and cache on GPU w mod n_gpus), fed by the coordinator's shared queue; ``clock="real"`` runs the
workers as threads of one process (same logic, cheaper start-up).

Readings (R25): FPS = last 30 displayed frames / their time span; control period 0.5 s with
at most one action; pose thresholds 0.01 m / 0.5 degree; queue capacity 8, timeout 100 ms; the
worker stopped is the most recently started (LIFO); "99% FPS" = 1st percentile of per-frame FPS.
"""
from __future__ import annotations

import collections
import dataclasses
import heapq
import math
import threading
import time
from typing import Callable, List, Optional

import numpy as np


# ------------------------------------------------------------------ queue (Alg. 2 "shared queue")
@dataclasses.dataclass
class QueueEntry:
    rig: object
    timestamp: float


def _pose_delta(a, b):
    """(position change, angle change in degrees) between two rigs (StereoRig: lp, lq, rp, rq),
    measured on the left eye."""
    pa, qa = np.asarray(a.lp, np.float64), np.asarray(a.lq, np.float64)
    pb, qb = np.asarray(b.lp, np.float64), np.asarray(b.lq, np.float64)
    dp = float(np.linalg.norm(pa - pb))
    d = abs(float(np.dot(qa / np.linalg.norm(qa), qb / np.linalg.norm(qb))))
    return dp, math.degrees(2.0 * math.acos(min(1.0, d)))


class CameraQueue:
    """Timestamped FIFO of poses, multi-producer / multi-consumer safe."""

    def __init__(self, timeout=0.100, capacity=8, delta_p=0.01, delta_theta_deg=0.5):
        self.timeout, self.capacity = timeout, capacity
        self.delta_p, self.delta_theta = delta_p, delta_theta_deg
        self._q: collections.deque = collections.deque()
        self._last = None
        self._lock = threading.Lock()
        self.dropped_full = 0
        self.dropped_stale = 0

    def submit_pose(self, rig, now: float) -> bool:
        """Alg. 2 "HMD device pose change exceeds threshold": accepted iff the first pose or the
        position moved more than delta_p or the orientation more than delta_theta since the last
        accepted pose; a full queue drops its oldest entry."""
        with self._lock:
            if self._last is not None:
                dp, dth = _pose_delta(rig, self._last)
                if not (dp > self.delta_p or dth > self.delta_theta):
                    return False
            self._last = rig
            if len(self._q) >= self.capacity:
                self._q.popleft()
                self.dropped_full += 1
            self._q.append(QueueEntry(rig, now))
            return True

    def take_work(self, now: float) -> Optional[QueueEntry]:
        """Pop the first entry younger than the timeout, discarding stale ones."""
        with self._lock:
            while self._q:
                e = self._q.popleft()
                if now - e.timestamp > self.timeout:
                    self.dropped_stale += 1
                    continue
                return e
            return None

    def __len__(self):
        with self._lock:
            return len(self._q)


# ------------------------------------------------------------------ controller
START, STOP, NONE = "start", "stop", None


class FpsController:
    """FPS-band worker control: StartWorker below min_fps (while n < w_max), StopWorker above
    (1 + 1/n) max_fps (while n > 1), at most one action per control period."""

    def __init__(self, min_fps=60.0, max_fps=120.0, w_max=2, window=30, period=0.5):
        assert 0 < min_fps <= max_fps and w_max >= 1
        self.min_fps, self.max_fps, self.w_max = min_fps, max_fps, w_max
        self.window, self.period = window, period
        self.n_workers = 1
        self._last_action_t = -math.inf

    def control_step(self, measured_fps: float, now: float = math.inf) -> Optional[str]:
        if now - self._last_action_t < self.period:
            return NONE
        act = NONE
        if measured_fps < self.min_fps and self.n_workers < self.w_max:
            act = START
        elif measured_fps > (1.0 + 1.0 / self.n_workers) * self.max_fps and self.n_workers > 1:
            act = STOP
        if act is not NONE:
            self.n_workers += 1 if act == START else -1
            self._last_action_t = now
        return act


class FpsMeter:
    """FPS of the last `window` displayed frames (count / time span)."""

    def __init__(self, window=30):
        self.t: collections.deque = collections.deque(maxlen=window)

    def add(self, t: float):
        self.t.append(t)

    def fps(self) -> float:
        if len(self.t) < 2 or self.t[-1] <= self.t[0]:
            return 0.0
        return (len(self.t) - 1) / (self.t[-1] - self.t[0])


# ------------------------------------------------------------------ display order (Alg. 2 l.275-282)
class DisplaySync:
    """Write a frame unless it is older than the last one written; linearizable."""

    def __init__(self):
        self.last_written = -math.inf
        self._lock = threading.Lock()

    def try_display(self, timestamp: float) -> bool:
        with self._lock:
            if timestamp < self.last_written:
                return False
            self.last_written = timestamp
            return True


# ------------------------------------------------------------------ session
@dataclasses.dataclass
class FrameRecord:
    timestamp: float
    worker: int
    t_start: float
    t_end: float
    displayed: bool
    stats: dict = dataclasses.field(default_factory=dict)


@dataclasses.dataclass
class SessionConfig:
    min_fps: float = 60.0
    max_fps: float = 120.0
    w_max: int = 2
    w_init: int = 1
    timeout: float = 0.100
    capacity: int = 8
    delta_p: float = 0.01
    delta_theta_deg: float = 0.5
    sample_interval: float = 1.0 / 90.0      # HMD pose sampling (90 Hz)
    control_period: float = 0.5
    window: int = 30
    control: bool = True


@dataclasses.dataclass
class SessionReport:
    records: List[FrameRecord]
    displayed_ts: List[float]
    worker_timeline: List[tuple]             # (time, n_workers)
    avg_fps: float
    p1_fps: float
    n_rendered: int
    n_displayed: int
    n_stale: int

    def as_dict(self):
        return {"avg_fps": self.avg_fps, "p1_fps": self.p1_fps, "n_rendered": self.n_rendered,
                "n_displayed": self.n_displayed, "n_stale_dropped": self.n_stale,
                "worker_timeline": self.worker_timeline}


def _report(records, displayed_t, timeline, queue):
    shown = sorted(t for t in displayed_t)
    if len(shown) >= 2:
        span = shown[-1] - shown[0]
        avg = (len(shown) - 1) / span if span > 0 else 0.0
        inst = 1.0 / np.maximum(np.diff(np.asarray(shown)), 1e-9)
        p1 = float(np.percentile(inst, 1))
    else:
        avg = p1 = 0.0
    return SessionReport(records=records, displayed_ts=[r.timestamp for r in records if r.displayed],
                         worker_timeline=timeline, avg_fps=avg, p1_fps=p1, n_rendered=len(records),
                         n_displayed=sum(r.displayed for r in records), n_stale=queue.dropped_stale)


def run_session(trajectory, cfg: SessionConfig, clock: str = "sim",
                cost_fn: Optional[Callable[[int, int, float], float]] = None,
                make_worker: Optional[Callable[[int], Callable]] = None, duration: Optional[float] = None,
                worker_spec: Optional[tuple] = None, prewarm: bool = True):
    """Alg. 2 top-level loop.  trajectory: list of rigs sampled every cfg.sample_interval.
    clock="sim": virtual time; worker w renders a frame submitted at t in cost_fn(w, frame, t) seconds.
    clock="real": wall time; make_worker(w) returns render(rig) -> stats dict (one private pipeline
    per worker, e.g. a Renderer on its own GPU).
    clock="proc": wall time, one process per worker; worker_spec = (module, function, kwargs) names a
    module-level factory function(w, **kwargs) -> render(rig), called inside the worker process.  With
    prewarm (default) all w_max worker processes build their pipelines (scene load: seconds at city
    scale) before the clock starts and the controller activates / deactivates them, so a start takes
    effect at once; without it a start spawns the process and the worker joins when its scene is loaded."""
    queue = CameraQueue(cfg.timeout, cfg.capacity, cfg.delta_p, cfg.delta_theta_deg)
    ctrl = FpsController(cfg.min_fps, cfg.max_fps, cfg.w_max, cfg.window, cfg.control_period)
    ctrl.n_workers = cfg.w_init
    sync = DisplaySync()
    meter = FpsMeter(cfg.window)
    if duration is None:
        duration = len(trajectory) * cfg.sample_interval
    if clock == "sim":
        return _run_sim(trajectory, cfg, queue, ctrl, sync, meter, cost_fn, duration)
    if clock == "real":
        return _run_real(trajectory, cfg, queue, ctrl, sync, meter, make_worker, duration)
    if clock == "proc":
        return _run_proc(trajectory, cfg, queue, ctrl, sync, meter, worker_spec, duration, prewarm)
    raise ValueError(clock)


def _run_sim(trajectory, cfg, queue, ctrl, sync, meter, cost_fn, duration):
    """Discrete-event simulation: events (time, seq, kind, payload) processed in time order."""
    assert cost_fn is not None
    ev = []
    seq = 0

    def push(t, kind, payload=None):
        nonlocal seq
        heapq.heappush(ev, (t, seq, kind, payload))
        seq += 1

    for k in range(len(trajectory)):
        push(k * cfg.sample_interval, "pose", k)
    if cfg.control:
        t = cfg.control_period
        while t <= duration:
            push(t, "control")
            t += cfg.control_period
    active = list(range(ctrl.n_workers))      # started workers, LIFO order
    busy = set()
    next_id = len(active)
    records, displayed, timeline = [], [], [(0.0, len(active))]
    frame_no = 0

    def dispatch(now):
        nonlocal frame_no
        for w in active:
            if w in busy:
                continue
            e = queue.take_work(now)
            if e is None:
                return
            busy.add(w)
            cost = cost_fn(w, frame_no, now)
            push(now + cost, "done", (w, e, now, frame_no))
            frame_no += 1

    while ev:
        now, _, kind, payload = heapq.heappop(ev)
        if now > duration + 10.0:
            break
        if kind == "pose":
            queue.submit_pose(trajectory[payload], now)
        elif kind == "done":
            w, e, t0, fno = payload
            busy.discard(w)
            shown = sync.try_display(e.timestamp)
            records.append(FrameRecord(e.timestamp, w, t0, now, shown))
            if shown:
                meter.add(now)
                displayed.append(now)
        elif kind == "control":
            act = ctrl.control_step(meter.fps(), now)
            if act == START:
                active.append(next_id)
                next_id += 1
            elif act == STOP:
                active.pop()                   # LIFO; a busy worker finishes its frame
            if act is not NONE:
                timeline.append((now, len(active)))
        dispatch(now)
    return _report(records, displayed, timeline, queue)


def _run_real(trajectory, cfg, queue, ctrl, sync, meter, make_worker, duration):
    assert make_worker is not None
    records, displayed = [], []
    lock = threading.Lock()
    stop_flags, threads, errors = {}, {}, []
    done = threading.Event()
    # the initial workers' pipelines are built before the clock starts (setup, not session time);
    # workers the controller starts later build theirs on their own thread, as a real start would
    ready = {w: make_worker(w) for w in range(ctrl.n_workers)}
    t0 = time.perf_counter()
    now = lambda: time.perf_counter() - t0  # noqa: E731
    timeline = [(0.0, ctrl.n_workers)]

    def worker_loop(w, flag):
        try:
            render = ready.pop(w, None) or make_worker(w)
            while not flag.is_set() and not done.is_set():
                e = queue.take_work(now())
                if e is None:
                    time.sleep(0.0005)
                    continue
                ts = now()
                st = render(e.rig)
                te = now()
                shown = sync.try_display(e.timestamp)
                with lock:
                    records.append(FrameRecord(e.timestamp, w, ts, te, shown, st or {}))
                    if shown:
                        meter.add(te)
                        displayed.append(te)
        except BaseException as exc:   # a worker crash aborts the session
            errors.append(exc)
            done.set()

    def start(w):
        flag = threading.Event()
        stop_flags[w] = flag
        th = threading.Thread(target=worker_loop, args=(w, flag), daemon=True)
        threads[w] = th
        th.start()

    order = []
    for w in range(ctrl.n_workers):
        start(w)
        order.append(w)
    next_id = ctrl.n_workers
    k = 0
    next_ctrl = cfg.control_period
    while not done.is_set():
        t = now()
        if t >= duration:
            break
        while k < len(trajectory) and k * cfg.sample_interval <= t:
            queue.submit_pose(trajectory[k], t)
            k += 1
        if cfg.control and t >= next_ctrl:
            with lock:
                fps = meter.fps()
            act = ctrl.control_step(fps, t)
            if act == START:
                start(next_id)
                order.append(next_id)
                next_id += 1
            elif act == STOP:
                stop_flags[order.pop()].set()
            if act is not NONE:
                timeline.append((t, len(order)))
            next_ctrl += cfg.control_period
        time.sleep(0.001)
    done.set()
    for th in threads.values():
        th.join(timeout=30)
    if errors:
        raise RuntimeError("rendering worker failed; session aborted") from errors[0]
    return _report(records, displayed, timeline, queue)


# ------------------------------------------------------------------ process workers
def _worker_main(w, spec, tasks, results):
    """Body of one rendering worker process: build the private pipeline, report ready, then render the
    poses the coordinator hands over until told to stop (None)."""
    import importlib
    import os
    try:
        mod, fn, kw = spec
        render = getattr(importlib.import_module(mod), fn)(w, **kw)
        results.put(("ready", w, os.getpid(), None))
        while True:
            item = tasks.get()
            if item is None:
                break
            k, rig = item
            t0 = time.perf_counter()
            st = render(rig)
            results.put(("done", w, k, (t0, time.perf_counter(), st or {})))
    except BaseException as exc:   # reported to the coordinator, which aborts the session
        results.put(("error", w, None, repr(exc)))
    results.put(("exit", w, None, None))


def _run_proc(trajectory, cfg, queue, ctrl, sync, meter, spec, duration, prewarm=True):
    """The coordinator: samples poses into the shared queue, hands the head of the queue to each idle
    worker process (Alg. 2: a worker takes the next camera when it finishes the previous one), displays in
    timestamp order, and runs the FPS-band controller, starting / stopping worker processes.  Times are
    CLOCK_MONOTONIC (time.perf_counter), shared by all processes of the machine."""
    import multiprocessing as mp
    assert spec is not None
    ctx = mp.get_context("spawn")
    results = ctx.Queue()
    procs, tasks = {}, {}
    ready, idle, busy = set(), [], {}
    pids = {}
    records, displayed = [], []
    order = []

    def start(w):
        tasks[w] = ctx.Queue()
        p = ctx.Process(target=_worker_main, args=(w, spec, tasks[w], results), daemon=True)
        p.start()
        procs[w] = p
        order.append(w)

    n_spawn = cfg.w_max if prewarm else ctrl.n_workers
    for w in range(n_spawn):
        start(w)
    standby = []                       # prewarmed workers not yet activated (ascending id)
    del order[ctrl.n_workers:]
    # the spawned workers' pipelines are built before the clock starts (setup, not session time)
    while len(ready) < n_spawn:
        kind, w, a, b = results.get(timeout=900)
        if kind == "error":
            raise RuntimeError(f"worker {w} failed to start: {b}")
        if kind == "ready":
            ready.add(w)
            pids[w] = a
    idle.extend(range(ctrl.n_workers))
    standby.extend(range(ctrl.n_workers, n_spawn))
    t0 = time.perf_counter()
    now = lambda: time.perf_counter() - t0  # noqa: E731
    timeline = [(0.0, len(order))]
    stopping = set()
    k = 0
    next_ctrl = cfg.control_period
    jobs = {}
    err = None
    while err is None:
        t = now()
        if t >= duration:
            break
        while k < len(trajectory) and k * cfg.sample_interval <= t:
            queue.submit_pose(trajectory[k], t)
            k += 1
        # hand work to idle workers (head of the queue, stale entries dropped)
        while idle:
            e = queue.take_work(now())
            if e is None:
                break
            w = idle.pop(0)
            jobs[w] = (e, now())
            tasks[w].put((len(records) + len(jobs), e.rig))
        try:
            kind, w, a, b = results.get(timeout=0.0005)
        except Exception:
            kind = None
        if kind == "done":
            e, ts = jobs.pop(w)
            te = now()
            shown = sync.try_display(e.timestamp)
            records.append(FrameRecord(e.timestamp, w, ts, te, shown, dict(b[2], pid=pids.get(w))))
            if shown:
                meter.add(te)
                displayed.append(te)
            if w in stopping:
                stopping.discard(w)
                if prewarm:
                    standby.insert(0, w)
                else:
                    tasks[w].put(None)
            else:
                idle.append(w)
        elif kind == "ready":
            ready.add(w)
            pids[w] = a
            if w in order:
                idle.append(w)
        elif kind == "error":
            err = RuntimeError(f"rendering worker {w} failed: {b}")
        if cfg.control and t >= next_ctrl:
            act = ctrl.control_step(meter.fps(), t)
            if act == START:
                if standby:
                    w = standby.pop(0)
                    order.append(w)
                    idle.append(w)
                else:
                    start(len(procs))
            elif act == STOP:
                w = order.pop()                # LIFO; a busy worker finishes its frame first
                if w in idle:
                    idle.remove(w)
                    if prewarm:
                        standby.insert(0, w)
                    else:
                        tasks[w].put(None)
                else:
                    stopping.add(w)
            if act is not NONE:
                timeline.append((t, len(order)))
            next_ctrl += cfg.control_period
    for w, p in procs.items():
        if p.is_alive():
            tasks[w].put(None)
    for p in procs.values():
        p.join(timeout=60)
        if p.is_alive():
            p.terminate()
    if err is not None:
        raise err
    rep = _report(records, displayed, timeline, queue)
    rep.worker_pids = dict(pids)
    return rep


def sleep_worker(w, cost: float = 0.01, cost_by_worker: Optional[dict] = None):
    """A synthetic rendering worker for CPU tests and simulations of the process mode: "renders" a pose
    by sleeping `cost` seconds (or cost_by_worker[w])."""
    c = (cost_by_worker or {}).get(w, cost)

    def render(rig):
        time.sleep(c)
        return {"cost": c}
    return render


def gsc_worker(w, config: str = "C4", fmt_rgba8: bool = True):
    """A GS-Cache rendering worker: its own Renderer (scene copy, cache, streams) on GPU w mod n_gpus,
    rendering each pose end to end into its pinned host images."""
    import torch
    import scenegen as sg
    import paper_2502_14938_b200 as gp
    cfg = sg.config(config)
    dev = w % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    r = gp.Renderer(dev, cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far, cfg.d_max).load(cfg.scene())
    fmt = gp.GSC_FMT_RGBA8 if fmt_rgba8 else gp.GSC_FMT_RGB_F32_PLANAR
    shape = (cfg.height, cfg.width, 4) if fmt_rgba8 else (3, cfg.height, cfg.width)
    dt = torch.uint8 if fmt_rgba8 else torch.float32
    hl = torch.empty(shape, dtype=dt).pin_memory()
    hr = torch.empty(shape, dtype=dt).pin_memory()

    def render(rig):
        r.render_host(rig, hl, hr, fmt)
        return {"device": dev}
    return render
