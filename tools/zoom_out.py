#!/usr/bin/env python
"""F2 zoom-out experiment (Figure "Rendering frame rate on the trajectory w.r.t
height"): the camera points at the centre of the C5 city and moves away from it, so more anchors are
decoded and more Gaussians rasterised per frame.

  PYTHONPATH=. python tools/zoom_out.py measure [frames] [out.json]   (GPU) per-frame end-to-end cost
      of one rendering worker (gsc_render_pair_host: pose in, both RGBA8 images in host memory) along
      the trajectory, plus a real-clock elastic session with worker PROCESSES (clock="proc")
  PYTHONPATH=. python tools/zoom_out.py simulate <measured.json> [out.json]   (CPU) the scheduler on
      the measured cost curve in simulated time: static (1 worker = 1 GPU) vs elastic (up to 8)

The FPS band is chosen relative to this GPU's range so that one worker crosses Min-FPS along the
trajectory (the paper's band [60, .] sits inside its consumer GPUs' range the same way).
"""
import json
import sys
import time

import numpy as np


def measure(frames=600, out=None):
    import torch
    import scenegen as sg
    import paper_2502_14938_b200 as gp
    from paper_2502_14938_b200 import elastic as el
    cfg = sg.config("C5Z")
    traj = sg.trajectory(cfg, frames)
    r = gp.Renderer(0, cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far, cfg.d_max).load(cfg.scene())
    hl = torch.empty((cfg.height, cfg.width, 4), dtype=torch.uint8).pin_memory()
    hr = torch.empty_like(hl).pin_memory()
    for rig in traj[:5]:
        r.render_host(rig, hl, hr, gp.GSC_FMT_RGBA8)
    r.reset_cache()
    ms, vis = [], []
    for rig in traj:
        t0 = time.perf_counter()
        r.render_host(rig, hl, hr, gp.GSC_FMT_RGBA8)
        ms.append(1000.0 * (time.perf_counter() - t0))
    hist = r.stats_history(len(traj))
    vis = [h["n_visible"] for h in hist][-len(traj):]
    dist = [float(np.linalg.norm(0.5 * (np.asarray(x.lp) + np.asarray(x.rp)) - cfg.center)) for x in traj]
    del r
    torch.cuda.empty_cache()
    res = {"config": "C5Z", "frames": len(traj), "distance_m": [round(d, 2) for d in dist],
           "ms_per_frame_e2e": [round(m, 4) for m in ms], "visible": vis}
    # real-clock session with one rendering worker PROCESS per worker; the poses replayed at 600 Hz
    ngpu = torch.cuda.device_count()
    mean_fps = 1000.0 / float(np.mean(ms))
    band = (round(0.9 * mean_fps), round(1.3 * mean_fps))
    rigs = [traj[min(len(traj) - 1, k // 2)] for k in range(2 * len(traj))]
    for name, wmax in (("static", 1), ("elastic", 2)):
        scfg = el.SessionConfig(min_fps=band[0], max_fps=band[1], w_max=wmax, w_init=1, sample_interval=1 / 600.0,
                                control_period=0.25, timeout=0.05)
        rep = el.run_session(rigs, scfg, clock="proc", duration=len(rigs) / 600.0,
                             worker_spec=("paper_2502_14938_b200.elastic", "gsc_worker", {"config": "C5Z"}))
        res["session_" + name] = dict(rep.as_dict(), n_gpus=ngpu, band=band, pids=sorted(set(rep.worker_pids.values())))
        print(name, json.dumps(res["session_" + name]), flush=True)
    print(json.dumps({k: v for k, v in res.items() if not isinstance(v, list)}), flush=True)
    if out:
        with open(out, "w") as fh:
            json.dump(res, fh)
    return res


def simulate(measured, out=None, w_max=8):
    """The scheduler on the measured cost curve (simulated time): pose k of the trajectory costs the
    measured end-to-end time of its frame on one GPU; each worker is one GPU.  Static = 1 worker; elastic
    = the FPS-band controller with up to w_max workers.  FPS traces per trajectory position."""
    from paper_2502_14938_b200 import elastic as el
    import scenegen as sg
    m = json.load(open(measured))
    cost = np.asarray(m["ms_per_frame_e2e"]) / 1000.0
    n = len(cost)
    fps1 = 1.0 / cost
    band = (float(np.percentile(fps1, 60)), float(np.percentile(fps1, 60)) * 1.5)
    hz = 4.0 * float(np.max(fps1))                # pose sampling well above any render rate
    per_pose = 4                                  # each trajectory frame held for 4 samples
    rigs = []
    traj = sg.trajectory(sg.config("C5Z"), n)
    for k in range(n):
        rigs += [traj[k]] * per_pose
    # distinct poses (the queue's pose threshold): nudge repeated samples
    for k in range(len(rigs)):
        r = rigs[k]
        rigs[k] = sg.Rig(lp=np.asarray(r.lp) + 0.02 * (k % per_pose), lq=r.lq, rp=np.asarray(r.rp) + 0.02 * (k % per_pose),
                         rq=r.rq, t=k / hz)

    def cost_fn(w, frame, t):
        return float(cost[min(n - 1, int(t * hz) // per_pose)])

    res = {"band_fps": [round(band[0], 1), round(band[1], 1)], "pose_hz": round(hz, 1), "w_max": w_max}
    for name, wm in (("static", 1), ("elastic", w_max)):
        cfg = el.SessionConfig(min_fps=band[0], max_fps=band[1], w_max=wm, w_init=1, sample_interval=1 / hz,
                               control_period=0.05, timeout=0.05, window=30)
        rep = el.run_session(rigs, cfg, clock="sim", cost_fn=cost_fn)
        shown = sorted(r.t_end for r in rep.records if r.displayed)
        # FPS per trajectory segment (60 frames of the trajectory)
        seg = []
        for s0 in range(0, n, 60):
            t0, t1 = s0 * per_pose / hz, min(n, s0 + 60) * per_pose / hz
            cnt = sum(1 for t in shown if t0 <= t < t1)
            seg.append({"frames": [s0, min(n, s0 + 60) - 1],
                        "distance_m": round(float(np.mean(m["distance_m"][s0:s0 + 60])), 1),
                        "fps": round(cnt / (t1 - t0), 1)})
        res[name] = dict(rep.as_dict(), segments=seg)
        print(name, json.dumps({k: v for k, v in res[name].items() if k != "worker_timeline"}), flush=True)
    if out:
        with open(out, "w") as fh:
            json.dump(res, fh, indent=1)
    return res


if __name__ == "__main__":
    if sys.argv[1] == "measure":
        measure(int(sys.argv[2]) if len(sys.argv) > 2 else 600, sys.argv[3] if len(sys.argv) > 3 else None)
    else:
        simulate(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
