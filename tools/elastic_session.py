#!/usr/bin/env python
"""Real-time elastic rendering session on this box's GPUs: the trajectory's poses are
sampled at 90 Hz into the shared queue, each worker owns a private pipeline (a Renderer: scene copy,
cache, streams) on GPU (worker mod n_gpus) and renders end to end (pinned host images), the FPS-band
controller starts / stops workers, display-order sync drops out-of-order frames.

  PYTHONPATH=. python tools/elastic_session.py [config] [seconds] [min_fps] [max_fps] [w_max] [out.json]
"""
import json
import sys


def main():
    import torch
    import scenegen as sg
    import paper_2502_14938_b200 as gp
    from paper_2502_14938_b200 import elastic as el
    config = sys.argv[1] if len(sys.argv) > 1 else "C4"
    seconds = float(sys.argv[2]) if len(sys.argv) > 2 else 10.0
    min_fps = float(sys.argv[3]) if len(sys.argv) > 3 else 72.0
    max_fps = float(sys.argv[4]) if len(sys.argv) > 4 else 120.0
    w_max = int(sys.argv[5]) if len(sys.argv) > 5 else 2
    cfg = sg.config(config)
    sc = cfg.scene()
    traj = sg.trajectory(cfg)
    ngpu = max(1, torch.cuda.device_count())

    def make_worker(w):
        dev = w % ngpu
        r = gp.Renderer(dev, cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far, cfg.d_max).load(sc)
        hl = torch.empty((cfg.height, cfg.width, 4), dtype=torch.uint8).pin_memory()
        hr = torch.empty((cfg.height, cfg.width, 4), dtype=torch.uint8).pin_memory()

        def render(rig):
            r.render_host(rig, hl, hr, gp.GSC_FMT_RGBA8)
            return {}
        return render

    # the trajectory replayed at 90 Hz for `seconds` (cycling)
    n = int(seconds * 90)
    poses = [traj[k % len(traj)] for k in range(n)]
    scfg = el.SessionConfig(min_fps=min_fps, max_fps=max_fps, w_max=w_max, sample_interval=1 / 90.0)
    rep = el.run_session(poses, scfg, clock="real", make_worker=make_worker, duration=seconds)
    ts = rep.displayed_ts
    out = dict(rep.as_dict(), config=config, seconds=seconds, min_fps=min_fps, max_fps=max_fps, w_max=w_max,
               n_gpus=ngpu, displayed_monotone=all(a <= b for a, b in zip(ts, ts[1:])),
               note="pose sampling 90 Hz: the displayed FPS is bounded by the pose rate")
    print(json.dumps(out), flush=True)
    if len(sys.argv) > 6:
        with open(sys.argv[6], "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
