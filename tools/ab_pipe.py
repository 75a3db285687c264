#!/usr/bin/env python
"""Pipelined frame rate (the bench's mode: frame f+1's front end overlaps frame f's blend) of the current
build and of ab/<variant> libraries, along the first frames of a config's trajectory (scratch A/B tool).

  tools/ab_pipe.py [config] [frames] [variant ...]      (variant 'cur' = the in-tree build)

Each variant runs in its own process (one library per process); device time by CUDA events on the
caller's stream, 3 repetitions, the median reported.
"""
import os
import subprocess
import sys


def child(cfg_name, nf):
    if os.environ.get("GSC_AB_LIB"):
        from paper_2502_14938_b200 import _abi
        _abi.SO_PATH = os.environ["GSC_AB_LIB"]
    import numpy as np
    import torch
    import scenegen as sg
    import paper_2502_14938_b200 as gp
    cfg = sg.config(cfg_name)
    traj = sg.trajectory(cfg)[:nf]
    r = gp.Renderer(0, cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far, cfg.d_max).load(cfg.scene())
    o = r.alloc_outputs(gp.GSC_FMT_RGBA8)
    st = torch.cuda.current_stream()
    res = []
    for rep in range(4):
        r.reset_cache()
        for rig in traj[:3]:
            r.render_into(rig, *o, gp.GSC_FMT_RGBA8, st)
        r.reset_cache()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for rig in traj:
            r.render_into(rig, *o, gp.GSC_FMT_RGBA8, st)
        e1.record(st)
        torch.cuda.synchronize()
        if rep:
            res.append(e0.elapsed_time(e1) / nf)
    ms = float(np.median(res))
    print(f"{ms:.4f} ms/frame  {1000 / ms:.1f} frames/s  (reps {', '.join(f'{x:.4f}' for x in res)})")


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child(sys.argv[2], int(sys.argv[3]))
        return
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
    nf = int(sys.argv[2]) if len(sys.argv) > 2 else 300
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for v in (sys.argv[3:] or ["cur"]):
        env = dict(os.environ, PYTHONPATH=root)
        if v != "cur":
            env["GSC_AB_LIB"] = os.path.join(root, "ab", v, "libgscache.so")
        out = subprocess.run([sys.executable, os.path.abspath(__file__), "--child", cfg, str(nf)], env=env,
                             capture_output=True, text=True)
        print(f"{v:12s} {out.stdout.strip()} {out.stderr.strip()[-300:] if out.returncode else ''}", flush=True)


if __name__ == "__main__":
    main()
