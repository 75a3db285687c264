#!/usr/bin/env python
"""Splat statistics along a trajectory (GPU): how many splats (live Gaussian, eye) keep at least one tile,
how the kept-tile counts are distributed, pairs per tile.  PYTHONPATH=. python tools/splat_stats.py [config] [frames...]"""
import sys

import numpy as np


def main():
    import scenegen as sg
    import paper_2502_14938_b200 as gp
    cfg = sg.config(sys.argv[1] if len(sys.argv) > 1 else "C4")
    frames = [int(a) for a in sys.argv[2:]] or [0, 10, 50, 100, 200, 300, 450, 599]
    sc = cfg.scene()
    traj = sg.trajectory(cfg)
    r = gp.Renderer(0, cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far, cfg.d_max).load(sc)
    want = set(frames)
    for f, rig in enumerate(traj[:max(frames) + 1]):
        _, _, st = r.render(rig)
        if f not in want:
            continue
        sp = r.debug("splats")
        kept = sp[:, 12]
        nz = kept > 0
        rg = r.debug("ranges")
        per_tile = (rg[:, 1] - rg[:, 0]).astype(np.int64)
        print(f"frame {f}: splats {len(sp)} with tiles {int(nz.sum())} ({nz.mean():.1%}); pairs {st['n_pairs']}; "
              f"kept/splat mean {kept[nz].mean():.2f} p50 {np.percentile(kept[nz], 50):.0f} p99 {np.percentile(kept[nz], 99):.0f} "
              f"max {kept.max():.0f}; pairs/tile mean {per_tile.mean():.0f} p99 {np.percentile(per_tile, 99):.0f} max {per_tile.max()}",
              flush=True)


if __name__ == "__main__":
    main()
