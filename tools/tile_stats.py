#!/usr/bin/env python
"""Per-tile pair-count statistics of a config's trajectory (GPU): how the
(tile, depth) sort's segments are distributed.

  tools/tile_stats.py [config] [frame ...]
"""
import sys

import numpy as np


def main():
    import scenegen as sg
    import paper_2502_14938_b200 as gp
    cfg = sg.config(sys.argv[1] if len(sys.argv) > 1 else "C4")
    frames = [int(a) for a in sys.argv[2:]] or [0, 50, 100, 200, 300, 450, 599]
    sc = cfg.scene()
    traj = sg.trajectory(cfg)
    r = gp.Renderer(0, cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far, cfg.d_max).load(sc)
    want = set(frames)
    for f in range(max(frames) + 1):
        _, _, st = r.render(traj[f])
        if f not in want:
            continue
        sp = r.debug("splats")
        kept = int((sp[:, 12] > 0).sum())
        rg = r.debug("ranges").astype(np.int64)
        n = rg[:, 1] - rg[:, 0]
        P = n.sum()
        q = np.percentile(n, [50, 90, 99, 99.9])
        big = {k: float(n[n > k].sum()) / max(P, 1) for k in (2048, 4096, 8192, 16384)}
        print(f"frame {f}: pairs {P} splats {st['n_splats']} tiles {len(n)} mean {n.mean():.0f} "
              f"p50/90/99/99.9 {q.astype(int).tolist()} max {n.max()} "
              f"share of pairs in tiles > 2k/4k/8k/16k: " + " ".join(f"{v:.3f}" for v in big.values()) +
              f" tiles>4096: {(n > 4096).sum()} splats with >= 1 kept tile: {kept} ({kept / max(1, len(sp)):.3f})", flush=True)


if __name__ == "__main__":
    main()
