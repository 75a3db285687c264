#!/usr/bin/env python
"""Per-stage times along a config's trajectory (serial replay with stage events), in frame buckets.

  tools/stage_profile.py [config] [frames] [bucket] [extra GSC_F_* flag names, comma separated]
"""
import sys

import numpy as np


def main():
    import os
    if os.environ.get("GSC_AB_LIB"):   # A/B measurement of a variant build (tools/ab_build.py)
        from paper_2502_14938_b200 import _abi
        _abi.SO_PATH = os.environ["GSC_AB_LIB"]
    import torch
    import scenegen as sg
    import paper_2502_14938_b200 as gp
    cfg = sg.config(sys.argv[1] if len(sys.argv) > 1 else "C4")
    nf = int(sys.argv[2]) if len(sys.argv) > 2 else 600
    bucket = int(sys.argv[3]) if len(sys.argv) > 3 else 50
    sc = cfg.scene()
    traj = sg.trajectory(cfg)[:nf]
    extra = 0
    if len(sys.argv) > 4 and sys.argv[4]:
        for name in sys.argv[4].split(","):
            extra |= getattr(gp, name)
    r = gp.Renderer(0, cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far, cfg.d_max,
                    flags=gp.GSC_F_STAGE_TIMING | gp.GSC_F_SERIAL | extra).load(sc)
    out_l, out_r = r.alloc_outputs(gp.GSC_FMT_RGBA8)
    st = torch.cuda.current_stream()
    for rig in traj[:5]:
        r.render_into(rig, out_l, out_r, gp.GSC_FMT_RGBA8, st)
    torch.cuda.synchronize()
    r.reset_cache()
    r.stats_history()
    for rig in traj:
        r.render_into(rig, out_l, out_r, gp.GSC_FMT_RGBA8, st)
    torch.cuda.synchronize()
    h = r.stats_history(nf)
    stages = ["cull", "derive", "project", "depth_sort", "emit", "tile_sort", "ranges", "blend"]
    print("frames  " + " ".join(f"{s:>10s}" for s in stages) + "      total  splats(M) pairs(M) fixups")
    for b0 in range(0, len(h), bucket):
        hb = h[b0:b0 + bucket]
        ms = [np.mean([x["ms_" + s] for x in hb]) for s in stages]
        tot = np.mean([x["ms_total"] for x in hb])
        print(f"{b0:3d}-{b0 + len(hb) - 1:3d} " + " ".join(f"{m:10.3f}" for m in ms) +
              f" {tot:10.3f} {np.mean([x['n_splats'] for x in hb]) / 1e6:9.2f} {np.mean([x['n_pairs'] for x in hb]) / 1e6:8.2f}"
              f" {np.mean([x.get('n_blend_fixup', 0) for x in hb]):7.0f}")


if __name__ == "__main__":
    main()
