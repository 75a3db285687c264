#!/usr/bin/env python
"""Blend lane-slot utilisation (scratch): with an instrumented build (ab/blendcnt, n_exp := 32 x staged
splats per warp) prints, per frame, useful lane evaluations (n_evals: up to each lane's stop) over the
lane slots the warps issue, and the regular build's n_evals / n_exp (accepted)."""
import os
import sys


def main():
    if os.environ.get("GSC_AB_LIB"):
        from paper_2502_14938_b200 import _abi
        _abi.SO_PATH = os.environ["GSC_AB_LIB"]
    import torch
    import scenegen as sg
    import paper_2502_14938_b200 as gp
    cfg = sg.config(sys.argv[1] if len(sys.argv) > 1 else "C4")
    frames = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,10,100,300,599").split(",")]
    traj = sg.trajectory(cfg)
    r = gp.Renderer(0, cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far, cfg.d_max,
                    flags=gp.GSC_F_COUNT_EVALS).load(cfg.scene())
    o = r.alloc_outputs(gp.GSC_FMT_RGBA8)
    for f in frames:
        r.reset_cache()
        for k in range(max(0, f - 3), f + 1):
            r.render_into(traj[k], *o, gp.GSC_FMT_RGBA8)
        torch.cuda.synchronize()
        h = r.stats_history(1)[-1]
        print(f"frame {f}: n_evals {h['n_evals'] / 1e6:.1f}M  n_exp {h['n_exp'] / 1e6:.1f}M  ratio {h['n_evals'] / max(h['n_exp'], 1):.3f}")


if __name__ == "__main__":
    main()
