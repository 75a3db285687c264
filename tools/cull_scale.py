#!/usr/bin/env python
"""Cull (a1 + a2) at the paper's City scale, cold in L2 ("L2-resident at N = 1M, so
measure cold and at the paper's City scale N ~ 17-18.6M").

A synthetic city of N anchors at C5's anchor density (side grows with sqrt(N)), the C5-shaped
ground-to-aerial trajectory; F frames rendered through the C ABI with per-stage CUDA events
(GSC_F_STAGE_TIMING | GSC_F_SERIAL).  The cull stage reads N x 21 B per frame (378 MB at 18M) --
three times the 126 MB L2 -- so every frame is cold for it.  Prints one JSON line (also written to
the path given as the last argument).

  tools/cull_scale.py [N=18000000] [frames=60] [out.json]
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(n=18_000_000, frames=60, out=None):
    if os.environ.get("GSC_AB_LIB"):   # A/B measurement of a variant build (tools/ab_build.py)
        from paper_2502_14938_b200 import _abi
        _abi.SO_PATH = os.environ["GSC_AB_LIB"]
    import torch
    import scenegen as sg
    import paper_2502_14938_b200 as gp
    import bench

    side = 900.0 * math.sqrt(n / 5_000_000)
    cfg = sg.Config(f"CITY{n // 1_000_000}M", n, side, 5, 1920, 1080, 70.0, 10)
    t0 = time.time()
    sc = cfg.scene()
    gen_s = time.time() - t0
    c = cfg.center
    traj = sg.make_orbit(c, 0.3 * side, 0.7 * side, 1.7, 300.0, frames, 0.25)
    r = gp.Renderer(0, cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far, cfg.d_max,
                    flags=gp.GSC_F_STAGE_TIMING | gp.GSC_F_SERIAL, pair_capacity=1 << 28).load(sc)
    out_l, out_r = r.alloc_outputs(gp.GSC_FMT_RGBA8)
    stream = torch.cuda.current_stream()
    for rig in traj[:3]:                       # warm-up
        r.render_into(rig, out_l, out_r, gp.GSC_FMT_RGBA8, stream)
    torch.cuda.synchronize()
    r.reset_cache()
    r.stats_history()
    for rig in traj:
        r.render_into(rig, out_l, out_r, gp.GSC_FMT_RGBA8, stream)
    torch.cuda.synchronize()
    hist = r.stats_history(frames)
    ms = sum(h["ms_cull"] for h in hist) / len(hist)
    byts = sum(bench._stage_bytes(h, n, 10, cfg.width, cfg.height, 4)["cull"] for h in hist) / len(hist)
    peak = bench._peaks()["hbm_gbs"]
    gbs = byts / (ms / 1e3) / 1e9
    line = {"what": "cull stage (cull_classify + cull_compact incl. the a2 policy step), cold in L2",
            "anchors": n, "side_m": round(side, 1), "frames": len(hist), "scene_gen_s": round(gen_s, 1),
            "visible_mean": round(sum(h["n_visible"] for h in hist) / len(hist)),
            "misses_mean": round(sum(h["n_misses"] for h in hist) / len(hist)),
            "ms_per_frame": round(ms, 4), "algorithmic_bytes_per_frame": round(byts),
            "GBps": round(gbs, 1), "hbm_peak_GBps": peak, "frac": round(gbs / peak, 4),
            "l2_bytes": 126 * 2 ** 20}
    print(json.dumps(line))
    if out:
        with open(out, "w") as fh:
            fh.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(int(a[0]) if a else 18_000_000, int(a[1]) if len(a) > 1 else 60, a[2] if len(a) > 2 else None)
