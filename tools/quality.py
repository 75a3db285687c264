#!/usr/bin/env python
"""Quality / speed harness for SURVEY §8(f) F1 (the methodology of the paper's Tables 4-6 on the
synthetic scenes): render a trajectory with the method and with its variants, and compare every
frame with the uncached reference (D_max = 1: every visible anchor derived at the current view,
S:260) by MSE / PSNR / SSIM, plus average and 99% FPS of each variant.

Variants: method (linear H, D_max from the config), no reuse (D_max = 1, the reference itself),
exponential / staged guiding functions (R23), fixed 3-sigma extent and AABB tiles.

  PYTHONPATH=. python tools/quality.py [config] [frames] [out.json] [variant,variant,...]

The metrics are measurement code (torch ops on the rendered images), not part of the hot path.
"""
import json
import sys

import numpy as np


def _gauss_window(torch, size=11, sigma=1.5, device=None):
    x = torch.arange(size, dtype=torch.float64, device=device) - (size - 1) / 2.0
    g = torch.exp(-(x * x) / (2 * sigma * sigma))
    g = g / g.sum()
    return (g[:, None] * g[None, :]).to(torch.float32)


def mse(a, b) -> float:
    """Mean squared error of two images with values in [0, 1]."""
    return float(((a.double() - b.double()) ** 2).mean())


def psnr(a, b) -> float:
    """10 log10(1 / MSE) for images in [0, 1]; inf when identical."""
    m = mse(a, b)
    return float("inf") if m == 0 else 10.0 * float(np.log10(1.0 / m))


def ssim(a, b) -> float:
    """Mean SSIM (Wang et al. 2004: 11x11 Gaussian window, sigma 1.5, K1 = 0.01, K2 = 0.03, L = 1)
    over the channels of (C, H, W) images in [0, 1]; 'valid' windows only."""
    import torch
    import torch.nn.functional as F
    C = a.shape[0]
    w = _gauss_window(torch, device=a.device).expand(C, 1, 11, 11).contiguous()
    x = a[None].float()
    y = b[None].float()
    mu_x = F.conv2d(x, w, groups=C)
    mu_y = F.conv2d(y, w, groups=C)
    sxx = F.conv2d(x * x, w, groups=C) - mu_x * mu_x
    syy = F.conv2d(y * y, w, groups=C) - mu_y * mu_y
    sxy = F.conv2d(x * y, w, groups=C) - mu_x * mu_y
    c1, c2 = 0.01 ** 2, 0.03 ** 2
    s = ((2 * mu_x * mu_y + c1) * (2 * sxy + c2)) / ((mu_x * mu_x + mu_y * mu_y + c1) * (sxx + syy + c2))
    return float(s.mean())


def run(config="C3", frames=150, only=None):
    import torch
    import scenegen as sg
    import paper_2502_14938_b200 as gp
    cfg = sg.config(config)
    sc = cfg.scene()
    traj = sg.trajectory(cfg)[:frames]
    variants = {
        "method": (cfg.d_max, 0),
        "guide_exponential": (cfg.d_max, gp.GSC_F_GUIDE_EXP),
        "guide_staged": (cfg.d_max, gp.GSC_F_GUIDE_STAGED),
        "stagger": (cfg.d_max, gp.GSC_F_STAGGER),         # staggered expiry (F3, R26)
        "abl_fixed_extent": (cfg.d_max, gp.GSC_F_ABL_FIXED_EXTENT),
        "abl_aabb_tiles": (cfg.d_max, gp.GSC_F_ABL_AABB_TILES),
        "no_reuse": (1, 0),
        "no_dered": (cfg.d_max, "per_eye"),      # one monocular pipeline per eye (F1)
    }
    if only:
        variants = {k: v for k, v in variants.items() if k in only}
    # reference images: uncached (D_max = 1), opacity-aware extent, exact tiles
    ref_r = gp.Renderer(0, cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far, 1).load(sc)
    refs = []
    for rig in traj:
        gl, gr, _ = ref_r.render(rig)
        refs.append((gl, gr))
    del ref_r
    out = {"config": config, "frames": len(traj), "reference": "uncached (D_max = 1) render of every frame",
           "variants": {}}
    for name, (dmax, flags) in variants.items():
        per_eye = flags == "per_eye"
        flags = 0 if per_eye else flags
        # (AABB tiles need more pair capacity than the default 4 N K)
        cap = max(3 << 24, 12 * sc.n * 10) if flags & gp.GSC_F_ABL_AABB_TILES else 0
        R = gp.PerEyeRenderer if per_eye else gp.Renderer
        r = R(0, cfg.width, cfg.height, cfg.fov_y_deg, cfg.near, cfg.far, dmax,
              flags=flags | gp.GSC_F_STAGE_TIMING | gp.GSC_F_SERIAL, pair_capacity=cap).load(sc)
        ps, ss, ms_, misses, pairs, depth, novelty = [], [], [], [], [], [], []
        for (rig, (rl, rr)) in zip(traj, refs):
            gl, gr, st = r.render(rig)
            p = min(psnr(gl, rl), psnr(gr, rr))
            ps.append(p if np.isfinite(p) else 99.0)
            ss.append(0.5 * (ssim(gl, rl) + ssim(gr, rr)))
            sts = st if isinstance(st, list) else [st]
            misses.append(sum(x["n_misses"] for x in sts) / max(1, sum(x["n_visible"] for x in sts)))
            pairs.append(sum(x["n_pairs"] for x in sts))
            depth.append(sts[0]["depth_next"])
            novelty.append(sts[0]["novelty_rate"])
            ms_.append(sum(x["ms_total"] for x in sts))
        ms_ = np.array(ms_)
        out["variants"][name] = {
            "d_max": dmax, "flags": "per-eye pipelines" if per_eye else flags,
            "psnr_mean_db": round(float(np.mean(ps)), 3), "psnr_min_db": round(float(np.min(ps)), 3),
            "ssim_mean": round(float(np.mean(ss)), 6), "ssim_min": round(float(np.min(ss)), 6),
            "update_rate_mean": round(float(np.mean(misses)), 4), "pairs_mean": round(float(np.mean(pairs))),
            "fps_avg": round(float(1000.0 / np.mean(ms_)), 2) if len(ms_) else None,
            "fps_99pct": round(float(1000.0 / np.percentile(ms_, 99)), 2) if len(ms_) else None,
            # per-frame traces (cache depth and update rate along the trajectory)
            "trace": {"depth_next": [int(d) for d in depth], "update_rate": [round(float(m), 4) for m in misses],
                      "novelty_rate": [round(float(n), 4) for n in novelty],
                      "psnr_db": [round(float(p), 2) for p in ps], "ms": [round(float(m), 4) for m in ms_]},
        }
        print(name, json.dumps({k: v for k, v in out["variants"][name].items() if k != "trace"}), flush=True)
        del r
        torch.cuda.empty_cache()
    return out


def main():
    config = sys.argv[1] if len(sys.argv) > 1 else "C3"
    frames = int(sys.argv[2]) if len(sys.argv) > 2 else 150
    only = sys.argv[4].split(",") if len(sys.argv) > 4 else None
    res = run(config, frames, only)
    if len(sys.argv) > 3:
        with open(sys.argv[3], "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
