"""B200-native GS-Cache per-frame hot path (arXiv 2502.14938).

The product is libgscache.so (hand-written CUDA for sm_100a behind the C ABI
of include/gscache.h).  This package is the thin Python binding: ``_abi``
(ctypes, same names as the C calls) and ``Renderer`` (torch used only for
device memory and streams).  No CPU fallback exists.
"""
from __future__ import annotations

import math

from . import _abi
from ._abi import (GSC_F_ABL_AABB_TILES, GSC_F_ABL_FIXED_EXTENT, GSC_F_COUNT_EVALS, GSC_F_DEPTH_LITERAL,
                   GSC_F_DERIVE_CUDA_CORES, GSC_F_GUIDE_EXP, GSC_F_MONO, GSC_F_STAGGER, GSC_F_BLEND_EXACT,
                   GSC_F_GUIDE_STAGED, GSC_F_SERIAL, GSC_F_STAGE_TIMING,
                   GSC_FMT_RGB_F32_PLANAR, GSC_FMT_RGBA8, GscError, gsc_frame_stats)

__all__ = ["Renderer", "GscError", "GSC_F_DEPTH_LITERAL", "GSC_F_STAGE_TIMING", "GSC_F_DERIVE_CUDA_CORES",
           "GSC_F_COUNT_EVALS", "GSC_F_SERIAL", "GSC_F_GUIDE_EXP", "GSC_F_GUIDE_STAGED", "GSC_F_ABL_FIXED_EXTENT",
           "GSC_F_ABL_AABB_TILES", "GSC_F_MONO", "GSC_F_STAGGER", "GSC_F_BLEND_EXACT", "PerEyeRenderer", "GSC_FMT_RGB_F32_PLANAR",
           "GSC_FMT_RGBA8", "build"]


def build(force: bool = False) -> str:
    from .build import build as _b
    return _b(force=force)


class Renderer:
    """One rendering worker with a private cache on one GPU."""

    def __init__(self, device: int = 0, width: int = 1920, height: int = 1080, fov_y_deg: float = 70.0,
                 near: float = 0.05, far: float = 5000.0, d_max: int = 10, bg=(0.0, 0.0, 0.0), flags: int = 0,
                 pair_capacity: int = 0):
        import ctypes as C
        self.device = device
        self.width, self.height = width, height
        cfg = _abi.gsc_config()
        cfg.width, cfg.height = width, height
        cfg.fov_y = math.radians(fov_y_deg)
        cfg.near_plane, cfg.far_plane = near, far
        for k in range(3):
            cfg.bg[k] = bg[k]
        cfg.d_max, cfg.flags, cfg.pair_capacity = d_max, flags, pair_capacity
        self._cfg = cfg
        h = C.c_void_p()
        _abi.check(None, _abi.lib().gsc_create(device, C.byref(cfg), C.byref(h)))
        self.h = h

    # -- lifecycle
    def close(self):
        if getattr(self, "h", None):
            _abi.lib().gsc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, st):
        _abi.check(self.h, st)

    # -- scene / pose
    def load(self, scene):
        """Load a scenegen.Scene (host arrays) or a GSC2 file path."""
        import ctypes as C
        if isinstance(scene, str):
            self._chk(_abi.lib().gsc_load_scene(self.h, scene.encode()))
        else:
            d = _abi.SceneDesc(scene)
            load = _abi.lib().gsc_load_scene_host_f32 if d.real else _abi.lib().gsc_load_scene_host
            self._chk(load(self.h, C.byref(d.desc)))
        return self

    def set_pose(self, rig):
        import ctypes as C
        r = _abi.make_rig(rig)
        self._chk(_abi.lib().gsc_set_pose(self.h, C.byref(r)))

    def reset_cache(self):
        self._chk(_abi.lib().gsc_reset_cache(self.h))

    def set_flags(self, flags: int):
        """Replace the GSC_F_* flags (DEPTH_LITERAL takes effect at the next reset_cache)."""
        self._chk(_abi.lib().gsc_set_flags(self.h, flags))

    # -- rendering
    def alloc_outputs(self, fmt: int = GSC_FMT_RGB_F32_PLANAR):
        import torch
        dev = torch.device("cuda", self.device)
        if fmt == GSC_FMT_RGB_F32_PLANAR:
            return (torch.empty((3, self.height, self.width), dtype=torch.float32, device=dev),
                    torch.empty((3, self.height, self.width), dtype=torch.float32, device=dev))
        return (torch.empty((self.height, self.width, 4), dtype=torch.uint8, device=dev),
                torch.empty((self.height, self.width, 4), dtype=torch.uint8, device=dev))

    def render_into(self, rig, out_l, out_r, fmt: int = GSC_FMT_RGB_F32_PLANAR, stream=None, sync_stats=False):
        """Enqueue one frame pair on ``stream`` (a torch.cuda.Stream or None = current)."""
        import ctypes as C
        import torch
        if rig is not None:
            self.set_pose(rig)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        st = _abi.gsc_frame_stats() if sync_stats else None
        self._chk(_abi.lib().gsc_render_pair(self.h, C.c_void_p(out_l.data_ptr()), C.c_void_p(out_r.data_ptr()),
                                             fmt, C.c_void_p(s.cuda_stream), C.byref(st) if st else None))
        return st

    def render(self, rig, fmt: int = GSC_FMT_RGB_F32_PLANAR):
        """Render one frame pair synchronously; returns (left, right, stats dict)."""
        out_l, out_r = self.alloc_outputs(fmt)
        st = self.render_into(rig, out_l, out_r, fmt, sync_stats=True)
        return out_l, out_r, st.as_dict()

    def render_host(self, rig, host_l, host_r, fmt: int = GSC_FMT_RGBA8):
        """End-to-end call: host pose in, images copied into host (pinned) tensors."""
        import ctypes as C
        r = _abi.make_rig(rig)
        self._chk(_abi.lib().gsc_render_pair_host(self.h, C.byref(r), C.c_void_p(host_l.data_ptr()),
                                                  C.c_void_p(host_r.data_ptr()), fmt, None))

    def render_host_async(self, rig, host_l, host_r, fmt: int = GSC_FMT_RGBA8) -> int:
        """Asynchronous end-to-end call: enqueue the frame and the copy of its images into host (pinned)
        tensors; returns the frame's sequence number for wait_frame.  Keep the tensors untouched until
        then (frame f's copy overlaps frame f+1's computation)."""
        import ctypes as C
        r = _abi.make_rig(rig)
        seq = C.c_longlong()
        self._chk(_abi.lib().gsc_render_pair_host_async(self.h, C.byref(r), C.c_void_p(host_l.data_ptr()),
                                                        C.c_void_p(host_r.data_ptr()), fmt, C.byref(seq)))
        return seq.value

    def wait_frame(self, seq: int):
        self._chk(_abi.lib().gsc_wait_frame(self.h, seq))

    def sync(self, stream=None):
        import ctypes as C
        self._chk(_abi.lib().gsc_sync(self.h, C.c_void_p(stream.cuda_stream if stream is not None else 0)))

    def stats_history(self, max_frames: int = 4096):
        import ctypes as C
        buf = (_abi.gsc_frame_stats * max_frames)()
        n = C.c_int()
        self._chk(_abi.lib().gsc_stats_history(self.h, buf, max_frames, C.byref(n)))
        return [buf[k].as_dict() for k in range(n.value)]

    # -- debug / parity
    def debug(self, what: str):
        import ctypes as C
        import numpy as np
        sel = _abi.DBG[what]
        n = C.c_size_t()
        self._chk(_abi.lib().gsc_debug_fetch(self.h, sel, None, 0, C.byref(n)))
        dt = {"visible": np.uint32, "misses": np.uint32, "pool": np.float32, "splats": np.float32,
              "splat_g": np.uint32, "pairs": np.uint64, "pair_g": np.uint32, "ranges": np.uint32,
              "birth": np.int32}[what]
        out = np.empty(n.value // np.dtype(dt).itemsize, dt)
        if n.value:
            self._chk(_abi.lib().gsc_debug_fetch(self.h, sel, out.ctypes.data, n.value, C.byref(n)))
        if what == "pool":
            out = out.reshape(-1, 13)
        elif what == "splats":
            out = out.reshape(-1, 13)
        elif what == "ranges":
            out = out.reshape(-1, 2)
        return out

    def elementary(self, fn: str, x):
        """Evaluate a device elementary function (exp/log/tanh/sigmoid, exp_blend = the blend's exact exp
        for x in [-87, 0], exp_fast = the blend's SFU exp ex2.approx(x log2e)) on a CUDA float32 tensor."""
        import ctypes as C
        import torch
        out = torch.empty_like(x)
        code = {"exp": 0, "log": 1, "tanh": 2, "sigmoid": 3, "exp_blend": 4, "exp_fast": 5}[fn]
        self._chk(_abi.lib().gsc_selftest_elementary(self.h, code, C.c_void_p(x.data_ptr()),
                                                     C.c_void_p(out.data_ptr()), x.numel()))
        return out


class PerEyeRenderer:
    """The no-de-redundancy ablation (the baseline of P:216-225): one monocular
    GS-Cache pipeline per eye -- its own cull, cache, derivation (through that eye's own viewpoint),
    projection, sort and blend -- instead of one unified cull + derivation shared by both eyes.  Each
    eye's context renders a rig whose two eyes coincide with that eye (GSC_F_MONO: left image only)."""

    def __init__(self, device: int, width: int, height: int, fov_y_deg: float = 70.0, near: float = 0.05,
                 far: float = 5000.0, d_max: int = 10, bg=(0.0, 0.0, 0.0), flags: int = 0, pair_capacity: int = 0):
        self.eyes = [Renderer(device, width, height, fov_y_deg, near, far, d_max, bg=bg, flags=flags | GSC_F_MONO,
                              pair_capacity=pair_capacity) for _ in range(2)]

    def load(self, scene):
        for r in self.eyes:
            r.load(scene)
        return self

    @staticmethod
    def _mono(rig, e):
        import dataclasses
        p, q = (rig.lp, rig.lq) if e == 0 else (rig.rp, rig.rq)
        return dataclasses.replace(rig, lp=p, lq=q, rp=p, rq=q)

    def render(self, rig, fmt: int = GSC_FMT_RGB_F32_PLANAR):
        """(left, right, [stats_left_pipeline, stats_right_pipeline])"""
        ol, _, sl = self.eyes[0].render(self._mono(rig, 0), fmt)
        orr, _, sr = self.eyes[1].render(self._mono(rig, 1), fmt)
        return ol, orr, [sl, sr]

