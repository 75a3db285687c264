"""ctypes binding of include/gscache.h -- argument marshalling only.

Every step of the frame path runs in libgscache.so (CUDA, sm_100a).  There is
no CPU or PyTorch fallback: if the library is missing, importing the binding
raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "libgscache.so")

GSC_OK, GSC_EINVAL, GSC_EFORMAT, GSC_EDEGENERATE, GSC_ENOMEM, GSC_ECUDA, GSC_EINTERNAL, GSC_ESTATE, GSC_ECAPACITY = range(9)
STATUS_NAMES = ["GSC_OK", "GSC_EINVAL", "GSC_EFORMAT", "GSC_EDEGENERATE", "GSC_ENOMEM", "GSC_ECUDA",
                "GSC_EINTERNAL", "GSC_ESTATE", "GSC_ECAPACITY"]
GSC_F_DEPTH_LITERAL = 0x1
GSC_F_STAGE_TIMING = 0x2
GSC_F_DERIVE_CUDA_CORES = 0x4
GSC_F_COUNT_EVALS = 0x8
GSC_F_SERIAL = 0x10
GSC_F_GUIDE_EXP = 0x20
GSC_F_GUIDE_STAGED = 0x40
GSC_F_ABL_FIXED_EXTENT = 0x80
GSC_F_ABL_AABB_TILES = 0x100
GSC_F_MONO = 0x200
GSC_F_STAGGER = 0x400
GSC_F_BLEND_EXACT = 0x800
GSC_FMT_RGB_F32_PLANAR = 0
GSC_FMT_RGBA8 = 1
DBG = {"visible": 1, "misses": 2, "pool": 3, "splats": 4, "splat_g": 5, "pairs": 6, "pair_g": 7, "ranges": 8,
       "birth": 9}


class gsc_config(C.Structure):
    _fields_ = [("width", C.c_int), ("height", C.c_int), ("fov_y", C.c_double), ("near_plane", C.c_double),
                ("far_plane", C.c_double), ("bg", C.c_float * 3), ("d_max", C.c_int), ("flags", C.c_uint),
                ("pair_capacity", C.c_int64)]


class gsc_eye(C.Structure):
    _fields_ = [("p", C.c_double * 3), ("q", C.c_double * 4)]


class gsc_rig(C.Structure):
    _fields_ = [("left", gsc_eye), ("right", gsc_eye), ("timestamp", C.c_double)]


class gsc_scene_desc(C.Structure):
    _fields_ = [("n_anchors", C.c_int32), ("lod_levels", C.c_int32), ("d0", C.c_float),
                ("pos", C.c_void_p), ("feat", C.c_void_p), ("offs", C.c_void_p), ("scale", C.c_void_p),
                ("level", C.c_void_p), ("W1", C.c_void_p), ("b1", C.c_void_p), ("W2a", C.c_void_p),
                ("b2a", C.c_void_p), ("W2c", C.c_void_p), ("b2c", C.c_void_p), ("W2s", C.c_void_p),
                ("b2s", C.c_void_p)]


class gsc_scene_desc_f32(C.Structure):
    _fields_ = [("n_anchors", C.c_int32), ("lod_levels", C.c_int32), ("d0", C.c_float),
                ("pos", C.c_void_p), ("feat", C.c_void_p), ("offs", C.c_void_p), ("scale", C.c_void_p),
                ("level", C.c_void_p), ("W1", C.c_void_p), ("b1", C.c_void_p), ("W2a", C.c_void_p),
                ("b2a", C.c_void_p), ("W2c", C.c_void_p), ("b2c", C.c_void_p), ("W2s", C.c_void_p),
                ("b2s", C.c_void_p), ("dist_input", C.c_int32), ("feature_bank", C.c_int32),
                ("Wb1", C.c_void_p), ("bb1", C.c_void_p), ("Wb2", C.c_void_p), ("bb2", C.c_void_p)]


class gsc_frame_stats(C.Structure):
    _fields_ = [("frame", C.c_int64), ("n_visible", C.c_uint32), ("n_hits", C.c_uint32),
                ("n_misses", C.c_uint32), ("n_new", C.c_uint32), ("n_splats", C.c_uint32),
                ("overflow", C.c_uint32), ("n_pairs", C.c_uint64), ("depth_used", C.c_int32),
                ("depth_next", C.c_int32), ("update_rate", C.c_float), ("novelty_rate", C.c_float),
                ("ms_cull", C.c_float), ("ms_derive", C.c_float), ("ms_project", C.c_float),
                ("ms_depth_sort", C.c_float), ("ms_emit", C.c_float), ("ms_tile_sort", C.c_float),
                ("ms_ranges", C.c_float), ("ms_blend", C.c_float), ("ms_total", C.c_float),
                ("n_evals", C.c_uint64), ("n_exp", C.c_uint64), ("n_nonfinite_skipped", C.c_uint32),
                ("n_blend_fixup", C.c_uint32), ("n_evals_list", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


# every symbol declared in include/gscache.h, with its ctypes signature
_SIGS = {
    "gsc_abi_version": (C.c_int, []),
    "gsc_create": (C.c_int, [C.c_int, C.POINTER(gsc_config), C.POINTER(C.c_void_p)]),
    "gsc_load_scene": (C.c_int, [C.c_void_p, C.c_char_p]),
    "gsc_load_scene_host": (C.c_int, [C.c_void_p, C.POINTER(gsc_scene_desc)]),
    "gsc_load_scene_host_f32": (C.c_int, [C.c_void_p, C.POINTER(gsc_scene_desc_f32)]),
    "gsc_set_pose": (C.c_int, [C.c_void_p, C.POINTER(gsc_rig)]),
    "gsc_render_pair": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                  C.POINTER(gsc_frame_stats)]),
    "gsc_render_pair_host": (C.c_int, [C.c_void_p, C.POINTER(gsc_rig), C.c_void_p, C.c_void_p, C.c_int,
                                       C.POINTER(gsc_frame_stats)]),
    "gsc_render_pair_host_async": (C.c_int, [C.c_void_p, C.POINTER(gsc_rig), C.c_void_p, C.c_void_p, C.c_int,
                                             C.POINTER(C.c_longlong)]),
    "gsc_wait_frame": (C.c_int, [C.c_void_p, C.c_longlong]),
    "gsc_sync": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gsc_stats_history": (C.c_int, [C.c_void_p, C.POINTER(gsc_frame_stats), C.c_int, C.POINTER(C.c_int)]),
    "gsc_reset_cache": (C.c_int, [C.c_void_p]),
    "gsc_set_flags": (C.c_int, [C.c_void_p, C.c_uint]),
    "gsc_debug_fetch": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "gsc_selftest_elementary": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_size_t]),
    "gsc_last_error": (C.c_char_p, [C.c_void_p]),
    "gsc_destroy": (None, [C.c_void_p]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise RuntimeError(f"libgscache.so not built ({SO_PATH}); run __graft_entry__.build()")
        L = C.CDLL(SO_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class GscError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")


def check(ctx, status):
    if status != GSC_OK:
        msg = lib().gsc_last_error(ctx).decode() if ctx else ""
        raise GscError(status, msg)


def make_rig(rig) -> gsc_rig:
    r = gsc_rig()
    for k in range(3):
        r.left.p[k] = float(rig.lp[k])
        r.right.p[k] = float(rig.rp[k])
    for k in range(4):
        r.left.q[k] = float(rig.lq[k])
        r.right.q[k] = float(rig.rq[k])
    r.timestamp = float(getattr(rig, "t", 0.0))
    return r


class SceneDesc:
    """Keeps the numpy arrays alive behind a gsc_scene_desc (borrowed by the call)."""

    def __init__(self, sc):
        self.keep = {}
        # grid scenes: int8 codes (gsc_scene_desc); real-weights scenes (F4): fp32 (gsc_scene_desc_f32)
        self.real = bool(getattr(sc, "real", False))
        q = np.float32 if self.real else np.int8
        d = gsc_scene_desc_f32() if self.real else gsc_scene_desc()
        d.n_anchors, d.lod_levels, d.d0 = sc.n, sc.L, sc.d0
        for name, dt in (("pos", np.float32), ("feat", q), ("offs", np.float32), ("scale", np.float32),
                         ("level", np.uint8), ("W1", q), ("b1", q), ("W2a", q), ("b2a", q),
                         ("W2c", q), ("b2c", q), ("W2s", q), ("b2s", q)):
            a = np.ascontiguousarray(getattr(sc, name), dtype=dt)
            self.keep[name] = a
            setattr(d, name, a.ctypes.data)
        if self.real:   # R32 combine inputs (distance input, feature bank)
            d.dist_input = int(bool(getattr(sc, "dist_input", False)))
            d.feature_bank = int(bool(getattr(sc, "bank", False)))
            if d.feature_bank:
                for name in ("Wb1", "bb1", "Wb2", "bb2"):
                    if getattr(sc, name) is None:   # (passed as NULL: the library rejects it)
                        continue
                    a = np.ascontiguousarray(getattr(sc, name), dtype=np.float32)
                    self.keep[name] = a
                    setattr(d, name, a.ctypes.data)
        self.desc = d
