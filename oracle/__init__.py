"""CPU ORACLE -- test infrastructure only.

Plain, slow, step-by-step C implementation (``orc.c``) of the GS-Cache
per-frame hot path as SURVEY.md §8(c) defines it, plus this ctypes binding.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  It shares no code
with ``paper_2502_14938_b200`` (the CUDA product path); both consume the
seeded inputs of ``scenegen``.

Parity status per function:
  exp_s/log_s/tanh_s/sigmoid_s  pinned (libm within ulp bounds, special values)
  unify (Eqs. 5-6)              pinned (S:300-302 examples, symmetry, coverage)
  cull + LoD                    pinned (fp64 brute force away from boundaries,
                                L=1, behind camera, optical-axis levels)
  cache state machine / H       pinned (S:219-248 examples, H endpoints,
                                closed-form integer H = float formula)
  derive                        pinned (fp64 numpy MLP, zero weights, Sigma
                                closed forms / det / symmetry, mu formula)
  project / extent / tiles      pinned (on-axis closed form, r(alpha) closed
                                forms, brute-force per-pixel tile sets; off-axis:
                                fp64 pinhole centres, finite-difference EWA
                                Jacobian inside/outside the clamp, fp64 single-
                                splat footprint, row-form kept set vs fp64 q_min
                                on every splat of C1/C3 frames --
                                tests/test_oracle_offaxis.py)
  sort                          pinned (numpy lexsort of the same pairs)
  blend                         pinned (empty, single splat, 13-splat stack,
                                T monotone, weight sum <= 1, O2 == O1)
  derive, real weights (F4)     pinned (fixed-order fp32 MLP: bit-exact against
                                the exact rational on grid-valued inputs, within
                                a derived bound of fp64 on real weights; epilogue
                                shared with the grid path)
  F4 combine inputs (R32)       pinned (one-hot logits reduce the bank to a
                                single stride, exactly; fp64 softmax / blend /
                                distance row within derived bounds; zero distance
                                row == no distance input -- test_oracle_bank.py)
  depth-schedule shape H        parity unpinned beyond "linear"
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liborc.so")
_SRC = [os.path.join(_HERE, "orc.c")]
_HDR = os.path.join(_HERE, "orc.h")

F, K, H = 32, 10, 32
NOUT = 11 * K


def build(force: bool = False) -> str:
    """Compile liborc.so (gcc, -ffp-contract=off -fno-fast-math, OpenMP)."""
    newest = max(os.path.getmtime(p) for p in _SRC + [_HDR])
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-fPIC", "-shared", "-o", _SO + ".tmp", *_SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_SO + ".tmp", _SO)
    return _SO


class Scene(C.Structure):
    _fields_ = [("N", C.c_int), ("L", C.c_int), ("d0", C.c_float),
                ("pos", C.c_void_p), ("feat", C.c_void_p), ("offs", C.c_void_p),
                ("scale", C.c_void_p), ("level", C.c_void_p),
                ("W1", C.c_void_p), ("b1", C.c_void_p), ("W2a", C.c_void_p), ("b2a", C.c_void_p),
                ("W2c", C.c_void_p), ("b2c", C.c_void_p), ("W2s", C.c_void_p), ("b2s", C.c_void_p),
                ("real", C.c_int), ("featf", C.c_void_p), ("W1f", C.c_void_p), ("b1f", C.c_void_p),
                ("W2af", C.c_void_p), ("b2af", C.c_void_p), ("W2cf", C.c_void_p), ("b2cf", C.c_void_p),
                ("W2sf", C.c_void_p), ("b2sf", C.c_void_p),
                ("dist_input", C.c_int), ("bank", C.c_int), ("Wb1", C.c_void_p), ("bb1", C.c_void_p),
                ("Wb2", C.c_void_p), ("bb2", C.c_void_p)]


class Config(C.Structure):
    _fields_ = [("width", C.c_int), ("height", C.c_int), ("fov_y", C.c_double),
                ("near_plane", C.c_double), ("far_plane", C.c_double), ("bg", C.c_float * 3),
                ("d_max", C.c_int), ("depth_literal", C.c_int), ("guide", C.c_int),
                ("ablate", C.c_int), ("stagger", C.c_int)]


class Eye(C.Structure):
    _fields_ = [("p", C.c_double * 3), ("q", C.c_double * 4)]


class EyeConsts(C.Structure):
    _fields_ = [("p", C.c_float * 3), ("r0", C.c_float * 3), ("r1", C.c_float * 3), ("r2", C.c_float * 3),
                ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("near_plane", C.c_float), ("far_plane", C.c_float), ("limx", C.c_float), ("limy", C.c_float)]


class Unified(C.Structure):
    _fields_ = [("p", C.c_float * 3), ("right", C.c_float * 3), ("up", C.c_float * 3), ("fwd", C.c_float * 3),
                ("near_plane", C.c_float), ("far_plane", C.c_float), ("tx", C.c_float), ("ty", C.c_float),
                ("kx", C.c_float), ("ky", C.c_float),
                ("p64", C.c_double * 3), ("fwd64", C.c_double * 3), ("up64", C.c_double * 3),
                ("pullback64", C.c_double)]


class Splat(C.Structure):
    _fields_ = [("u", C.c_float), ("v", C.c_float), ("A", C.c_float), ("B", C.c_float), ("C", C.c_float),
                ("alpha", C.c_float), ("rgb", C.c_float * 3), ("depth", C.c_float), ("thr", C.c_float),
                ("tx0", C.c_int), ("tx1", C.c_int), ("ty0", C.c_int), ("ty1", C.c_int), ("ntiles", C.c_int)]


class FrameStats(C.Structure):
    _fields_ = [("frame", C.c_int64), ("n_visible", C.c_int), ("n_hits", C.c_int), ("n_misses", C.c_int),
                ("n_new", C.c_int), ("n_live", C.c_int), ("depth_used", C.c_int), ("depth_next", C.c_int),
                ("n_splats", C.c_int64 * 2), ("n_pairs", C.c_int64 * 2), ("n_evals", C.c_int64),
                ("n_nonfinite", C.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        f32, i32, vp = C.c_float, C.c_int, C.c_void_p
        for name in ("orc_exp_s", "orc_log_s", "orc_tanh_s", "orc_sigmoid_s"):
            getattr(L, name).restype = f32
            getattr(L, name).argtypes = [f32]
        L.orc_elem_vec.argtypes = [i32, vp, vp, C.c_size_t]
        L.orc_eye_constants.argtypes = [C.POINTER(Config), C.POINTER(Eye), C.POINTER(EyeConsts)]
        L.orc_unify.argtypes = [C.POINTER(Config), C.POINTER(Eye), C.POINTER(Eye), C.POINTER(Unified)]
        L.orc_margin.restype = f32
        L.orc_margin.argtypes = [vp, vp]
        L.orc_lod_cut.argtypes = [C.POINTER(Unified), i32, f32, vp]
        L.orc_visible.argtypes = [C.POINTER(Unified), i32, f32, vp, f32, i32]
        L.orc_build_cov.argtypes = [vp, vp, vp]
        L.orc_build_cov.restype = None
        L.orc_derive_anchor.argtypes = [C.POINTER(Scene), i32, vp, vp, vp, vp, vp, vp]
        L.orc_mlp_f32.argtypes = [C.POINTER(Scene), vp, vp]
        L.orc_mlp_f32.restype = None
        L.orc_bank_weights.argtypes = [C.POINTER(Scene), vp, vp]
        L.orc_bank_weights.restype = None
        L.orc_bank_blend.argtypes = [vp, vp, vp]
        L.orc_bank_blend.restype = None
        L.orc_derive_anchor.restype = None
        L.orc_project.argtypes = [C.POINTER(Config), C.POINTER(EyeConsts), f32, vp, vp, vp, C.POINTER(Splat)]
        L.orc_tile_kept.argtypes = [C.POINTER(Config), C.POINTER(Splat), i32, i32]
        L.orc_tile_qmin.argtypes = [C.POINTER(Config), C.POINTER(Splat), i32, i32]
        L.orc_tile_qmin.restype = f32
        L.orc_blend_pixel.argtypes = [vp, i32, f32, f32, vp, vp, vp, vp]
        L.orc_blend_pixel.restype = None
        L.orc_depth_H.argtypes = [i32, C.c_int64, C.c_int64]
        L.orc_depth_H_guide.argtypes = [i32, i32, C.c_int64, C.c_int64]
        L.orc_create.restype = vp
        L.orc_create.argtypes = [C.POINTER(Scene), C.POINTER(Config)]
        L.orc_destroy.argtypes = [vp]
        L.orc_reset.argtypes = [vp]
        L.orc_frame.argtypes = [vp, C.POINTER(Eye), C.POINTER(Eye), C.c_uint, C.POINTER(FrameStats), vp, vp]
        L.orc_get_visible.argtypes = [vp, vp, i32]
        L.orc_get_misses.argtypes = [vp, vp, i32]
        L.orc_get_birth.argtypes = [vp, i32]
        L.orc_get_birth.restype = C.c_int32
        L.orc_get_pool.argtypes = [vp, C.c_int64, C.c_int64, vp, vp, vp, vp]
        L.orc_get_pool.restype = None
        L.orc_get_pairs.argtypes = [vp, vp, vp, C.c_int64]
        L.orc_get_pairs.restype = C.c_int64
        L.orc_get_splats.argtypes = [vp, i32, vp, vp, C.c_int64]
        L.orc_get_splats.restype = C.c_int64
        L.orc_num_threads.restype = i32
        L.orc_set_threads.argtypes = [i32]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------------------
# small helpers
# ---------------------------------------------------------------------------

def elem(fn: str, x) -> np.ndarray:
    x = np.ascontiguousarray(np.asarray(x, np.float32).ravel())
    out = np.empty_like(x)
    lib().orc_elem_vec({"exp": 0, "log": 1, "tanh": 2, "sigmoid": 3}[fn], _p(x), _p(out), x.size)
    return out


def make_config(width, height, fov_y_deg=70.0, near=0.05, far=5000.0, d_max=10, bg=(0, 0, 0),
                depth_literal=False, guide=0, ablate=0, stagger=False) -> Config:
    c = Config()
    c.width, c.height = width, height
    c.fov_y = np.deg2rad(fov_y_deg)
    c.near_plane, c.far_plane = near, far
    for k in range(3):
        c.bg[k] = bg[k]
    c.d_max = d_max
    c.depth_literal = int(depth_literal)
    c.guide = int(guide)       # 0 linear, 1 exponential, 2 staged (R23)
    c.ablate = int(ablate)     # ORC_ABL_* bits: 1 fixed 3-sigma extent, 2 AABB tiles (F1 ablations)
    c.stagger = int(bool(stagger))   # staggered expiry (F3, R26)
    return c


def make_eye(p, q) -> Eye:
    e = Eye()
    for k in range(3):
        e.p[k] = float(p[k])
    for k in range(4):
        e.q[k] = float(q[k])
    return e


def rig_eyes(rig):
    return make_eye(rig.lp, rig.lq), make_eye(rig.rp, rig.rq)


def unify(cfg: Config, left: Eye, right: Eye) -> Unified:
    u = Unified()
    rc = lib().orc_unify(C.byref(cfg), C.byref(left), C.byref(right), C.byref(u))
    if rc:
        raise ValueError(f"orc_unify failed ({rc})")
    return u


def eye_consts(cfg: Config, e: Eye) -> EyeConsts:
    ec = EyeConsts()
    if lib().orc_eye_constants(C.byref(cfg), C.byref(e), C.byref(ec)):
        raise ValueError("bad eye")
    return ec


class SceneHolder:
    """Keeps numpy arrays alive behind an ``orc_scene``."""

    def __init__(self, sc):
        self.arrays = {}
        s = Scene()
        s.N, s.L, s.d0 = sc.n, sc.L, sc.d0
        for name, dt in (("pos", np.float32), ("offs", np.float32), ("scale", np.float32), ("level", np.uint8)):
            a = np.ascontiguousarray(getattr(sc, name), dtype=dt)
            self.arrays[name] = a
            setattr(s, name, a.ctypes.data)
        real = bool(getattr(sc, "real", False))
        s.real = int(real)
        # grid scenes: int8 codes in feat, W1, ...; real-weights scenes (F4): fp32 values in featf, W1f, ...
        for name in ("feat", "W1", "b1", "W2a", "b2a", "W2c", "b2c", "W2s", "b2s"):
            a = np.ascontiguousarray(getattr(sc, name), dtype=np.float32 if real else np.int8)
            self.arrays[name] = a
            setattr(s, name + "f" if real else name, a.ctypes.data)
        # R32 combine inputs (real-weights scenes): distance input, feature bank
        s.dist_input = int(real and bool(getattr(sc, "dist_input", False)))
        s.bank = int(real and bool(getattr(sc, "bank", False)))
        if s.bank:
            for name in ("Wb1", "bb1", "Wb2", "bb2"):
                a = np.ascontiguousarray(getattr(sc, name), dtype=np.float32)
                self.arrays[name] = a
                setattr(s, name, a.ctypes.data)
        self.s = s


def derive_anchor(sh: SceneHolder, i: int, pu):
    pu = np.asarray(pu, np.float32)
    alpha = np.zeros(K, np.float32)
    mu = np.zeros((K, 3), np.float32)
    cov = np.zeros((K, 6), np.float32)
    rgb = np.zeros((K, 3), np.float32)
    o = np.zeros(NOUT, np.float32)
    lib().orc_derive_anchor(C.byref(sh.s), i, _p(pu), _p(alpha), _p(mu), _p(cov), _p(rgb), _p(o))
    return alpha, mu, cov, rgb, o


def mlp_f32(sh: SceneHolder, x) -> np.ndarray:
    """The real-weights path's fixed-order fp32 MLP (F4): x[35 + dist_input] -> o[110]."""
    x = np.ascontiguousarray(np.asarray(x, np.float32))
    assert x.shape == (F + 3 + sh.s.dist_input,)
    o = np.zeros(NOUT, np.float32)
    lib().orc_mlp_f32(C.byref(sh.s), _p(x), _p(o))
    return o


def bank_weights(sh: SceneHolder, y) -> np.ndarray:
    """R32 feature-bank softmax weights (strides 4, 2, 1) for y = (d_view, distance)."""
    y = np.ascontiguousarray(np.asarray(y, np.float32))
    w = np.zeros(3, np.float32)
    lib().orc_bank_weights(C.byref(sh.s), _p(y), _p(w))
    return w


def bank_blend(f, w) -> np.ndarray:
    """R32 blended features fh[k] = fma(w2, f_k, fma(w1, f_{2 (k mod F/2)}, w0 f_{4 (k mod F/4)}))."""
    f = np.ascontiguousarray(np.asarray(f, np.float32))
    w = np.ascontiguousarray(np.asarray(w, np.float32))
    fh = np.zeros(F, np.float32)
    lib().orc_bank_blend(_p(f), _p(w), _p(fh))
    return fh


def project(cfg: Config, ec: EyeConsts, alpha, mu, cov, rgb):
    s = Splat()
    mu = np.asarray(mu, np.float32)
    cov = np.asarray(cov, np.float32)
    rgb = np.asarray(rgb, np.float32)
    ok = lib().orc_project(C.byref(cfg), C.byref(ec), float(alpha), _p(mu), _p(cov), _p(rgb), C.byref(s))
    return (s if ok > 0 else None)


@dataclass
class FrameResult:
    stats: FrameStats
    img_l: np.ndarray | None
    img_r: np.ndarray | None


class Oracle:
    """The cache state machine + renderer of one worker (private cache)."""

    RASTER = 1
    BRUTE = 2

    def __init__(self, scene, cfg: Config):
        self.sh = SceneHolder(scene)
        self.cfg = cfg
        self.h = lib().orc_create(C.byref(self.sh.s), C.byref(cfg))
        if not self.h:
            raise ValueError("orc_create failed")

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            lib().orc_destroy(h)
            self.h = None

    def reset(self):
        lib().orc_reset(self.h)

    def frame(self, rig, raster=True, brute=False, images=True) -> FrameResult:
        el, er = rig_eyes(rig)
        st = FrameStats()
        W, Hh = self.cfg.width, self.cfg.height
        il = ir = None
        if raster and images:
            il = np.zeros((3, Hh, W), np.float32)
            ir = np.zeros((3, Hh, W), np.float32)
        flags = (self.RASTER if raster else 0) | (self.BRUTE if brute else 0)
        rc = lib().orc_frame(self.h, C.byref(el), C.byref(er), flags, C.byref(st),
                             _p(il) if il is not None else None, _p(ir) if ir is not None else None)
        if rc:
            raise ValueError(f"orc_frame failed ({rc})")
        return FrameResult(st, il, ir)

    def visible(self) -> np.ndarray:
        n = lib().orc_get_visible(self.h, None, 0)
        out = np.zeros(n, np.uint32)
        lib().orc_get_visible(self.h, _p(out), n)
        return out

    def misses(self) -> np.ndarray:
        n = lib().orc_get_misses(self.h, None, 0)
        out = np.zeros(n, np.uint32)
        lib().orc_get_misses(self.h, _p(out), n)
        return out

    def birth(self, i: int) -> int:
        return lib().orc_get_birth(self.h, i)

    def pool(self, slot0: int, count: int):
        a = np.zeros(count, np.float32)
        mu = np.zeros((count, 3), np.float32)
        cov = np.zeros((count, 6), np.float32)
        rgb = np.zeros((count, 3), np.float32)
        lib().orc_get_pool(self.h, slot0, count, _p(a), _p(mu), _p(cov), _p(rgb))
        return a, mu, cov, rgb

    def pairs(self):
        n = lib().orc_get_pairs(self.h, None, None, 0)
        keys = np.zeros(n, np.uint64)
        gs = np.zeros(n, np.uint32)
        lib().orc_get_pairs(self.h, _p(keys), _p(gs), n)
        return keys, gs

    def splats(self, eye: int):
        n = lib().orc_get_splats(self.h, eye, None, None, 0)
        gs = np.zeros(n, np.uint32)
        rec = np.zeros((n, 12), np.float32)
        lib().orc_get_splats(self.h, eye, _p(gs), _p(rec), n)
        return gs, rec


def num_threads() -> int:
    return lib().orc_num_threads()


def set_threads(n: int) -> None:
    lib().orc_set_threads(n)
