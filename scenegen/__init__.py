"""Seeded synthetic inputs shared by the CPU oracle and the CUDA path.

This module is INPUT GENERATION ONLY: it draws anchors, decoder weight codes
and camera rigs from a counter-based SplitMix64 stream and writes/reads the
GSC2 scene file and the JSON-lines trajectory file.  It holds none of the
method's arithmetic (no culling, LoD, derivation, projection, sorting or
blending); both the oracle (``oracle/``) and the product
(``paper_2502_14938_b200``) consume its outputs and nothing else of each other.

Workload recipe:
  * city block of side A, ground plane z = 0, world z up;
  * building grid (40 m blocks / 12 m streets, scaled for tiny scenes),
    heights lognormal (median 25 m, sigma_ln 0.6, clipped to [6, 150] m);
  * anchors sampled on ground, facades and roofs in proportion to area;
    L levels with counts proportional to 4^level (Octree-GS-like);
    positions snapped to the level's voxel centre (v_l = v_fine * 2^(L-1-l))
    plus jitter; v_fine = sqrt(1.33 * surface_area / N);
  * anchor scale s_i = v_level * loguniform(0.5, 1.5) per axis,
    offsets O_ij ~ U[-1, 1]^3 (K = 10 per anchor);
  * feature codes ~ U{-127..127} (value = code / 128, F = 32);
  * decoder weight codes Kaiming-uniform on the 2^-7 grid (W1 +-21, W2 +-22),
    the opacity head's layer-2 codes widened to +-64 so opacities spread over
    (0, ~0.7) as in trained scenes;
  * d0 = f_px * v_fine (finest voxel ~1 px at d0);
  * orbit trajectories per SPEC S:74-82: look at the block centre, eyes
    +-ipd/2 along the local horizontal, ipd 0.064 m, fov_y 70 deg.
"""
from __future__ import annotations

import json
import math
import struct
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "splitmix64", "uniform01", "Scene", "Rig", "make_city_scene",
    "make_orbit", "make_pan", "look_at_rig", "write_gsc2", "read_gsc2", "with_real_weights",
    "write_trajectory", "read_trajectory", "config", "CONFIGS",
    "F_DIM", "K_GAUSS", "H_DIM",
]

F_DIM = 32      # anchor feature dimension
K_GAUSS = 10    # neural Gaussians per anchor
H_DIM = 32      # hidden width of each MLP head

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """Counter-based SplitMix64: output for counter ``idx`` of ``stream``.

    state = seed_key + (idx + 1) * golden; then the SplitMix64 finaliser.
    The seed key mixes (seed, stream) with the same finaliser so streams are
    independent.
    """
    with np.errstate(over="ignore"):
        key = np.uint64((seed * 0x100000001B3 + stream * 0x9E3779B1 + 0x632BE59BD9B4E019)
                        & 0xFFFFFFFFFFFFFFFF)
        z = key + (np.asarray(idx, dtype=np.uint64) + np.uint64(1)) * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform01(seed: int, stream: int, n: int) -> np.ndarray:
    """n doubles in [0, 1) with 53 random bits: (z >> 11) * 2^-53."""
    z = splitmix64(seed, stream, np.arange(n, dtype=np.uint64))
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def _int_codes(seed: int, stream: int, n: int, bound: int) -> np.ndarray:
    """n integers uniform in [-bound, bound] (int8 codes)."""
    z = splitmix64(seed, stream, np.arange(n, dtype=np.uint64))
    return ((z % np.uint64(2 * bound + 1)).astype(np.int64) - bound).astype(np.int8)


@dataclass
class Scene:
    """A GSC2 scene: anchor SoA plus the three-head decoder weight codes."""
    pos: np.ndarray        # f32 [N,3]
    feat: np.ndarray       # i8  [N,F]   value = code/128
    offs: np.ndarray       # f32 [N,K,3]
    scale: np.ndarray      # f32 [N,3]
    level: np.ndarray      # u8  [N]
    W1: np.ndarray         # i8  [F+3, 3H]  columns: alpha 0..H-1, colour H..2H-1, cov 2H..3H-1
    b1: np.ndarray         # i8  [3H]
    W2a: np.ndarray        # i8  [H, K]
    b2a: np.ndarray        # i8  [K]
    W2c: np.ndarray        # i8  [H, 3K]
    b2c: np.ndarray        # i8  [3K]
    W2s: np.ndarray        # i8  [H, 7K]   per Gaussian j: 3 raw scales, 4 raw quaternion (w,x,y,z)
    b2s: np.ndarray        # i8  [7K]
    L: int
    d0: float
    bbox: np.ndarray = field(default_factory=lambda: np.zeros(6, np.float32))
    # real-weights scene: feat and the decoder weights are fp32 values, not int8 codes
    real: bool = False
    # F4 Scaffold-GS combine inputs (R32; real-weights scenes only): the anchor-camera distance
    # as a 36th MLP input (W1 then has F + 4 rows), and the multi-resolution feature bank -- weights
    # w = softmax(Wb2^T ReLU(Wb1^T (d_view, dist) + bb1) + bb2) blending the features at strides 4, 2, 1
    dist_input: bool = False
    bank: bool = False
    Wb1: np.ndarray = None   # f32 [4, F]
    bb1: np.ndarray = None   # f32 [F]
    Wb2: np.ndarray = None   # f32 [F, 3]
    bb2: np.ndarray = None   # f32 [3]

    @property
    def n(self) -> int:
        return int(self.pos.shape[0])


@dataclass
class Rig:
    """Binocular rig (StereoRig S:46-49): world-from-camera quaternions (w,x,y,z)."""
    lp: np.ndarray  # f64[3]
    lq: np.ndarray  # f64[4]
    rp: np.ndarray
    rq: np.ndarray
    t: float = 0.0


# ----------------------------------------------------------------------------
# city scene
# ----------------------------------------------------------------------------

def _buildings(seed: int, side: float):
    nb = max(1, int(round(side / 52.0)))
    period = side / nb
    bsize = period * (40.0 / 52.0)
    street = period - bsize
    u = uniform01(seed, 101, 2 * nb * nb)
    # lognormal heights via Box-Muller on the SplitMix stream
    u1 = np.maximum(u[0::2], 1e-300)
    u2 = u[1::2]
    g = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)
    h = np.clip(25.0 * np.exp(0.6 * g), 6.0, 150.0)
    ix, iy = np.meshgrid(np.arange(nb), np.arange(nb), indexing="ij")
    x0 = ix.ravel() * period + street * 0.5
    y0 = iy.ravel() * period + street * 0.5
    return x0, y0, bsize, h


def make_city_scene(seed: int, n: int, side: float, L: int = 5, width: int = 1920,
                    height: int = 1080, fov_y_deg: float = 70.0) -> Scene:
    """Octree-shaped synthetic city (DESIGN.md input recipe)."""
    if n < 1 or L < 1 or side <= 0:
        raise ValueError("n >= 1, L >= 1 and side > 0 required")
    K, F, H = K_GAUSS, F_DIM, H_DIM
    x0, y0, bs, bh = _buildings(seed, side)
    nbld = len(bh)
    ground_area = side * side - nbld * bs * bs
    roof_area = nbld * bs * bs
    facade_areas = 4.0 * bs * bh
    total_area = ground_area + roof_area + facade_areas.sum()
    v_fine = math.sqrt(1.33 * total_area / n)

    # level counts proportional to 4^l, finest level absorbs the remainder
    w = 4.0 ** np.arange(L)
    counts = np.floor(n * w / w.sum()).astype(np.int64)
    counts[-1] += n - counts.sum()
    level = np.repeat(np.arange(L, dtype=np.uint8), counts)

    # surface choice: 0 ground, 1 roof, 2 facade (building b, face f)
    u = uniform01(seed, 1, 6 * n).reshape(n, 6)
    p_ground = ground_area / total_area
    p_roof = roof_area / total_area
    kind = np.where(u[:, 0] < p_ground, 0, np.where(u[:, 0] < p_ground + p_roof, 1, 2))
    pos = np.zeros((n, 3), np.float64)
    # ground: rejection-free approximation -- sample the whole square, points
    # falling inside a footprint are lifted onto that roof (kept as ground level z=0
    # otherwise); this keeps the density per area uniform enough for a workload.
    g = kind == 0
    pos[g, 0] = u[g, 1] * side
    pos[g, 1] = u[g, 2] * side
    # roofs
    r = kind == 1
    b = np.minimum((u[r, 3] * nbld).astype(np.int64), nbld - 1)
    pos[r, 0] = x0[b] + u[r, 1] * bs
    pos[r, 1] = y0[b] + u[r, 2] * bs
    pos[r, 2] = bh[b]
    # facades: building chosen proportional to its facade area
    f = kind == 2
    cdf = np.cumsum(facade_areas) / facade_areas.sum()
    b = np.minimum(np.searchsorted(cdf, u[f, 3], side="right"), nbld - 1)
    face = np.minimum((u[f, 4] * 4).astype(np.int64), 3)
    t = u[f, 1] * bs
    zz = u[f, 2] * bh[b]
    fx = np.where(face == 0, x0[b] + t, np.where(face == 1, x0[b] + bs, np.where(face == 2, x0[b] + t, x0[b])))
    fy = np.where(face == 0, y0[b], np.where(face == 1, y0[b] + t, np.where(face == 2, y0[b] + bs, y0[b] + t)))
    pos[f, 0] = fx
    pos[f, 1] = fy
    pos[f, 2] = zz

    # snap to the level voxel centre, plus jitter of +-0.25 voxel
    vl = v_fine * (2.0 ** (L - 1 - level.astype(np.float64)))
    jit = uniform01(seed, 2, 3 * n).reshape(n, 3) - 0.5
    pos = (np.floor(pos / vl[:, None]) + 0.5 + 0.5 * jit) * vl[:, None]

    # spatially coherent id order inside each level (voxel-cell lexicographic)
    cell = np.floor(pos / (8.0 * v_fine)).astype(np.int64)
    order = np.lexsort((cell[:, 2], cell[:, 1], cell[:, 0], level))
    pos = pos[order]
    level = level[order]
    vl = vl[order]

    us = uniform01(seed, 3, 3 * n).reshape(n, 3)
    scale = vl[:, None] * np.exp(math.log(0.5) + us * (math.log(1.5) - math.log(0.5)))
    offs = uniform01(seed, 4, 3 * K * n).reshape(n, K, 3) * 2.0 - 1.0
    feat = _int_codes(seed, 5, n * F, 127).reshape(n, F)

    W1 = _int_codes(seed, 10, (F + 3) * 3 * H, 21).reshape(F + 3, 3 * H)
    b1 = _int_codes(seed, 11, 3 * H, 21)
    W2a = _int_codes(seed, 12, H * K, 64).reshape(H, K)
    b2a = _int_codes(seed, 13, K, 22)
    W2c = _int_codes(seed, 14, H * 3 * K, 22).reshape(H, 3 * K)
    b2c = _int_codes(seed, 15, 3 * K, 22)
    W2s = _int_codes(seed, 16, H * 7 * K, 22).reshape(H, 7 * K)
    b2s = _int_codes(seed, 17, 7 * K, 22)

    f_px = (height / 2.0) / math.tan(math.radians(fov_y_deg) / 2.0)
    d0 = f_px * v_fine
    pos32 = pos.astype(np.float32)
    bbox = np.concatenate([pos32.min(0), pos32.max(0)]).astype(np.float32)
    return Scene(pos=pos32, feat=feat, offs=offs.astype(np.float32),
                 scale=scale.astype(np.float32), level=level.astype(np.uint8),
                 W1=W1, b1=b1, W2a=W2a, b2a=b2a, W2c=W2c, b2c=b2c, W2s=W2s, b2s=b2s,
                 L=L, d0=float(np.float32(d0)), bbox=bbox)


def with_real_weights(scene: Scene, seed: int = 11, dist: bool = False, bank: bool = False) -> Scene:
    """F4 input: the same anchors with trained-style fp32 features and decoder
    weights -- continuous values, not on the 2^-7 grid.  Features U(-1, 1); each weight and bias
    uniform in +-(the grid scene's Kaiming code bound)/128 (W1, b1: 21; W2a: 64; b2a and the colour /
    covariance heads: 22), so activations and opacities spread like the grid scene's.

    dist / bank (R32, Scaffold-GS combine inputs): W1 gains a distance row, U(+-2^-9) per metre so a few
    hundred metres move a hidden unit by ~0.5; the feature-bank MLP 4 -> F -> 3 has Wb1 U(+-1) on the
    view direction and U(+-2^-7) on the distance, bb1 U(+-0.25), Wb2 U(+-0.5), bb2 U(+-1): softmax
    weights that vary with the view, none degenerate."""
    import dataclasses
    n, F, K, H = scene.n, F_DIM, K_GAUSS, H_DIM

    def U(stream, shape, bound):
        cnt = int(np.prod(shape))
        return ((uniform01(seed, stream, cnt) * 2.0 - 1.0) * (bound / 128.0)).astype(np.float32).reshape(shape)

    W1 = U(31, (F + 3, 3 * H), 21)
    extra = {}
    if dist:
        W1 = np.concatenate([W1, U(39, (1, 3 * H), 0.25)], axis=0)
    if bank:
        Wb1 = np.concatenate([U(40, (3, F), 128.0), U(41, (1, F), 1.0)], axis=0)
        extra = dict(Wb1=Wb1, bb1=U(42, (F,), 32.0), Wb2=U(43, (F, 3), 64.0), bb2=U(44, (3,), 128.0))
    return dataclasses.replace(
        scene, feat=U(30, (n, F), 128.0), W1=W1, b1=U(32, (3 * H,), 21),
        W2a=U(33, (H, K), 64), b2a=U(34, (K,), 22), W2c=U(35, (H, 3 * K), 22), b2c=U(36, (3 * K,), 22),
        W2s=U(37, (H, 7 * K), 22), b2s=U(38, (7 * K,), 22), real=True, dist_input=dist, bank=bank, **extra)


# ----------------------------------------------------------------------------
# cameras
# ----------------------------------------------------------------------------

def _quat_from_matrix(R: np.ndarray) -> np.ndarray:
    """Unit quaternion (w,x,y,z), w >= 0, of a rotation matrix (Shepperd)."""
    tr = R[0, 0] + R[1, 1] + R[2, 2]
    if tr > 0:
        s = math.sqrt(tr + 1.0) * 2
        q = [0.25 * s, (R[2, 1] - R[1, 2]) / s, (R[0, 2] - R[2, 0]) / s, (R[1, 0] - R[0, 1]) / s]
    elif R[0, 0] > R[1, 1] and R[0, 0] > R[2, 2]:
        s = math.sqrt(1.0 + R[0, 0] - R[1, 1] - R[2, 2]) * 2
        q = [(R[2, 1] - R[1, 2]) / s, 0.25 * s, (R[0, 1] + R[1, 0]) / s, (R[0, 2] + R[2, 0]) / s]
    elif R[1, 1] > R[2, 2]:
        s = math.sqrt(1.0 + R[1, 1] - R[0, 0] - R[2, 2]) * 2
        q = [(R[0, 2] - R[2, 0]) / s, (R[0, 1] + R[1, 0]) / s, 0.25 * s, (R[1, 2] + R[2, 1]) / s]
    else:
        s = math.sqrt(1.0 + R[2, 2] - R[0, 0] - R[1, 1]) * 2
        q = [(R[1, 0] - R[0, 1]) / s, (R[0, 2] + R[2, 0]) / s, (R[1, 2] + R[2, 1]) / s, 0.25 * s]
    q = np.array(q, np.float64)
    q /= np.linalg.norm(q)
    if q[0] < 0:
        q = -q
    return q


def look_at_rig(eye: np.ndarray, target: np.ndarray, ipd: float, t: float = 0.0) -> Rig:
    """Parallel binocular rig centred at ``eye`` looking at ``target``.

    Camera frame: columns of R are (right, up, back); forward = -Z.
    Eyes sit at eye -+ right * ipd/2.
    """
    eye = np.asarray(eye, np.float64)
    fwd = np.asarray(target, np.float64) - eye
    fwd /= np.linalg.norm(fwd)
    zup = np.array([0.0, 0.0, 1.0])
    right = np.cross(fwd, zup)
    if np.linalg.norm(right) < 1e-9:
        right = np.array([1.0, 0.0, 0.0])
    right /= np.linalg.norm(right)
    up = np.cross(right, fwd)
    R = np.stack([right, up, -fwd], axis=1)
    q = _quat_from_matrix(R)
    return Rig(lp=eye - right * (ipd / 2), lq=q.copy(), rp=eye + right * (ipd / 2), rq=q.copy(), t=t)


def make_orbit(center, radius0: float, radius1: float, h0: float, h1: float,
               n_frames: int, deg_per_frame: float, ipd: float = 0.064,
               az0_deg: float = 0.0, fps: float = 90.0):
    """Ground-to-aerial orbit: look at ``center``; radius and
    height interpolate linearly over the trajectory; azimuth advances
    ``deg_per_frame`` per frame."""
    if n_frames < 1:
        raise ValueError("n_frames >= 1")
    c = np.asarray(center, np.float64)
    rigs = []
    for f in range(n_frames):
        a = f / max(1, n_frames - 1)
        r = radius0 + (radius1 - radius0) * a
        h = h0 + (h1 - h0) * a
        az = math.radians(az0_deg + deg_per_frame * f)
        eye = np.array([c[0] + r * math.cos(az), c[1] + r * math.sin(az), h])
        rigs.append(look_at_rig(eye, c, ipd, t=f / fps))
    return rigs


def make_pan(eye0, eye1, yaw0_deg: float, steps_deg, pitch_deg: float = -5.0, ipd: float = 0.064,
             fps: float = 90.0):
    """Head-turn trajectory for the F3 depth-policy study ("movement with acceleration and with
    staged speed changes"): the eye moves linearly from eye0 to eye1 while the view direction turns
    about the vertical by steps_deg[f] degrees at frame f (yaw speed profile), pitched by pitch_deg."""
    e0, e1 = np.asarray(eye0, np.float64), np.asarray(eye1, np.float64)
    n = len(steps_deg)
    rigs = []
    yaw = math.radians(yaw0_deg)
    pitch = math.radians(pitch_deg)
    for f in range(n):
        if f:
            yaw += math.radians(steps_deg[f])
        a = f / max(1, n - 1)
        eye = e0 + (e1 - e0) * a
        d = np.array([math.cos(yaw) * math.cos(pitch), math.sin(yaw) * math.cos(pitch), math.sin(pitch)])
        rigs.append(look_at_rig(eye, eye + d, ipd, t=f / fps))
    return rigs


# ----------------------------------------------------------------------------
# files
# ----------------------------------------------------------------------------

_HDR = struct.Struct("<4sIIIIIIf6f")  # magic, version, N, F, K, L, H, d0, bbox


def write_gsc2(scene: Scene, path: str) -> None:
    """GSC2: GSC1 as SoA with int8 grid codes and the three-head weights.

    header  : "GSC2" u32 version, u32 N, u32 F, u32 K, u32 L, u32 H, f32 d0, f32 bbox[6]
    arrays  : pos f32[N*3] | feat q[N*F] | offs f32[N*K*3] | scale f32[N*3] | level u8[N]
    weights : W1 q[(F+3)*3H] | b1 q[3H] | W2a q[H*K] | b2a q[K] | W2c q[H*3K] |
              b2c q[3K] | W2s q[H*7K] | b2s q[7K]
    version 2: q = i8 grid codes (value = code / 128); version 3 (real-weights scenes, F4): q = f32.
    version 4 (real weights with the R32 combine inputs): after the header a u32 flags word (bit 0:
    distance input, W1 then has F+4 rows; bit 1: feature bank), and after b2s, with the bank:
    Wb1 f32[4*F] | bb1 f32[F] | Wb2 f32[F*3] | bb2 f32[3].
    """
    q = "<f4" if scene.real else "i1"
    v4 = scene.real and (scene.dist_input or scene.bank)
    with open(path, "wb") as fh:
        fh.write(_HDR.pack(b"GSC2", 4 if v4 else (3 if scene.real else 2), scene.n, F_DIM, K_GAUSS, scene.L,
                           H_DIM, scene.d0, *[float(x) for x in scene.bbox]))
        if v4:
            fh.write(struct.pack("<I", (1 if scene.dist_input else 0) | (2 if scene.bank else 0)))
        arrays = [(scene.pos, "<f4"), (scene.feat, q), (scene.offs, "<f4"),
                  (scene.scale, "<f4"), (scene.level, "u1"), (scene.W1, q),
                  (scene.b1, q), (scene.W2a, q), (scene.b2a, q),
                  (scene.W2c, q), (scene.b2c, q), (scene.W2s, q),
                  (scene.b2s, q)]
        if v4 and scene.bank:
            arrays += [(scene.Wb1, "<f4"), (scene.bb1, "<f4"), (scene.Wb2, "<f4"), (scene.bb2, "<f4")]
        for a, dt in arrays:
            fh.write(np.ascontiguousarray(a, dtype=dt).tobytes())


def read_gsc2(path: str) -> Scene:
    with open(path, "rb") as fh:
        data = fh.read()
    if len(data) < _HDR.size:
        raise ValueError(f"GSC2 truncated header at offset {len(data)}")
    magic, ver, n, F, K, L, H, d0, *bbox = _HDR.unpack_from(data, 0)
    if magic != b"GSC2" or ver not in (2, 3, 4):
        raise ValueError("GSC2 bad magic/version at offset 0")
    q = "<f4" if ver >= 3 else "i1"
    off = _HDR.size
    flags = 0
    if ver == 4:
        if off + 4 > len(data):
            raise ValueError(f"GSC2 truncated at offset {off}")
        flags = struct.unpack_from("<I", data, off)[0]
        off += 4
    dist, bank = bool(flags & 1), bool(flags & 2)

    def take(count, dt, shape):
        nonlocal off
        nb = count * np.dtype(dt).itemsize
        if off + nb > len(data):
            raise ValueError(f"GSC2 truncated at offset {off}")
        a = np.frombuffer(data, dtype=dt, count=count, offset=off).reshape(shape).copy()
        off += nb
        return a

    pos = take(n * 3, "<f4", (n, 3))
    feat = take(n * F, q, (n, F))
    offs = take(n * K * 3, "<f4", (n, K, 3))
    scale = take(n * 3, "<f4", (n, 3))
    level = take(n, "u1", (n,))
    W1 = take((F + 3 + dist) * 3 * H, q, (F + 3 + dist, 3 * H))
    b1 = take(3 * H, q, (3 * H,))
    W2a = take(H * K, q, (H, K))
    b2a = take(K, q, (K,))
    W2c = take(H * 3 * K, q, (H, 3 * K))
    b2c = take(3 * K, q, (3 * K,))
    W2s = take(H * 7 * K, q, (H, 7 * K))
    b2s = take(7 * K, q, (7 * K,))
    extra = {}
    if bank:
        extra = dict(Wb1=take(4 * F, "<f4", (4, F)), bb1=take(F, "<f4", (F,)), Wb2=take(F * 3, "<f4", (F, 3)),
                     bb2=take(3, "<f4", (3,)))
    return Scene(pos=pos, feat=feat, offs=offs, scale=scale, level=level, W1=W1, b1=b1,
                 W2a=W2a, b2a=b2a, W2c=W2c, b2c=b2c, W2s=W2s, b2s=b2s, L=L, d0=d0, real=ver >= 3,
                 dist_input=dist, bank=bank, bbox=np.array(bbox, np.float32), **extra)


def write_trajectory(rigs, path: str, fov_y_deg: float, width: int, height: int) -> None:
    """JSON-lines trajectory; floats written with repr (exact round trip)."""
    with open(path, "w") as fh:
        for r in rigs:
            fh.write(json.dumps({"t": r.t, "lp": [float(x) for x in r.lp], "lq": [float(x) for x in r.lq],
                                 "rp": [float(x) for x in r.rp], "rq": [float(x) for x in r.rq],
                                 "fov": fov_y_deg, "w": width, "h": height}) + "\n")


def read_trajectory(path: str):
    rigs = []
    with open(path) as fh:
        for line in fh:
            d = json.loads(line)
            rigs.append(Rig(lp=np.array(d["lp"]), lq=np.array(d["lq"]), rp=np.array(d["rp"]),
                            rq=np.array(d["rq"]), t=d["t"]))
    return rigs


# ----------------------------------------------------------------------------
# BASELINE.json configs
# ----------------------------------------------------------------------------

@dataclass
class Config:
    name: str
    n: int
    side: float
    L: int
    width: int
    height: int
    fov_y_deg: float
    d_max: int
    seed: int = 7
    near: float = 0.05
    far: float = 5000.0
    real: bool = False     # F4: fp32 non-grid features / decoder weights (with_real_weights)
    dist: bool = False     # F4 / R32: distance input
    bank: bool = False     # F4 / R32: feature bank

    def scene(self) -> Scene:
        sc = make_city_scene(self.seed, self.n, self.side, self.L, self.width, self.height, self.fov_y_deg)
        return with_real_weights(sc, dist=self.dist, bank=self.bank) if self.real else sc

    @property
    def center(self):
        return np.array([self.side / 2, self.side / 2, 0.0])


CONFIGS = {
    # configs[0]: 1k anchors x k=10, 64x64 single view (ipd 0), 4 poses
    "C1": Config("C1", 1000, 20.0, 3, 64, 64, 70.0, 10),
    # configs[1]: 100k static binocular 2K, no reuse (D_max = 1)
    "C2": Config("C2", 100_000, 130.0, 5, 1920, 1080, 70.0, 1),
    # configs[2]: 100k, 300-frame orbit, reuse (D_max = 10) vs full
    "C3": Config("C3", 100_000, 130.0, 5, 1920, 1080, 70.0, 10),
    # configs[3]: 1M city block, 2K binocular, ground-to-aerial, 1 B200
    "C4": Config("C4", 1_000_000, 400.0, 5, 1920, 1080, 70.0, 10),
    # configs[4]: 5M city, 2K binocular, split across GPUs
    "C5": Config("C5", 5_000_000, 900.0, 5, 1920, 1080, 70.0, 10),
    # SURVEY §8(f) F4 (real-weights path): the C1 / C3 scenes with fp32 non-grid features and decoder
    # weights, and a Scaffold-GS-style scene (L = 1: no LoD) with real weights on the C3 orbit
    "C1R": Config("C1R", 1000, 20.0, 3, 64, 64, 70.0, 10, real=True),
    "C3R": Config("C3R", 100_000, 130.0, 5, 1920, 1080, 70.0, 10, real=True),
    "C3S": Config("C3S", 100_000, 130.0, 1, 1920, 1080, 70.0, 10, real=True),
    "C4R": Config("C4R", 1_000_000, 400.0, 5, 1920, 1080, 70.0, 10, real=True),
    # F4 with the Scaffold-GS combine inputs (R32): distance input + feature bank, on C1 / C3 / C3S
    "C1B": Config("C1B", 1000, 20.0, 3, 64, 64, 70.0, 10, real=True, dist=True, bank=True),
    "C3B": Config("C3B", 100_000, 130.0, 5, 1920, 1080, 70.0, 10, real=True, dist=True, bank=True),
    "C3SB": Config("C3SB", 100_000, 130.0, 1, 1920, 1080, 70.0, 10, real=True, dist=True, bank=True),
    # SURVEY §8(f) F3 (depth-policy study): the C3 scene with a street-level head turn whose speed
    # accelerates (C3A: 0.2 -> 40 deg/frame over 300 frames) or changes in stages (C3T: 1 / 10 / 35 deg
    # per frame, 100 frames each) -- the novelty rate then spans 0 -> ~30%, where the guides differ
    "C3A": Config("C3A", 100_000, 130.0, 5, 1920, 1080, 70.0, 10),
    "C3T": Config("C3T", 100_000, 130.0, 5, 1920, 1080, 70.0, 10),
    # SURVEY §8(f) F2 zoom-out experiment: the C5 city, the camera pointing at the centre and
    # moving away from it (40 m -> 1800 m along a rising diagonal, 600 frames)
    "C5Z": Config("C5Z", 5_000_000, 900.0, 5, 1920, 1080, 70.0, 10),
}


def config(name: str) -> Config:
    return CONFIGS[name]


def c1_poses(cfg: Config):
    """Four C1 poses: frontal, 45 deg oblique, close-up that cuts
    the near plane, far (LoD drop).  ipd = 0 (single view through the pair API)."""
    c = cfg.center + np.array([0.0, 0.0, 5.0])
    s = cfg.side
    return [
        look_at_rig(c + np.array([0.0, -1.6 * s, 1.7]), c, 0.0, 0.0),
        look_at_rig(c + np.array([1.1 * s, -1.1 * s, 1.1 * s]), c, 0.0, 1.0),
        look_at_rig(c + np.array([0.05 * s, -0.42 * s, -2.0]), c + np.array([0.0, 0.0, -3.0]), 0.0, 2.0),
        look_at_rig(c + np.array([0.0, -18.0 * s, 4.0 * s]), c, 0.0, 3.0),
    ]


def trajectory(cfg: Config, n_frames: int | None = None):
    """The trajectory of a config."""
    s = cfg.side
    c = cfg.center
    name = cfg.name[:2]          # C1R / C3R / C3S follow their base config's trajectory
    if name == "C1":
        return c1_poses(cfg)
    if name == "C2":
        # two static poses, 100 frames each
        n = n_frames or 200
        a = look_at_rig(c + np.array([0.35 * s, 0.0, 1.7]), c, 0.064)
        b = look_at_rig(c + np.array([0.35 * s, 0.0, 60.0]), c, 0.064)
        return [a if f < n // 2 else b for f in range(n)]
    if cfg.name == "C5Z":
        n = n_frames or 600
        d = np.array([-1.0, -0.6, 0.7])
        d /= np.linalg.norm(d)
        return [look_at_rig(c + d * (40.0 + (1800.0 - 40.0) * f / max(1, n - 1)), c, 0.064, t=f / 90.0)
                for f in range(n)]
    if cfg.name in ("C3A", "C3T"):
        n = n_frames or 300
        if cfg.name == "C3A":
            steps = [0.2 + (40.0 - 0.2) * f / max(1, n - 1) for f in range(n)]
        else:
            steps = [1.0 if f < n // 3 else (10.0 if f < 2 * n // 3 else 35.0) for f in range(n)]
        return make_pan(c + np.array([0.25 * s, 0.05 * s, 1.7]), c + np.array([0.05 * s, 0.05 * s, 1.7]),
                        180.0, steps)
    if name == "C3":
        return make_orbit(c, 0.35 * s, 0.35 * s, 1.7, 60.0, n_frames or 300, 0.3)
    if name == "C4":
        return make_orbit(c, 0.3 * s, 0.7 * s, 1.7, 300.0, n_frames or 600, 0.25)
    if name == "C5":
        return make_orbit(c, 0.3 * s, 0.7 * s, 1.7, 300.0, n_frames or 2400, 0.25)
    raise KeyError(cfg.name)
