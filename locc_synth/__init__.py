"""Seeded synthetic inputs for LOCC (shapes, poses, weights) — shared by both sides.

This module is the ONLY code the CPU oracle (`oracle/`) and the CUDA path
(`paper_2304_09439_b200/`) have in common, and it holds none of the method's
arithmetic: no transform, no crop, no voxel binning, no network.  It only draws
random numbers and writes files.

Workload recipe:

* Shapes — procedural, mostly non-convex household-like objects standing in for
  the 1030 Google Scanned Objects ("1030 object meshes most of which
  are non-convex").  Families: box, wedge, torus, hollow tube, bowl, cup, mug
  with handle, L-bracket.  Size log-normal (median AABB diagonal 12 cm,
  sigma_log 0.4), per-axis stretch U(0.7, 1.3).  K points drawn uniformly on the
  surface ("uniformly sample 1500 points from the surface"; SPEC.md
  S:61-69 area-weighted triangle pick + uniform barycentric), then every cloud is
  shifted so its AABB centre is the origin ("define the center of the
  mesh as the center of AABB").
* Poses — PAPER.md:34 "uniform sampling": rotations uniform on SO(3) (normalised
  4-D Gaussian), t_A ~ U[-0.5, 0.5]^3 m, t_B = t_A + U[-L, L]^3 with
  L = s * (r_a + r_b), r = half the AABB diagonal; pairs (a, b) uniform with
  replacement.  `s` is the pose-density knob (s = 0.5 for C1-C3).
* Weights — no checkpoint exists (BASELINE.json north_star: "seeded random-init
  weights").  `he`: SPEC.md S:311 init (He-uniform for ReLU layers, Xavier for
  the final linear layers), biases U(+-1/sqrt(fan_in)).  `spread`: W1 He bound
  x10, all biases 0, then out.W scaled and out.b set from a calibration file
  written by `tools/calibrate_spread.py` (which calls only the oracle).
  `spread_bias`: the `spread` weights with every hidden and projection bias drawn
  as in `he` (U(+-1/sqrt(fan_in))), out.W / out.b calibrated the same way (its own
  file) — the set that exercises every bias path of the GPU kernels.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

__all__ = [
    "FAMILIES", "make_shapes", "make_pairs_poses", "weight_layout", "make_weights",
    "flatten_weights", "write_weights", "read_weights", "default_calibration_path",
    "load_calibration", "Workload", "make_workload", "WEIGHT_SETS", "weight_set",
]

FAMILIES = ("box", "wedge", "torus", "tube", "bowl", "cup", "mug", "lbracket")


# --------------------------------------------------------------------------- meshes
def _grid(fn, nu, nv, u0, u1, v0, v1):
    """Triangulate a parametric patch fn(u, v) -> (..., 3) on an nu x nv grid."""
    u = np.linspace(u0, u1, nu + 1)
    v = np.linspace(v0, v1, nv + 1)
    U, V = np.meshgrid(u, v, indexing="ij")
    P = fn(U, V)  # (nu+1, nv+1, 3)
    a = P[:-1, :-1].reshape(-1, 3)
    b = P[1:, :-1].reshape(-1, 3)
    c = P[1:, 1:].reshape(-1, 3)
    d = P[:-1, 1:].reshape(-1, 3)
    return np.concatenate([np.stack([a, b, c], 1), np.stack([a, c, d], 1)], 0)


def _box(lo, hi):
    lo = np.asarray(lo, float)
    hi = np.asarray(hi, float)
    c = np.array([[lo[0] if i & 1 == 0 else hi[0], lo[1] if i & 2 == 0 else hi[1],
                   lo[2] if i & 4 == 0 else hi[2]] for i in range(8)])
    quads = [(0, 1, 3, 2), (4, 6, 7, 5), (0, 4, 5, 1), (2, 3, 7, 6), (0, 2, 6, 4), (1, 5, 7, 3)]
    tris = []
    for q in quads:
        tris.append([c[q[0]], c[q[1]], c[q[2]]])
        tris.append([c[q[0]], c[q[2]], c[q[3]]])
    return np.array(tris)


def _cyl(r, z0, z1, n=32):
    return _grid(lambda u, v: np.stack([r * np.cos(u), r * np.sin(u), v], -1), n, 2, 0, 2 * np.pi, z0, z1)


def _annulus(r0, r1, z, n=32):
    return _grid(lambda u, v: np.stack([v * np.cos(u), v * np.sin(u), np.full_like(u, z)], -1),
                 n, 2, 0, 2 * np.pi, r0, r1)


def _family_mesh(fam, rng):
    if fam == "box":
        return _box([0, 0, 0], [1, 1, 1])
    if fam == "wedge":
        p = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 0, 1], [0, 1, 1]], float)
        t = [(0, 2, 1), (3, 4, 5), (0, 1, 4), (0, 4, 3), (0, 3, 5), (0, 5, 2), (1, 2, 5), (1, 5, 4)]
        return p[np.array(t)]
    if fam == "torus":
        R, r = 1.0, rng.uniform(0.2, 0.45)
        return _grid(lambda u, v: np.stack([(R + r * np.cos(v)) * np.cos(u), (R + r * np.cos(v)) * np.sin(u),
                                            r * np.sin(v)], -1), 32, 12, 0, 2 * np.pi, 0, 2 * np.pi)
    if fam == "tube":
        ri = rng.uniform(0.6, 0.9)
        return np.concatenate([_cyl(1.0, 0, 2), _cyl(ri, 0, 2), _annulus(ri, 1.0, 0), _annulus(ri, 1.0, 2)])
    if fam == "bowl":
        ri = rng.uniform(0.85, 0.95)

        def sph(rad):
            return lambda u, v: np.stack([rad * np.sin(v) * np.cos(u), rad * np.sin(v) * np.sin(u),
                                          -rad * np.cos(v)], -1)
        return np.concatenate([_grid(sph(1.0), 32, 12, 0, 2 * np.pi, 0, np.pi / 2),
                               _grid(sph(ri), 32, 12, 0, 2 * np.pi, 0, np.pi / 2), _annulus(ri, 1.0, 0)])
    if fam in ("cup", "mug"):
        ri, hb = rng.uniform(0.85, 0.93), 0.1
        parts = [_cyl(1.0, 0, 2), _annulus(0, 1.0, 0), _cyl(ri, hb, 2), _annulus(0, ri, hb), _annulus(ri, 1.0, 2)]
        if fam == "mug":
            R, r = 0.55, 0.1
            parts.append(_grid(lambda u, v: np.stack([1.0 + (R + r * np.cos(v)) * np.cos(u), r * np.sin(v),
                                                      1.0 + (R + r * np.cos(v)) * np.sin(u)], -1),
                               16, 8, -np.pi / 2, np.pi / 2, 0, 2 * np.pi))
        return np.concatenate(parts)
    if fam == "lbracket":
        w = rng.uniform(0.2, 0.5)
        return np.concatenate([_box([0, 0, 0], [2, w, 1]), _box([0, w, 0], [w, 2, 1])])
    raise ValueError(fam)


def _sample_surface(tris, K, rng):
    """K points uniform on the surface: area-weighted triangle pick + barycentric."""
    e1 = tris[:, 1] - tris[:, 0]
    e2 = tris[:, 2] - tris[:, 0]
    area = 0.5 * np.linalg.norm(np.cross(e1, e2), axis=1)
    idx = rng.choice(len(tris), size=K, p=area / area.sum())
    r1 = np.sqrt(rng.random(K))
    r2 = rng.random(K)
    a = 1.0 - r1
    b = r1 * (1.0 - r2)
    c = r1 * r2
    t = tris[idx]
    return a[:, None] * t[:, 0] + b[:, None] * t[:, 1] + c[:, None] * t[:, 2]


def make_shapes(S: int, K: int, seed: int = 1, families=FAMILIES):
    """S point clouds [S][K][3] float32 in metres, each centred on its AABB centre.

    Returns (points, family_names)."""
    rng = np.random.default_rng(seed)
    out = np.empty((S, K, 3), np.float32)
    fams = []
    for s in range(S):
        fam = families[s % len(families)] if s < len(families) else families[rng.integers(len(families))]
        tris = _family_mesh(fam, rng)
        # random orientation of the family template in its own frame, then AABB-normalise
        Qm, Rr = np.linalg.qr(rng.standard_normal((3, 3)))
        Rm = Qm * np.sign(np.diag(Rr))
        if np.linalg.det(Rm) < 0:
            Rm[:, 0] = -Rm[:, 0]
        tris = tris @ Rm.T
        lo = tris.reshape(-1, 3).min(0)
        hi = tris.reshape(-1, 3).max(0)
        tris = (tris - lo) / np.linalg.norm(hi - lo)
        tris = tris * rng.uniform(0.7, 1.3, size=3)
        tris = tris * (0.12 * np.exp(0.4 * rng.standard_normal()))
        p = _sample_surface(tris, K, rng)
        c = 0.5 * (p.min(0) + p.max(0))
        out[s] = (p - c).astype(np.float32)
        fams.append(fam)
    return out, fams


def _half_diag(points):
    p = points.astype(np.float64)
    return 0.5 * np.linalg.norm(p.max(1) - p.min(1), axis=1)


def make_pairs_poses(points, N: int, s: float = 0.5, seed: int = 2):
    """N uniform pairs with uniform poses at density s.  pairs int32 [N][2]; poses float32
    [N][2][7] as (qw, qx, qy, qz, tx, ty, tz); side 0 = A = pairs[i][0]."""
    rng = np.random.default_rng(seed)
    S = points.shape[0]
    r = _half_diag(points)
    pairs = rng.integers(0, S, size=(N, 2)).astype(np.int32)
    q = rng.standard_normal((N, 2, 4))
    q /= np.linalg.norm(q, axis=-1, keepdims=True)
    tA = rng.uniform(-0.5, 0.5, size=(N, 3))
    L = s * (r[pairs[:, 0]] + r[pairs[:, 1]])
    tB = tA + rng.uniform(-1.0, 1.0, size=(N, 3)) * L[:, None]
    poses = np.empty((N, 2, 7), np.float32)
    poses[:, :, :4] = q
    poses[:, 0, 4:] = tA
    poses[:, 1, 4:] = tB
    return pairs, poses


# --------------------------------------------------------------------------- weights
def weight_layout(H: int = 256, F: int = 64, P: int = 128):
    """Canonical parameter order (SURVEY.md §8(c) "Parameter layout"): (name, out, in).
    Row-major [out][in]; each layer's W then its bias b[out]."""
    L = [("enc.l1", H, 3), ("enc.l2", H, H), ("enc.l3", H, H), ("enc.proj", F, H),
         ("obj.l1", P, F + 7), ("obj.l2", P, P), ("obj.l3", P, P),
         ("pair.l1", P, P), ("pair.l2", P, P), ("pair.l3", P, P), ("out", 1, P)]
    out = []
    for name, o, i in L:
        out.append((name + ".W", o, i))
        out.append((name + ".b", o, 1))
    return out


_LINEAR_FINAL = ("enc.proj", "out")  # linear (no ReLU) layers -> Xavier init


def make_weights(kind: str = "spread", H: int = 256, F: int = 64, seed: int = 3, calib=None):
    """Seeded random-init weights as an ordered dict name -> float32 array.

    kind='he': He-uniform (ReLU layers) / Xavier-uniform (enc.proj, out) weights,
    biases U(+-1/sqrt(fan_in)).  kind='spread': same draws, enc.l1.W bound x10 and
    all biases 0; if `calib` ({'scale', 'bias'}) is given, out.W *= scale and
    out.b = bias.  kind='spread_bias': 'spread' with the 'he' biases (calibrated
    the same way).  kind='zero': every parameter 0."""
    rng = np.random.default_rng(seed)
    w = {}
    for name, o, i in weight_layout(H, F):
        layer = name.rsplit(".", 1)[0]
        if name.endswith(".W"):
            if layer in _LINEAR_FINAL:
                bound = np.sqrt(6.0 / (i + o))
            else:
                bound = np.sqrt(6.0 / i)
            if kind in ("spread", "spread_bias") and layer == "enc.l1":
                bound *= 10.0
            w[name] = rng.uniform(-bound, bound, size=(o, i)).astype(np.float32)
        else:
            fan_in = w[layer + ".W"].shape[1]
            b = rng.uniform(-1, 1, size=(o,)) / np.sqrt(fan_in)
            w[name] = (b if kind in ("he", "spread_bias") else np.zeros(o)).astype(np.float32)
    if kind == "zero":
        for k in w:
            w[k] = np.zeros_like(w[k])
    if kind in ("spread", "spread_bias") and calib is not None:
        w["out.W"] = (w["out.W"] * np.float32(calib["scale"])).astype(np.float32)
        w["out.b"] = np.array([calib["bias"]], np.float32)
    return w


WEIGHT_SETS = ("spread", "spread_bias")  # the calibrated sets the GPU parity suites run over


def weight_set(kind: str = "spread"):
    """A calibrated weight set ('spread' or 'spread_bias') as the flat canonical float32 vector."""
    return flatten_weights(make_weights(kind, calib=load_calibration(kind=kind)))


def unet_layout(H: int = 256, F: int = 64, C: int = 128):
    """NEXT-1 U-Net parameter order (Q30): (name, shape).  3D kernels [out][in][27]."""
    L = [("unet.c1", C, H), ("unet.c2", C, C), ("unet.c3", C, C), ("unet.c4", C, C),
         ("unet.d4", C, C), ("unet.d3", C, 2 * C), ("unet.d2", C, 2 * C), ("unet.d1", C, 2 * C)]
    out = []
    for name, o, i in L:
        out.append((name + ".W", (o, i, 27)))
        out.append((name + ".b", (o,)))
    out.append(("unet.proj.W", (F, 2 * C)))
    out.append(("unet.proj.b", (F,)))
    return out


def make_unet_weights(kind: str = "spread", H: int = 256, F: int = 64, seed: int = 4):
    """Seeded U-Net weights: He-uniform 3D kernels (fan_in = 27 Cin), Xavier-uniform projection;
    biases 0 ('spread') or U(+-1/sqrt(fan_in)) ('he'); 'zero' = all 0."""
    rng = np.random.default_rng(seed)
    w = {}
    for name, shape in unet_layout(H, F):
        if name.endswith(".W"):
            if name == "unet.proj.W":
                bound = np.sqrt(6.0 / (shape[0] + shape[1]))
            else:
                bound = np.sqrt(6.0 / (shape[1] * 27))
            w[name] = rng.uniform(-bound, bound, size=shape).astype(np.float32)
        else:
            fan_in = int(np.prod(w[name[:-2] + ".W"].shape[1:]))
            b = rng.uniform(-1, 1, size=shape) / np.sqrt(fan_in)
            w[name] = (b if kind == "he" else np.zeros(shape)).astype(np.float32)
    if kind == "zero":
        for k in w:
            w[k] = np.zeros_like(w[k])
    return w


def flatten_unet(w, H: int = 256, F: int = 64):
    return np.concatenate([np.asarray(w[name], np.float32).reshape(-1) for name, _ in unet_layout(H, F)])


def flatten_weights(w, H: int = 256, F: int = 64):
    """Concatenate in canonical order -> 1-D float32."""
    parts = []
    for name, o, i in weight_layout(H, F):
        a = np.asarray(w[name], np.float32).reshape(-1)
        assert a.size == o * i, (name, a.size, o, i)
        parts.append(a)
    return np.concatenate(parts)


def write_weights(path_txt: str, w, M: int = 6, H: int = 256, F: int = 64):
    """Write the S:319/S:407-style checkpoint: text manifest `path_txt` + raw little-endian
    fp32 `<stem>.bin`.  Manifest: header `locc-weights 1 M H F`, then `name out in offset_bytes`."""
    stem = os.path.splitext(path_txt)[0]
    flat = flatten_weights(w, H, F)
    flat.astype("<f4").tofile(stem + ".bin")
    off = 0
    with open(path_txt, "w") as f:
        f.write(f"locc-weights 1 {M} {H} {F}\n")
        for name, o, i in weight_layout(H, F):
            f.write(f"{name} {o} {i} {off}\n")
            off += 4 * o * i
    return path_txt


def read_weights(path_txt: str):
    stem = os.path.splitext(path_txt)[0]
    with open(path_txt) as f:
        hdr = f.readline().split()
        M, H, F = int(hdr[2]), int(hdr[3]), int(hdr[4])
        rows = [ln.split() for ln in f if ln.strip()]
    raw = np.fromfile(stem + ".bin", "<f4")
    w = {}
    for name, o, i, off in rows:
        o, i, off = int(o), int(i), int(off)
        a = raw[off // 4: off // 4 + o * i]
        w[name] = a.reshape(o, i) if name.endswith(".W") else a.copy()
    return w, (M, H, F)


def default_calibration_path(kind: str = "spread"):
    return os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                        f"{kind}_calibration.json")


def load_calibration(path=None, kind: str = "spread"):
    path = path or default_calibration_path(kind)
    if not os.path.exists(path):
        return None
    with open(path) as f:
        return json.load(f)


# --------------------------------------------------------------------------- closed-loop scenes
SIM_DEFAULTS = dict(h=0.01 / 4 / 4, substeps=4, detector="crop", gravity=(0.0, 0.0, -9.81), ks=2.0, kd=0.02,
                    amp=(0.01, 0.01, 0.0), freq=2.0, slack=0.01)


def make_sim_scene(points, E: int, seed: int = 5, bowl: int = 4, drop: float = 0.03):
    """E environments of PAPER.md:91's scene: body 0 = the bowl (shape `bowl`, the synthetic bowl family),
    bodies 1, 2 = two random shapes dropped just above its rim.  Returns ids int32 [E][3], body float32
    [E][3][4] (m, Ixx, Iyy, Izz: 0.1 kg boxes of the shape's AABB) and state float32 [E][3][13]
    (q, t, v, w).  SIM_DEFAULTS holds the step constants (dt = 0.01/4 s, 4 substeps)."""
    rng = np.random.default_rng(seed)
    S = points.shape[0]
    ids = np.empty((E, 3), np.int32)
    ids[:, 0] = bowl
    ids[:, 1:] = rng.integers(0, S, size=(E, 2))
    ext = (points.max(1) - points.min(1)).astype(np.float64)
    m = 0.1
    body = np.empty((E, 3, 4), np.float32)
    for b in range(3):
        e = ext[ids[:, b]]
        body[:, b, 0] = m
        body[:, b, 1] = m / 12 * (e[:, 1] ** 2 + e[:, 2] ** 2)
        body[:, b, 2] = m / 12 * (e[:, 0] ** 2 + e[:, 2] ** 2)
        body[:, b, 3] = m / 12 * (e[:, 0] ** 2 + e[:, 1] ** 2)
    state = np.zeros((E, 3, 13), np.float32)
    state[:, 0, 0] = 1.0
    q = rng.standard_normal((E, 2, 4))
    q /= np.linalg.norm(q, axis=-1, keepdims=True)
    state[:, 1:, :4] = q
    rb = 0.5 * ext[bowl][2]
    state[:, 1, 4:7] = np.stack([rng.uniform(-0.02, 0.02, E), rng.uniform(-0.02, 0.02, E),
                                 rb + rng.uniform(0.0, drop, E)], 1)
    state[:, 2, 4:7] = np.stack([rng.uniform(-0.02, 0.02, E), rng.uniform(-0.02, 0.02, E),
                                 rb + drop + rng.uniform(0.0, drop, E)], 1)
    return ids, body, state


# --------------------------------------------------------------------------- workloads
@dataclass
class Workload:
    name: str
    points: np.ndarray
    pairs: np.ndarray
    poses: np.ndarray
    M: int = 6
    H: int = 256
    F: int = 64
    s: float = 0.5


def make_workload(name: str = "C1", N: int | None = None, K: int = 1500, s: float = 0.5,
                  S: int | None = None):
    """Named configs of BASELINE.json: C1 = 64 pairs over 16 shapes; C2 = 16,384 pairs over
    1030 shapes; C3 = 1,048,576 pairs over 1030 shapes (K = 1500, s = 0.5 unless given)."""
    defaults = {"C1": (64, 16), "C2": (16384, 1030), "C3": (1 << 20, 1030)}
    n0, s0 = defaults.get(name, (N or 64, S or 1030))
    N = N or n0
    S = S or s0
    pts, _ = make_shapes(S, K, seed=1)
    pairs, poses = make_pairs_poses(pts, N, s=s, seed=2)
    return Workload(name, pts, pairs, poses, s=s)
