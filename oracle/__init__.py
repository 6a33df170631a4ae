"""ctypes binding of the CPU oracle (liblocc_oracle.so).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  It shares no code
with the CUDA path (paper_2304_09439_b200/); see locc_oracle.h for what it computes.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liblocc_oracle.so")
# tools/oracle_mutations.py points this at a deliberately broken build to check the pins' power
_LIB_OVERRIDE = os.environ.get("LOCC_ORACLE_LIB")
_lib = None


def build(force: bool = False) -> str:
    if _LIB_OVERRIDE:
        return _LIB_OVERRIDE
    src = os.path.join(_HERE, "locc_oracle.cpp")
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "locc_oracle.h"))):
        subprocess.check_call(["make", "-s", "-C", _HERE, "liblocc_oracle.so"])
    return _LIB


class _Cfg(C.Structure):
    _fields_ = [("M", C.c_int32), ("H", C.c_int32), ("F", C.c_int32), ("bf16_emul", C.c_int32),
                ("n_threads", C.c_int32), ("global_max", C.c_int32)]


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        vp = C.c_void_p
        L.oracle_shape_prep.argtypes = [vp, C.c_int32, C.c_int32, vp, vp, vp, vp]
        L.oracle_rel_transform.argtypes = [vp] * 6
        L.oracle_query.argtypes = [C.POINTER(_Cfg), vp, C.c_size_t, vp, C.c_int32, C.c_int32, vp, vp,
                                   C.c_int64] + [vp] * 7
        L.oracle_head_grad.argtypes = [C.POINTER(_Cfg), vp, C.c_size_t, vp, vp, vp, vp, vp, vp]
        L.oracle_query_grad.argtypes = [C.POINTER(_Cfg), vp, C.c_size_t, vp, C.c_int32, C.c_int32, vp, vp, C.c_int64,
                                        vp, vp, vp]
        L.oracle_unet_n_params.argtypes = [C.c_int32, C.c_int32]
        L.oracle_unet_n_params.restype = C.c_int64
        L.oracle_conv3d.argtypes = [vp, C.c_int32, C.c_int32, vp, vp, C.c_int32, C.c_int32, C.c_int32, vp]
        L.oracle_encode_grid.argtypes = [C.POINTER(_Cfg), vp, C.c_size_t, vp, C.c_size_t, vp, C.c_int32, vp, vp]
        L.oracle_query_cells.argtypes = [C.POINTER(_Cfg), vp, C.c_size_t, vp, C.c_size_t, vp, C.c_int32, C.c_int32,
                                         vp, vp, C.c_int64] + [vp] * 7
        L.oracle_sim_run.argtypes = [C.POINTER(_Cfg), vp, C.c_size_t, vp, C.c_size_t, vp, C.c_int32, C.c_int32, vp,
                                     C.c_int32, vp, vp, vp, C.c_double, vp, vp]
        L.oracle_load_weights.argtypes = [C.c_char_p, vp, C.c_size_t, vp, vp, vp]
        L.oracle_load_weights.restype = C.c_int64
        L.oracle_n_params.argtypes = [C.c_int32, C.c_int32]
        L.oracle_n_params.restype = C.c_int64
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def n_params(H=256, F=64):
    return int(lib().oracle_n_params(H, F))


def shape_prep(points_k3, M=6):
    """O0 for one shape -> (lo[3], hi[3], eps2, cell[K])."""
    p = np.ascontiguousarray(points_k3, np.float32)
    K = p.shape[0]
    lo = np.zeros(3, np.float32)
    hi = np.zeros(3, np.float32)
    e2 = np.zeros(1, np.float32)
    cell = np.zeros(K, np.int32)
    rc = lib().oracle_shape_prep(_p(p), K, M, _p(lo), _p(hi), _p(e2), _p(cell))
    if rc:
        raise ValueError(f"oracle_shape_prep: {rc}")
    return lo, hi, np.float32(e2[0]), cell


def rel_transform(poseA, poseB):
    """O1-O3 -> (R_BA[3,3], t_BA[3], R_AB[3,3], t_AB[3]) float32."""
    a = np.ascontiguousarray(poseA, np.float32)
    b = np.ascontiguousarray(poseB, np.float32)
    out = [np.zeros(9, np.float32), np.zeros(3, np.float32), np.zeros(9, np.float32), np.zeros(3, np.float32)]
    rc = lib().oracle_rel_transform(_p(a), _p(b), *[_p(o) for o in out])
    if rc:
        raise ValueError(f"oracle_rel_transform: {rc}")
    return out[0].reshape(3, 3), out[1], out[2].reshape(3, 3), out[3]


def query(weights_flat, points, pairs, poses, M=6, H=256, F=64, bf16_emul=False, n_threads=0):
    """Whole query O0-O9.  Returns dict with probs, labels, logits (float64), kept, occ (int32 [N][2]),
    masks (uint32 [N][2][ceil(K/32)]) and emb (float64 [N][2][F])."""
    w = np.ascontiguousarray(weights_flat, np.float32)
    pts = np.ascontiguousarray(points, np.float32)
    pr = np.ascontiguousarray(pairs, np.int32).reshape(-1, 2)
    po = np.ascontiguousarray(poses, np.float32).reshape(-1, 2, 7)
    S, K = pts.shape[0], pts.shape[1]
    N = pr.shape[0]
    words = (K + 31) // 32
    out = dict(probs=np.zeros(N), labels=np.zeros(N, np.uint8), logits=np.zeros(N),
               kept=np.zeros((N, 2), np.int32), occ=np.zeros((N, 2), np.int32),
               masks=np.zeros((N, 2, words), np.uint32), emb=np.zeros((N, 2, F)))
    cfg = _Cfg(M, H, F, 1 if bf16_emul else 0, n_threads)
    rc = lib().oracle_query(C.byref(cfg), _p(w), w.size, _p(pts), S, K, _p(pr), _p(po), N,
                            _p(out["probs"]), _p(out["labels"]), _p(out["logits"]), _p(out["kept"]),
                            _p(out["occ"]), _p(out["masks"]), _p(out["emb"]))
    if rc:
        raise ValueError(f"oracle_query: {rc}")
    return out


def head_grad(weights_flat, eA, eB, poseA, poseB, H=256, F=64):
    """NEXT-2: predictor logit and d logit / d [q_A, t_A, q_B, t_B] (14) at given embeddings (fp64)."""
    w = np.ascontiguousarray(weights_flat, np.float32)
    a = np.ascontiguousarray(eA, np.float64)
    b = np.ascontiguousarray(eB, np.float64)
    pa = np.ascontiguousarray(poseA, np.float64)
    pb = np.ascontiguousarray(poseB, np.float64)
    lg = np.zeros(1)
    g = np.zeros(14)
    cfg = _Cfg(6, H, F, 0, 1)
    rc = lib().oracle_head_grad(C.byref(cfg), _p(w), w.size, _p(a), _p(b), _p(pa), _p(pb), _p(lg), _p(g))
    if rc:
        raise ValueError(f"oracle_head_grad: {rc}")
    return float(lg[0]), g


def query_grad(weights_flat, points, pairs, poses, M=6, H=256, F=64, bf16_emul=False, n_threads=0):
    """Whole query plus d logit / d pose per pair: returns (logits [N], grad [N][14], margin [N]) with
    margin the pair's smallest ReLU / max-routing distance from its threshold (inf: short-circuit)."""
    w = np.ascontiguousarray(weights_flat, np.float32)
    pts = np.ascontiguousarray(points, np.float32)
    pr = np.ascontiguousarray(pairs, np.int32).reshape(-1, 2)
    po = np.ascontiguousarray(poses, np.float32).reshape(-1, 2, 7)
    N = pr.shape[0]
    lg = np.zeros(N)
    g = np.zeros((N, 14))
    mg = np.zeros(N)
    cfg = _Cfg(M, H, F, 1 if bf16_emul else 0, n_threads)
    rc = lib().oracle_query_grad(C.byref(cfg), _p(w), w.size, _p(pts), pts.shape[0], pts.shape[1], _p(pr), _p(po), N,
                                 _p(lg), _p(g), _p(mg))
    if rc:
        raise ValueError(f"oracle_query_grad: {rc}")
    return lg, g, mg


# ----------------------------------------------------------------------------- NEXT-1 (encode once)
def unet_n_params(H=256, F=64):
    return int(lib().oracle_unet_n_params(H, F))


def conv3d(x, W, b=None, pad=0, transposed=False):
    """One 3x3x3 layer in fp64: x [D,D,D,Cin] (z, y, x, channel), W [Cout][Cin][27] -> y grid."""
    x = np.ascontiguousarray(x, np.float64)
    W = np.ascontiguousarray(W, np.float64)
    D, Cin = x.shape[0], x.shape[3]
    Cout = W.shape[0]
    Do = D + 2 - 2 * pad if transposed else D + 2 * pad - 2
    y = np.zeros((Do, Do, Do, Cout))
    bb = None if b is None else np.ascontiguousarray(b, np.float64)
    rc = lib().oracle_conv3d(_p(x), D, Cin, _p(W), _p(bb), Cout, pad, 1 if transposed else 0, _p(y))
    if rc:
        raise ValueError(f"oracle_conv3d: {rc}")
    return y


def encode_grid(weights_flat, unet_flat, points_k3, M=6, H=256, F=64, global_max=False):
    """Encode one shape -> (G [M^3][H] cell-max grid, E [M^3][F] embedding grid), fp64."""
    w = np.ascontiguousarray(weights_flat, np.float32)
    u = np.ascontiguousarray(unet_flat, np.float32)
    p = np.ascontiguousarray(points_k3, np.float32)
    G = np.zeros((M ** 3, H))
    E = np.zeros((M ** 3, F))
    cfg = _Cfg(M, H, F, 0, 1, 1 if global_max else 0)
    rc = lib().oracle_encode_grid(C.byref(cfg), _p(w), w.size, _p(u), u.size, _p(p), p.shape[0], _p(G), _p(E))
    if rc:
        raise ValueError(f"oracle_encode_grid: {rc}")
    return G, E


def query_cells(weights_flat, unet_flat, points, pairs, poses, M=6, H=256, F=64, n_threads=0, global_max=False):
    """Encode-once query: dict with probs, labels, logits, nsel [N][2], cells [N][2][ceil(M^3/32)],
    emb [N][2][F] and grids [S][M^3][F] (zeros for unreferenced shapes)."""
    w = np.ascontiguousarray(weights_flat, np.float32)
    u = np.ascontiguousarray(unet_flat, np.float32)
    pts = np.ascontiguousarray(points, np.float32)
    pr = np.ascontiguousarray(pairs, np.int32).reshape(-1, 2)
    po = np.ascontiguousarray(poses, np.float32).reshape(-1, 2, 7)
    S, K = pts.shape[0], pts.shape[1]
    N = pr.shape[0]
    words = (M ** 3 + 31) // 32
    out = dict(probs=np.zeros(N), labels=np.zeros(N, np.uint8), logits=np.zeros(N),
               nsel=np.zeros((N, 2), np.int32), cells=np.zeros((N, 2, words), np.uint32),
               emb=np.zeros((N, 2, F)), grids=np.zeros((S, M ** 3, F)))
    cfg = _Cfg(M, H, F, 0, n_threads, 1 if global_max else 0)
    rc = lib().oracle_query_cells(C.byref(cfg), _p(w), w.size, _p(u), u.size, _p(pts), S, K, _p(pr), _p(po), N,
                                  _p(out["probs"]), _p(out["labels"]), _p(out["logits"]), _p(out["nsel"]),
                                  _p(out["cells"]), _p(out["emb"]), _p(out["grids"]))
    if rc:
        raise ValueError(f"oracle_query_cells: {rc}")
    return out


# ----------------------------------------------------------------------------- NEXT-3 (closed loop)
def sim_run(weights_flat, points, sim, ids, body, state, t0=0.0, unet_flat=None, M=6, H=256, F=64, n_threads=0):
    """Advance `state` [E][3][13] (float64, copied) by sim['substeps'] substeps.  sim: dict with h,
    substeps, detector ('crop' | 'cells'), gravity, ks, kd, amp, freq, slack.  Returns (state,
    contacts [E][3], margins [E][4])."""
    w = np.ascontiguousarray(weights_flat, np.float32)
    u = None if unet_flat is None else np.ascontiguousarray(unet_flat, np.float32)
    pts = np.ascontiguousarray(points, np.float32)
    ids = np.ascontiguousarray(ids, np.int32).reshape(-1, 3)
    E = ids.shape[0]
    body = np.ascontiguousarray(body, np.float64).reshape(E, 3, 4)
    st = np.array(state, np.float64).reshape(E, 3, 13).copy()
    sv = np.array([sim["h"], sim["substeps"], 1 if sim.get("detector", "crop") == "cells" else 0, *sim["gravity"],
                   sim["ks"], sim["kd"], *sim["amp"], sim["freq"], sim["slack"]], np.float64)
    contacts = np.zeros((E, 3), np.int32)
    margins = np.zeros((E, 4))
    cfg = _Cfg(M, H, F, 0, n_threads)
    rc = lib().oracle_sim_run(C.byref(cfg), _p(w), w.size, _p(u), 0 if u is None else u.size, _p(pts), pts.shape[0],
                              pts.shape[1], _p(sv), E, _p(ids), _p(body), _p(st), t0, _p(contacts), _p(margins))
    if rc:
        raise ValueError(f"oracle_sim_run: {rc}")
    return st, contacts, margins


def load_weights(manifest):
    cap = 1 << 24
    buf = np.zeros(cap, np.float32)
    M = np.zeros(1, np.int32)
    H = np.zeros(1, np.int32)
    F = np.zeros(1, np.int32)
    n = lib().oracle_load_weights(manifest.encode(), _p(buf), cap, _p(M), _p(H), _p(F))
    if n < 0:
        raise ValueError(f"oracle_load_weights: {n}")
    return buf[:n].copy(), (int(M[0]), int(H[0]), int(F[0]))
