"""Pins of the oracle's encode-once path (NEXT-1, Q27-Q30): the 3D conv / transposed conv
against scipy's correlate / convolve and each other's adjoint, the U-Net's index conventions on a
delta-kernel probe with a closed form, the cell selection against a brute-force box-intersection
superset property and a hand-derived worked example, and the whole query on a closed-form head."""
import json
import os

import numpy as np
import pytest
from scipy import signal

import locc_synth as ls
from conftest import cube26, pose
from test_oracle_network import head_weights, probe_weights

GOLD = os.path.join(os.path.dirname(__file__), "golden")
H, F, C = 256, 64, 128


# ----------------------------------------------------------------------------- conv / deconv
@pytest.mark.parametrize("pad", [0, 1, 2])
def test_conv3d_matches_scipy_correlate(oracle_mod, pad):
    rng = np.random.default_rng(50)
    D, Cin, Cout = 5, 3, 2
    x = rng.normal(size=(D, D, D, Cin))
    W = rng.normal(size=(Cout, Cin, 27))
    b = rng.normal(size=Cout)
    y = oracle_mod.conv3d(x, W, b, pad=pad)
    xp = np.pad(x, ((pad, pad),) * 3 + ((0, 0),))
    for o in range(Cout):
        want = b[o] + sum(signal.correlate(xp[..., i], W[o, i].reshape(3, 3, 3), mode="valid") for i in range(Cin))
        np.testing.assert_allclose(y[..., o], want, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("pad", [0, 1])
def test_deconv3d_matches_scipy_convolve(oracle_mod, pad):
    """Transposed conv (stride 1) = full convolution with the same kernel, cropped by pad."""
    rng = np.random.default_rng(51)
    D, Cin, Cout = 4, 3, 2
    x = rng.normal(size=(D, D, D, Cin))
    W = rng.normal(size=(Cout, Cin, 27))
    y = oracle_mod.conv3d(x, W, None, pad=pad, transposed=True)
    for o in range(Cout):
        full = sum(signal.convolve(x[..., i], W[o, i].reshape(3, 3, 3), mode="full") for i in range(Cin))
        want = full[pad:full.shape[0] - pad, pad:full.shape[1] - pad, pad:full.shape[2] - pad]
        np.testing.assert_allclose(y[..., o], want, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("pad", [0, 1])
def test_conv_deconv_adjoint(oracle_mod, pad):
    """<conv_W(x), y> = <x, deconv_{W^T}(y)>: the scatter definition against the gather one."""
    rng = np.random.default_rng(52)
    D, Cin, Cout = 6, 4, 3
    x = rng.normal(size=(D, D, D, Cin))
    W = rng.normal(size=(Cout, Cin, 27))
    cx = oracle_mod.conv3d(x, W, None, pad=pad)
    y = rng.normal(size=cx.shape)
    dy = oracle_mod.conv3d(y, W.transpose(1, 0, 2), None, pad=pad, transposed=True)
    assert dy.shape == x.shape
    a, b = float(np.sum(cx * y)), float(np.sum(x * dy))
    assert abs(a - b) <= 1e-10 * max(1.0, abs(a))


# ----------------------------------------------------------------------------- U-Net probe
def unet_probe():
    """Delta kernels: c1 reads G at offset (x, y, z) = (2, 0, 1) (valid), c2..c4 / d4..d2 the centre
    tap of their first 128 inputs, d1 (transposed valid) scatters to offset (0, 2, 1).  proj:
    E0 = d1[0], E1 = g[0], E2 = d1[3] + 0.5.  Closed form (D = 4 block):
    E0[p + (0,2,1)] = G[p + (2,0,1)][0] for p in [0,4)^3, else 0; E1 = mean_p G[p + (2,0,1)][0]."""
    u = ls.make_unet_weights("zero", H, F)
    k1 = 2 + 3 * (0 + 3 * 1)   # kx=2, ky=0, kz=1
    kd = 0 + 3 * (2 + 3 * 1)   # kx=0, ky=2, kz=1
    for o in range(C):
        u["unet.c1.W"][o, o, k1] = 1.0
        for l in ("c2", "c3", "c4", "d4", "d3", "d2"):
            u[f"unet.{l}.W"][o, o, 13] = 1.0
        u["unet.d1.W"][o, o, kd] = 1.0
    u["unet.proj.W"][0, 0] = 1.0
    u["unet.proj.W"][1, C + 0] = 1.0
    u["unet.proj.W"][2, 3] = 1.0
    u["unet.proj.b"][2] = 0.5
    return ls.flatten_unet(u)


def identity_encoder():
    return ls.flatten_weights(probe_weights(np.arange(H), np.arange(H)))


def test_unet_probe_closed_form(oracle_mod):
    pts, _ = ls.make_shapes(2, 600, seed=53)
    G, E = oracle_mod.encode_grid(identity_encoder(), unet_probe(), pts[0])
    # G pinned first: cell-wise max of (x+, y+, z+, x-, y-, z-) over the shape's points (empty -> 0)
    _, _, _, cell = oracle_mod.shape_prep(pts[0])
    p = pts[0].astype(np.float64)
    feats = np.concatenate([np.maximum(p, 0), np.maximum(-p, 0)], 1)
    g = np.zeros((216, 6))
    np.maximum.at(g, cell, feats)
    np.testing.assert_allclose(G[:, :6], g, rtol=0, atol=0)
    assert np.all(G[:, 6:] == 0)
    Gz = G.reshape(6, 6, 6, H)  # [z][y][x]
    blk = Gz[1:5, 0:4, 2:6, 0]   # G[p + (x2, y0, z1)] for p in [0,4)^3, indexed [z][y][x]
    want0 = np.zeros((6, 6, 6))
    want0[1:5, 2:6, 0:4] = blk   # scattered to p + (x0, y2, z1)
    Ez = E.reshape(6, 6, 6, F)
    np.testing.assert_allclose(Ez[..., 0], want0, rtol=0, atol=1e-15)
    np.testing.assert_allclose(Ez[..., 1], np.full((6, 6, 6), blk.mean()), rtol=1e-14, atol=1e-15)
    want2 = np.full((6, 6, 6), 0.5)
    want2[1:5, 2:6, 0:4] += Gz[1:5, 0:4, 2:6, 3]
    np.testing.assert_allclose(Ez[..., 2], want2, rtol=0, atol=1e-15)
    assert np.all(E[:, 3:] == 0)


def test_unet_zero_weights_give_bias(oracle_mod):
    u = ls.make_unet_weights("zero", H, F)
    u["unet.proj.b"][:] = np.arange(F, dtype=np.float32) / 8
    pts, _ = ls.make_shapes(1, 300, seed=54)
    _, E = oracle_mod.encode_grid(ls.flatten_weights(ls.make_weights("he")), ls.flatten_unet(u), pts[0])
    assert np.array_equal(E, np.tile(np.arange(F) / 8, (216, 1)))


def test_grid_point_order_invariance(oracle_mod):
    pts, _ = ls.make_shapes(1, 500, seed=55)
    w = ls.flatten_weights(ls.make_weights("spread", calib=ls.load_calibration()))
    u = ls.flatten_unet(ls.make_unet_weights())
    G0, E0 = oracle_mod.encode_grid(w, u, pts[0])
    perm = np.random.default_rng(56).permutation(500)
    G1, E1 = oracle_mod.encode_grid(w, u, pts[0][perm])
    assert np.array_equal(G0, G1) and np.array_equal(E0, E1)


# ----------------------------------------------------------------------------- cell selection
def cell_boxes(lo, hi, M=6):
    ext = hi.astype(np.float64) - lo.astype(np.float64)
    a = ext / M
    idx = np.array([(c % M, (c // M) % M, c // (M * M)) for c in range(M ** 3)], np.float64)
    blo = lo + idx * a
    return blo, blo + a


def test_selection_superset_of_true_intersections(oracle_mod):
    """the margin guarantees no false negative — every cell whose box meets the other
    object's AABB (exact box-vs-box test in fp64, corners through the fp64 pose) is selected."""
    pts, _ = ls.make_shapes(8, 400, seed=57)
    pairs, poses = ls.make_pairs_poses(pts, 300, s=0.5, seed=58)
    u = ls.flatten_unet(ls.make_unet_weights())
    w = ls.flatten_weights(ls.make_weights("spread", calib=ls.load_calibration()))
    r = oracle_mod.query_cells(w, u, pts, pairs, poses)
    info = [oracle_mod.shape_prep(p) for p in pts]
    corners = np.array([[i & 1, (i >> 1) & 1, (i >> 2) & 1] for i in range(8)], np.float64)
    checked = 0
    for i in range(len(pairs)):
        for side in range(2):
            a, b = pairs[i, side], pairs[i, 1 - side]
            pa, pb = poses[i, side].astype(np.float64), poses[i, 1 - side].astype(np.float64)
            Ra, Rb = quat_R(pa[:4]), quat_R(pb[:4])
            blo, bhi = cell_boxes(info[a][0], info[a][1])
            olo, ohi = info[b][0].astype(np.float64), info[b][1].astype(np.float64)
            sel = np.array([(r["cells"][i, side, c // 32] >> (c % 32)) & 1 for c in range(216)], bool)
            assert sel.sum() == r["nsel"][i, side]
            for c in np.nonzero(~sel)[0]:
                # cell box corners in the other object's frame; separating-axis test (box vs AABB)
                cw = blo[c] + corners * (bhi[c] - blo[c])
                cb = (Rb.T @ ((Ra @ cw.T).T + pa[4:] - pb[4:]).T).T
                assert not boxes_intersect(cb, Ra, Rb, olo, ohi), (i, side, c)
                checked += 1
    assert checked > 1000


def quat_R(q):
    w, x, y, z = q / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def boxes_intersect(corners, Ra, Rb, lo, hi):
    """Separating-axis test of an oriented box (8 corners, in the AABB's frame) against [lo, hi]:
    15 axes (3 AABB faces, 3 box faces, 9 cross products); touching counts as intersecting."""
    Rrel = Rb.T @ Ra
    axes = [np.eye(3)[i] for i in range(3)] + [Rrel[:, j] for j in range(3)]
    axes += [np.cross(np.eye(3)[i], Rrel[:, j]) for i in range(3) for j in range(3)]
    box = np.array([[lo[0], hi[0]], [lo[1], hi[1]], [lo[2], hi[2]]])
    acorn = np.array([[box[0, i & 1], box[1, (i >> 1) & 1], box[2, (i >> 2) & 1]] for i in range(8)])
    for ax in axes:
        n = np.linalg.norm(ax)
        if n < 1e-12:
            continue
        p1, p2 = corners @ ax, acorn @ ax
        if p1.max() < p2.min() - 1e-9 * n or p2.max() < p1.min() - 1e-9 * n:
            return False
    return True


def test_selection_worked_example(oracle_mod):
    """tests/golden/cells_w2.json (hand-derived, cited there): two 26-point unit cubes, B shifted by
    0.9 along x; only A's x = 5 slab and B's x = 0 slab are within sqrt(3)/12 of the other box."""
    gold = json.load(open(os.path.join(GOLD, "cells_w2.json")))
    c = cube26()
    pts = np.stack([c, c])
    u = ls.flatten_unet(ls.make_unet_weights())
    w = ls.flatten_weights(ls.make_weights("spread", calib=ls.load_calibration()))
    pr = np.array([[0, 1]], np.int32)
    for case in gold["cases"]:
        po = np.stack([pose(t=case["tA"]), pose(q=case.get("qB", (1, 0, 0, 0)), t=case["tB"])])[None]
        r = oracle_mod.query_cells(w, u, pts, pr, po, n_threads=1)
        for side, key in ((0, "selA"), (1, "selB")):
            sel = [c for c in range(216) if (r["cells"][0, side, c // 32] >> (c % 32)) & 1]
            assert sel == case[key], (case["name"], side)
        assert np.isneginf(r["logits"][0]) == case["short_circuit"]


# ----------------------------------------------------------------------------- whole query
def test_query_cells_closed_form(oracle_mod):
    """Identity encoder + U-Net probe + head_weights(): logit = max(tx) + 2 max(e0) + 3 max(qcx) with
    e0 = mean of E0 over the selected cells (E0 from the probe's closed form, pinned above)."""
    pts, _ = ls.make_shapes(6, 400, seed=59)
    pairs, poses = ls.make_pairs_poses(pts, 40, s=0.4, seed=60)
    w = head_weights()
    r = oracle_mod.query_cells(w, unet_probe(), pts, pairs, poses)
    n = 0
    for i in range(len(pairs)):
        if r["nsel"][i].sum() == 0:
            assert np.isneginf(r["logits"][i])
            continue
        e0 = []
        for side in range(2):
            sel = np.array([(r["cells"][i, side, c // 32] >> (c % 32)) & 1 for c in range(216)], bool)
            E = r["grids"][pairs[i, side]]
            e0.append(E[sel, 0].mean() if sel.any() else 0.0)
            assert abs(r["emb"][i, side, 0] - e0[-1]) <= 1e-15
        qx = [canon1(poses[i, s, :4]) for s in range(2)]
        want = max(poses[i, 0, 4], poses[i, 1, 4]) + 2 * max(e0) + 3 * max(qx)
        assert abs(r["logits"][i] - want) <= 1e-12
        n += 1
    assert n > 10


def canon1(q):
    q = q.astype(np.float64) / np.linalg.norm(q.astype(np.float64))
    return q[1] * np.sign(q[np.nonzero(q)[0][0]])


def test_query_cells_symmetries(oracle_mod):
    pts, _ = ls.make_shapes(5, 300, seed=61)
    pairs, poses = ls.make_pairs_poses(pts, 20, s=0.5, seed=62)
    u = ls.flatten_unet(ls.make_unet_weights())
    w = ls.flatten_weights(ls.make_weights("spread", calib=ls.load_calibration()))
    r0 = oracle_mod.query_cells(w, u, pts, pairs, poses)
    r1 = oracle_mod.query_cells(w, u, pts, pairs[:, ::-1].copy(), poses[:, ::-1].copy())
    assert np.array_equal(r0["logits"], r1["logits"]) and np.array_equal(r0["nsel"], r1["nsel"][:, ::-1])
    neg = poses.copy()
    neg[:, :, :4] *= -1
    r2 = oracle_mod.query_cells(w, u, pts, pairs, neg)
    for k in ("logits", "nsel", "cells", "emb"):
        assert np.array_equal(r0[k], r2[k]), k


def test_unet_global_max_probe(oracle_mod):
    """Q28's alternative reading (P:421 'max pooling to get global features'): with the delta-kernel
    probe the global channel is the MAX of the block instead of its mean; everything else unchanged."""
    pts, _ = ls.make_shapes(2, 600, seed=53)
    G, E = oracle_mod.encode_grid(identity_encoder(), unet_probe(), pts[0], global_max=True)
    _, E_avg = oracle_mod.encode_grid(identity_encoder(), unet_probe(), pts[0])
    blk = G.reshape(6, 6, 6, H)[1:5, 0:4, 2:6, 0]
    np.testing.assert_allclose(E[:, 1], np.full(216, blk.max()), rtol=0, atol=0)
    assert np.array_equal(E[:, [0, 2]], E_avg[:, [0, 2]]) and blk.max() > blk.mean()
