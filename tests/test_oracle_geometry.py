"""Pins of the oracle's geometry (O0-O5) against things other than itself.

Each test names what fixes the expected value: the hand-derived worked example W1
(tests/golden/w1_boxes.json), closed forms, library routines used independently
(scipy Rotation), brute force in exact/fp64 arithmetic, or exact invariants.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import locc_synth as ls
from conftest import cube26, pose

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def zero_weights(H=256, F=64):
    return ls.flatten_weights(ls.make_weights("zero", H, F), H, F)


def run_pair(oracle_mod, ptsA, ptsB, pA, pB, w=None, M=6, H=256, F=64, emul=False):
    K = ptsA.shape[0]
    assert ptsB.shape[0] == K
    pts = np.stack([ptsA, ptsB])
    pairs = np.array([[0, 1]], np.int32)
    poses = np.stack([pA, pB])[None]
    if w is None:
        w = zero_weights(H, F)
    return oracle_mod.query(w, pts, pairs, poses, M=M, H=H, F=F, bf16_emul=emul, n_threads=1)


def mask_bits(words, K):
    return np.array([(words[k // 32] >> (k % 32)) & 1 for k in range(K)], bool)


# ----------------------------------------------------------------------------- W1 worked example
def test_w1_worked_example_counts(oracle_mod):
    g = json.load(open(os.path.join(GOLD, "w1_boxes.json")))
    c = cube26()
    lo, hi, eps2, cell = oracle_mod.shape_prep(c, g["M"])
    assert eps2 == np.float32(g["eps2"])  # 1/48 rounded once to fp32
    assert len(set(cell.tolist())) == 26  # every point owns a cell (cells 0, 3, 5 per axis)
    for row in g["rows"]:
        r = run_pair(oracle_mod, c, c, pose(), pose(row["qB"], row["tB"]))
        assert tuple(r["kept"][0]) == (row["nA"], row["nB"]), row
        assert tuple(r["occ"][0]) == (row["CA"], row["CB"]), row
        if row["short"]:
            assert r["probs"][0] == 0.0 and r["labels"][0] == 0 and r["logits"][0] == -np.inf
        else:
            # zero weights: logit = 0 exactly, p = sigma(0) = 0.5, tie -> negative
            assert r["logits"][0] == 0.0 and r["probs"][0] == 0.5 and r["labels"][0] == 0


def test_w1_mask_order_rotation(oracle_mod):
    """Row 6 of W1: 180 deg about z keeps B's x=+1/2 face; identity keeps B's x=-1/2 face."""
    c = cube26()
    r_id = run_pair(oracle_mod, c, c, pose(), pose((1, 0, 0, 0), (1, 0, 0)))
    r_rot = run_pair(oracle_mod, c, c, pose(), pose((0, 0, 0, 1), (1, 0, 0)))
    K = c.shape[0]
    mA_id, mB_id = mask_bits(r_id["masks"][0, 0], K), mask_bits(r_id["masks"][0, 1], K)
    mA_rot, mB_rot = mask_bits(r_rot["masks"][0, 0], K), mask_bits(r_rot["masks"][0, 1], K)
    assert np.array_equal(mA_id, c[:, 0] == 0.5) and np.array_equal(mA_rot, c[:, 0] == 0.5)
    assert np.array_equal(mB_id, c[:, 0] == -0.5)
    assert np.array_equal(mB_rot, c[:, 0] == 0.5)


# ----------------------------------------------------------------------------- O0 pins
def test_eps_is_half_cell_diagonal(oracle_mod):
    """eps = distance from a cell centre to its vertex, computed geometrically."""
    pts, _ = ls.make_shapes(24, 300, seed=11)
    for M in (5, 6, 7):
        for s in range(pts.shape[0]):
            lo, hi, eps2, _ = oracle_mod.shape_prep(pts[s], M)
            lo64, hi64 = lo.astype(np.float64), hi.astype(np.float64)
            centre = lo64 + (hi64 - lo64) / M / 2  # centre of cell (0,0,0)
            vertex = lo64
            d2 = float(np.sum((centre - vertex) ** 2))
            assert abs(float(eps2) - d2) <= 2e-7 * d2
            assert np.array_equal(lo, pts[s].min(0)) and np.array_equal(hi, pts[s].max(0))


def test_cell_ids_contain_their_points(oracle_mod):
    """Each point lies in the closed box of its cell (exact rational check); max face -> M-1."""
    pts, _ = ls.make_shapes(6, 200, seed=12)
    for M in (1, 3, 6):
        for s in range(pts.shape[0]):
            lo, hi, _, cell = oracle_mod.shape_prep(pts[s], M)
            for k in range(pts.shape[1]):
                c = [cell[k] % M, (cell[k] // M) % M, cell[k] // (M * M)]
                for d in range(3):
                    p, l, h = Fraction(float(pts[s, k, d])), Fraction(float(lo[d])), Fraction(float(hi[d]))
                    a = (h - l) / M
                    assert l + c[d] * a <= p <= l + (c[d] + 1) * a
                    if p == h:
                        assert c[d] == M - 1
                    u = (p - l) / a
                    if c[d] < M - 1 and abs(u - round(u)) > Fraction(1, 10 ** 9):
                        assert c[d] == int(u)  # floor, away from fp64-ambiguous boundaries


def test_degenerate_axis_goes_to_cell_zero(oracle_mod):
    p = np.array([[0, 0, 0], [1, 0, 0], [0.5, 0, 0]], np.float32)  # y, z extents 0
    lo, hi, eps2, cell = oracle_mod.shape_prep(p, 6)
    assert cell.tolist() == [0, 5, 3]
    assert eps2 == np.float32(0.25 * (1 / 36))


# ----------------------------------------------------------------------------- O1-O3 pins
def random_quats(n, rng):
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return q.astype(np.float32)


def test_same_pose_gives_exact_identity(oracle_mod):
    """q_A = q_B, t_A = t_B => R = I and t = 0 exactly (the grouped product cancels exactly)."""
    rng = np.random.default_rng(5)
    for q in random_quats(500, rng):
        t = rng.uniform(-1, 1, 3).astype(np.float32)
        R, tt, R2, t2 = oracle_mod.rel_transform(pose(q, t), pose(q, t))
        assert np.array_equal(R, np.eye(3, dtype=np.float32)) and np.array_equal(R2, R)
        assert np.all(tt == 0) and np.all(t2 == 0)


def test_relative_transform_matches_scipy(oracle_mod):
    rng = np.random.default_rng(6)
    qa, qb = random_quats(300, rng), random_quats(300, rng)
    for i in range(300):
        ta, tb = rng.uniform(-1, 1, 3).astype(np.float32), rng.uniform(-1, 1, 3).astype(np.float32)
        R, t, R2, t2 = oracle_mod.rel_transform(pose(qa[i], ta), pose(qb[i], tb))
        RA = Rotation.from_quat(qa[i].astype(np.float64)[[1, 2, 3, 0]]).as_matrix()
        RB = Rotation.from_quat(qb[i].astype(np.float64)[[1, 2, 3, 0]]).as_matrix()
        d = ta.astype(np.float64) - tb.astype(np.float64)
        np.testing.assert_allclose(R, RB.T @ RA, atol=2e-7)
        np.testing.assert_allclose(t, RB.T @ d, atol=5e-7)
        np.testing.assert_allclose(R2, RA.T @ RB, atol=2e-7)
        np.testing.assert_allclose(t2, -RA.T @ d, atol=5e-7)
        # round trip T_AB o T_BA ~ I
        np.testing.assert_allclose(R2.astype(np.float64) @ R, np.eye(3), atol=1e-6)
        np.testing.assert_allclose(R2.astype(np.float64) @ t + t2, 0, atol=1e-6)


def test_quaternion_sign_is_irrelevant(oracle_mod):
    """q -> -q on either pose gives bitwise-identical R and t."""
    rng = np.random.default_rng(7)
    qa, qb = random_quats(300, rng), random_quats(300, rng)
    for i in range(300):
        ta, tb = rng.uniform(-1, 1, 3).astype(np.float32), rng.uniform(-1, 1, 3).astype(np.float32)
        a = oracle_mod.rel_transform(pose(qa[i], ta), pose(qb[i], tb))
        b = oracle_mod.rel_transform(pose(-qa[i], ta), pose(qb[i], tb))
        c = oracle_mod.rel_transform(pose(qa[i], ta), pose(-qb[i], tb))
        for x, y, z in zip(a, b, c):
            assert np.array_equal(x, y) and np.array_equal(x, z)


def test_axis_half_turns_are_integer(oracle_mod):
    for q, R in [((0, 1, 0, 0), np.diag([1, -1, -1])), ((0, 0, 1, 0), np.diag([-1, 1, -1])),
                 ((0, 0, 0, 1), np.diag([-1, -1, 1]))]:
        Rr, t, _, _ = oracle_mod.rel_transform(pose(q, (0.25, 0.5, -0.75)), pose())
        assert np.array_equal(Rr, R.astype(np.float32))
        assert np.array_equal(t, np.array([0.25, 0.5, -0.75], np.float32))


# ----------------------------------------------------------------------------- O4 pins
def brute_force_keep(ptsA, ptsB, pA, pB, M):
    """Exact-ish fp64 crop of A against B: scipy rotations, unrounded transform, exact distance."""
    RA = Rotation.from_quat(pA[[1, 2, 3, 0]].astype(np.float64)).as_matrix()
    RB = Rotation.from_quat(pB[[1, 2, 3, 0]].astype(np.float64)).as_matrix()
    w = ptsA.astype(np.float64) @ RA.T + pA[4:].astype(np.float64)
    pb = (w - pB[4:].astype(np.float64)) @ RB
    lo, hi = ptsB.min(0).astype(np.float64), ptsB.max(0).astype(np.float64)
    d = np.linalg.norm(np.maximum(np.maximum(lo - pb, pb - hi), 0), axis=1)
    eps = 0.5 * np.linalg.norm((hi - lo) / M)
    return d <= eps, d - eps


def test_crop_matches_brute_force(oracle_mod):
    pts, _ = ls.make_shapes(12, 600, seed=13)
    pairs, poses = ls.make_pairs_poses(pts, 200, s=0.5, seed=14)
    r = oracle_mod.query(zero_weights(), pts, pairs, poses, n_threads=0)
    K = pts.shape[1]
    in_band = mismatched = 0
    for i in range(len(pairs)):
        a, b = pairs[i]
        for side, (x, y, px, py) in enumerate([(a, b, poses[i, 0], poses[i, 1]), (b, a, poses[i, 1], poses[i, 0])]):
            exact, margin = brute_force_keep(pts[x], pts[y], px, py, 6)
            got = mask_bits(r["masks"][i, side], K)
            assert r["kept"][i, side] == got.sum()  # n = popcount(mask)
            bad = got != exact
            in_band += int((np.abs(margin) <= 2e-6).sum())
            mismatched += int(bad.sum())
            assert np.all(np.abs(margin[bad]) <= 2e-6), (i, side, margin[bad])
    assert in_band < 50


def binary_tetrahedral():
    h = Fraction(1, 2)
    qs = []
    for i in range(4):
        for s in (1, -1):
            q = [Fraction(0)] * 4
            q[i] = Fraction(s)
            qs.append(q)
    for sw in (1, -1):
        for sx in (1, -1):
            for sy in (1, -1):
                for sz in (1, -1):
                    qs.append([sw * h, sx * h, sy * h, sz * h])
    return qs


def qmul(a, b):
    return [a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3],
            a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2],
            a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1],
            a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0]]


def qrot(q, v):
    p = qmul(qmul(q, [Fraction(0)] + v), [q[0], -q[1], -q[2], -q[3]])
    return p[1:]


def test_common_rigid_motion_exact_group(oracle_mod):
    """Poses and a common motion G from the 24-element binary tetrahedral group with dyadic
    translations: every product is exact, so the masks must be bitwise identical."""
    G = binary_tetrahedral()
    assert len(G) == 24
    pts, _ = ls.make_shapes(4, 400, seed=15)
    rng = np.random.default_rng(16)
    dy = lambda: [Fraction(int(v), 64) for v in rng.integers(-8, 9, 3)]
    pairs = np.array([[0, 1], [2, 3], [1, 1]], np.int32)
    for trial in range(40):
        qa, qb, g = G[rng.integers(24)], G[rng.integers(24)], G[rng.integers(24)]
        ta, tb, tg = dy(), dy(), dy()
        base = np.array([[[float(x) for x in qa + ta], [float(x) for x in qb + tb]]] * 3, np.float32)
        qa2, qb2 = qmul(g, qa), qmul(g, qb)
        ta2 = [x + y for x, y in zip(qrot(g, ta), tg)]
        tb2 = [x + y for x, y in zip(qrot(g, tb), tg)]
        moved = np.array([[[float(x) for x in qa2 + ta2], [float(x) for x in qb2 + tb2]]] * 3, np.float32)
        r0 = oracle_mod.query(zero_weights(), pts, pairs, base, n_threads=1)
        r1 = oracle_mod.query(zero_weights(), pts, pairs, moved, n_threads=1)
        assert np.array_equal(r0["masks"], r1["masks"]) and np.array_equal(r0["kept"], r1["kept"])


def test_separated_and_coincident(oracle_mod):
    """far apart -> empty on both sides; coincident identical -> everything kept."""
    pts, _ = ls.make_shapes(3, 500, seed=17)
    for s in range(3):
        far = run_pair(oracle_mod, pts[s], pts[s], pose(), pose(t=(3, 0, 0)))
        assert tuple(far["kept"][0]) == (0, 0) and far["probs"][0] == 0.0
        same = run_pair(oracle_mod, pts[s], pts[s], pose(), pose())
        assert tuple(same["kept"][0]) == (500, 500)


def test_input_validation(oracle_mod):
    pts, _ = ls.make_shapes(2, 50, seed=18)
    w = zero_weights()
    bad_pair = np.array([[0, 2]], np.int32)
    with pytest.raises(ValueError):
        oracle_mod.query(w, pts, bad_pair, np.zeros((1, 2, 7), np.float32) + pose())
    zq = np.zeros((1, 2, 7), np.float32)
    with pytest.raises(ValueError):
        oracle_mod.query(w, pts, np.array([[0, 1]], np.int32), zq)
